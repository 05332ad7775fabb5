O=gpurun_out/ai
mkdir -p $O
timeout 600 env SVF_LIB=paper_2601_08528_b200/libsvf_kspf.so python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "search or handoff or forget" > $O/parity.log 2>&1
for v in main kspf main2 kspf2; do
  L=paper_2601_08528_b200/libsvf.so; case $v in kspf*) L=paper_2601_08528_b200/libsvf_kspf.so;; esac
  SVF_LIB=$L timeout 600 python bench.py --config C2 --no-extra --no-cpu --no-insert --steps 100 --warmup 10 --itopk 10 --max-iter 16 > $O/c2_$v.json 2> $O/c2_$v.err
done
for v in main kspf; do
  L=paper_2601_08528_b200/libsvf.so; case $v in kspf*) L=paper_2601_08528_b200/libsvf_kspf.so;; esac
  SVF_LIB=$L timeout 900 python bench.py --config C3 --no-extra --no-cpu --no-insert --steps 50 --warmup 10 --itopk 20 --max-iter 35 > $O/c3_$v.json 2> $O/c3_$v.err
done
