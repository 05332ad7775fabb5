O=gpurun_out/aj
mkdir -p $O
for v in main nofpf; do
  L=paper_2601_08528_b200/libsvf_$v.so; [ $v = main ] && L=paper_2601_08528_b200/libsvf.so
  SVF_LIB=$L timeout 900 python bench.py --config C3 --no-extra --no-cpu --steps 20 --warmup 5 --itopk 20 --max-iter 35 > $O/c3_$v.json 2> $O/c3_$v.err
  SVF_LIB=$L timeout 600 python tools/pool_probe.py --itopks 128 --batches 4096 --no-trace --out $O/c2_$v.json > $O/c2_$v.log 2>&1
done
