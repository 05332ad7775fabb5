# final round-2 evidence: GPU tests, smoke, default bench, reference arm, N=2 plumbing (gloo, one device),
# and ncu (--set full + launch lists) of every default-bench search launch and of one 10K insert into C2
O=gpurun_out/fin5
mkdir -p $O
(time timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900) > $O/gpu_tests.log 2>&1
(time timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > $O/smoke.log 2>&1
(time timeout 2400 python bench.py) > $O/bench.json 2> $O/bench.err
(time timeout 1200 python bench.py --impl reference --steps 3 --warmup 1) > $O/bench_ref.json 2> $O/bench_ref.err
SVF_SAME_DEVICE=1 SVF_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config C2 --steps 20 --warmup 5 --no-extra --no-cpu > $O/bench_n2_samedevice.json 2> $O/bench_n2.err
NCU="ncu --clock-control none --profile-from-start off"
summ() {  # rep launches nq itopk out config note
  python tools/ncu_summary.py --rep $1.ncu-rep ${2:+--launches $2} --nq $3 --itopk $4 --out $5 --latest --config $6 --note "$7" > $5.log 2>&1
  ncu -i $1.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $5_sass.csv.gz
  rm -f $1.ncu-rep
}
for C in "C2 10 16" "C3 20 35" "C4 192 288" "C2G 96 120"; do
  set -- $C
  timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_$1.csv \
    python bench.py --config $1 --ncu --itopk $2 --max-iter $3 --steps 10 --warmup 3 > $O/ncu_list_$1.log 2>&1
  timeout 1200 $NCU --set full --import-source on -k regex:search -c 2 -o $O/search_$1 \
    python bench.py --config $1 --ncu --itopk $2 --max-iter $3 --steps 2 --warmup 3 > $O/ncu_full_$1.log 2>&1
  summ $O/search_$1 $O/launches_$1.csv 10000 $2 $O/r02_search_$1 $1 "bench.py --config $1 --itopk $2 --max-iter $3 (the bench's launch)"
done
timeout 1200 $NCU --set full -o $O/insert_c2 python tools/insert_prof.py > $O/ncu_insert.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_insert.csv python tools/insert_prof.py > $O/ncu_insert_list.log 2>&1
python tools/ncu_summary.py --rep $O/insert_c2.ncu-rep --launches $O/launches_insert.csv --nq 10000 --itopk 128 --out $O/r02_insert_c2 --note "one 10K insert into C2 (L_build 256, L_insert 128): every kernel of svf_insert" > /dev/null 2>&1
timeout 900 $NCU --set full --import-source on -k regex:search_lp -c 1 -o $O/lp_c2 python tools/lp_prof.py > $O/ncu_lp_c2.log 2>&1
python tools/ncu_summary.py --rep $O/lp_c2.ncu-rep --nq 4096 --itopk 128 --out $O/r02_lp_c2 --note "K-S-L, C2 itopk 128, 4096 fresh vectors (the insert sub-batch shape), final round-2 kernel" > /dev/null 2>&1
ncu -i $O/lp_c2.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $O/lp_c2_sass.csv.gz
rm -f $O/*.ncu-rep
du -sh $O
