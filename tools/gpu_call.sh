# parity + timing of the K-S-L search after the row-prefetch change
O=gpurun_out/h
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 > $O/parity.log 2>&1
timeout 600 python tools/pool_probe.py --itopks 128 --batches 4096,10000 --no-trace --out $O/c2.json > $O/c2.log 2>&1
timeout 900 python tools/pool_probe.py --config C4 --build-itopk 512 --itopks 192 --batches 10000 --no-insert --no-trace --out $O/c4.json > $O/c4.log 2>&1
NCU="ncu --clock-control none --profile-from-start off"
timeout 900 $NCU --set full --import-source on -k regex:search_lp -c 1 -o $O/lp_c2 python tools/lp_prof.py > $O/ncu_lp_c2.log 2>&1
python tools/ncu_summary.py --rep $O/lp_c2.ncu-rep --nq 4096 --itopk 128 --out $O/r02_lp_c2 --note "K-S-L, C2 itopk 128, 4096 fresh vectors" > /dev/null 2>&1
ncu -i $O/lp_c2.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $O/lp_c2_sass.csv.gz
rm -f $O/*.ncu-rep
