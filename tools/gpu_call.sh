# K-S-L gather: unconditional row loads at exact geometries, one query float4 per v per round
O=gpurun_out/v
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 > $O/parity.log 2>&1
timeout 600 python tools/pool_probe.py --itopks 128 --batches 4096,10000 --no-trace --out $O/c2.json > $O/c2.log 2>&1
timeout 600 python bench.py --config C2G --no-extra --no-cpu --no-insert --steps 50 --warmup 10 --itopk 96 --max-iter 120 > $O/c2g.json 2> $O/c2g.err
timeout 600 python bench.py --config C2 --no-extra --no-cpu --no-insert --steps 100 --warmup 10 --itopk 10 --max-iter 16 > $O/c2h.json 2> $O/c2h.err
