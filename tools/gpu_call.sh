O=gpurun_out/ak
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 > $O/parity.log 2>&1
timeout 600 python tools/pool_probe.py --itopks 128 --batches 4096,10000 --no-trace --out $O/c2.json > $O/c2.log 2>&1
timeout 600 python bench.py --config C2G --no-extra --no-cpu --no-insert --steps 50 --warmup 10 --itopk 96 --max-iter 120 > $O/c2g.json 2> $O/c2g.err
