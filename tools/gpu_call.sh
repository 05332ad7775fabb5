O=gpurun_out/x
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 > $O/parity.log 2>&1
timeout 600 python tools/pool_probe.py --itopks 128 --batches 4096,10000 --no-trace --out $O/c2.json > $O/c2.log 2>&1
timeout 600 python bench.py --config C2G --no-extra --no-cpu --no-insert --steps 50 --warmup 10 --itopk 96 --max-iter 120 > $O/c2g.json 2> $O/c2g.err
timeout 600 python bench.py --config C2 --no-extra --no-cpu --no-insert --steps 100 --warmup 10 --itopk 10 --max-iter 16 > $O/c2h.json 2> $O/c2h.err
timeout 900 python tools/pool_probe.py --config C4 --build-itopk 512 --itopks 192 --batches 10000 --no-insert --no-trace --out $O/c4.json > $O/c4.log 2>&1
