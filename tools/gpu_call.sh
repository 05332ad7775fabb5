O=gpurun_out/aa
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_traces.py -q -x --timeout 300 > $O/parity.log 2>&1
timeout 600 python tools/pool_probe.py --itopks 128 --batches 4096 --no-trace --out $O/c2.json > $O/c2.log 2>&1
