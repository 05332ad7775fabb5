# insert: detour selection PDL-chained behind the insert search (per-vertex done flags) vs serial
O=gpurun_out/q
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "insert or build or large_pool" > $O/parity1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_traces.py -q -x --timeout 120 > $O/parity.log 2>&1
for ch in 1 0; do
  SVF_INS_CHAIN=$ch timeout 300 python tools/pool_probe.py --itopks 128 --batches 4096 --no-trace --out $O/c2_chain$ch.json > $O/c2_chain$ch.log 2>&1
done
