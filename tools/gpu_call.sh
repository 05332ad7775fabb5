O=gpurun_out/ac
mkdir -p $O
timeout 600 python tools/pool_probe.py --itopks 128 --batches 1808,2500,3334,4096,5000 --no-trace --no-insert --out $O/c2.json > $O/c2.log 2>&1
