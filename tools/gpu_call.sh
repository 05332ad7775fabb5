O=gpurun_out/af
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 > $O/parity.log 2>&1
timeout 900 python bench.py --config C4 --no-extra --no-cpu --no-insert --steps 20 --warmup 5 --itopk 192 --max-iter 288 > $O/c4.json 2> $O/c4.err
