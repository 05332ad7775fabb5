O=gpurun_out/ae
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/gpu_tests.log 2>&1
