# full GPU tests + smoke + the default bench (C2 headline, C3, C4, C2G) + the reference (oracle) arm
O=gpurun_out/y
mkdir -p $O
(time timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900) > $O/gpu_tests.log 2>&1
(time timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > $O/smoke.log 2>&1
(time timeout 2400 python bench.py) > $O/bench.json 2> $O/bench.err
(time timeout 1200 python bench.py --impl reference --steps 3 --warmup 1) > $O/bench_ref.json 2> $O/bench_ref.err
