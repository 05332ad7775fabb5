O=gpurun_out/z
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "large_pool or search" > $O/parity.log 2>&1
timeout 900 python bench.py --config C4 --no-extra --no-cpu --no-insert --steps 20 --warmup 5 --itopk 192 --max-iter 288 > $O/c4.json 2> $O/c4.err
NCU="ncu --clock-control none --profile-from-start off"
timeout 1200 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:search -c 1 python bench.py --config C4 --ncu --itopk 192 --max-iter 288 --steps 2 --warmup 3 > $O/ncu_c4.log 2>&1
