timeout 120 python scripts/leaf_one.py 1024 0 > gpurun_out/dmma1024.log 2>&1
timeout 120 python scripts/leaf_one.py 512 0 >> gpurun_out/dmma1024.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5_24.log 2>&1
