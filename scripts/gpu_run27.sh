timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5_27.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_27.log 2>&1
