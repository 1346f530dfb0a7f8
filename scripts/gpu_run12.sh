set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "midsize or config_full or partition or leaf_i8" > gpurun_out/pytest_raw16.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_raw16.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_r16.log 2>&1
timeout 300 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_r16.log 2>&1
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1
