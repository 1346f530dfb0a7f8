set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "midsize or config_full or leaf_i8" > gpurun_out/pytest_frame.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_frame.log
timeout 300 python bench.py --steps 5 --warmup 3 --fuse 1 --leaf 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_f.log 2>&1
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --fuse 1 --leaf 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_f.log 2>&1
