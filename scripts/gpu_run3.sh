set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "leaf_i8 or classical_vs_oracle or primitive" > gpurun_out/pytest_i8.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_i8.log
timeout 300 python scripts/microbench.py > gpurun_out/microbench.log 2>&1
echo "micro rc=$?" >> gpurun_out/microbench.log
timeout 300 python bench.py --steps 5 --warmup 3 --fuse 0 --leaf 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_i8.log 2>&1
timeout 120 python bench.py --config C1 --steps 5 --warmup 3 --fuse 0 --leaf 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_i8.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "midsize or config_full or golden" > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
