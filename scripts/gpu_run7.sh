set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "leaf_i8 or classical_vs_oracle" > gpurun_out/pytest_i8c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_i8c.log
timeout 300 python scripts/leaf_sweep.py > gpurun_out/leaf_sweep2.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --fuse 0 --leaf 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_i.log 2>&1
