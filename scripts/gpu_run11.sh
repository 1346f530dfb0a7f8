set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "leaf_i8 or classical_vs_oracle or midsize" > gpurun_out/pytest_tma.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tma.log
timeout 300 python scripts/leaf_sweep.py > gpurun_out/leaf_sweep4.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_tma.log 2>&1
timeout 300 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_tma.log 2>&1
