set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "leaf_i8 or classical_vs_oracle" > gpurun_out/pytest_i8d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_i8d.log
timeout 300 python scripts/leaf_sweep.py > gpurun_out/leaf_sweep3.log 2>&1
