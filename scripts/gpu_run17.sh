set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "midsize or config_full or golden or partition or host" > gpurun_out/pytest_dag.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_dag.log
for cfg in C1 C2 C3 C4; do
timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${cfg}_dag.log 2>&1
done
