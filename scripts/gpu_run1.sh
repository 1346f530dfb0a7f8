set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not options or default" --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --fuse 0 > gpurun_out/bench_c2.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_c2.log
timeout 120 python bench.py --config C1 --steps 5 --warmup 3 --fuse 0 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
