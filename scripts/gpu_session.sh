timeout 900 python -m pytest tests -m gpu -x -q -k "acceptance or golden_small or native_dist or error_goldens" > gpurun_out/pytest_gpu_e.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_e.log
cat gpurun_out/acceptance_b200.log
timeout 300 python scripts/direct_probe.py > gpurun_out/direct_probe.log 2>&1; echo probe rc=$?
