timeout 600 python -m pytest tests -m gpu -x -q -k "arena or host_u32" > gpurun_out/pytest_gpu_j.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_j.log
for sp in 0 1; do
WM_OPTS=io_split=$sp,dag=3 WM_TRACE_DUMP=gpurun_out/trace_e2e_split$sp.json timeout 300 python scripts/trace_step.py C2 --e2e > gpurun_out/trace_e2e_split$sp.log 2>&1; echo trace rc=$?; tail -c 1500 gpurun_out/trace_e2e_split$sp.log
done
