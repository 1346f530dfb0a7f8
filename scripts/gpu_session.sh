WM_OPTS=dag=3 WM_TRACE_DUMP=gpurun_out/trace_c2.json timeout 300 python scripts/trace_step.py C2 > gpurun_out/trace_c2.log 2>&1; echo trace rc=$?; tail -c 1800 gpurun_out/trace_c2.log
