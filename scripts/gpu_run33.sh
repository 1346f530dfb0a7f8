for cfg in C2 C1 C4; do timeout 300 python scripts/trace_step.py $cfg >> gpurun_out/r33_trace.log 2>&1; done
WM_OPTS=dag=4 timeout 300 python scripts/trace_step.py C2 >> gpurun_out/r33_trace.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-400 >> gpurun_out/r33_trace.log
