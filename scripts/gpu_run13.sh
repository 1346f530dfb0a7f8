set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "midsize or config_full or partition or golden" > gpurun_out/pytest_13.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_13.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2_13.log 2>&1
timeout 300 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_13.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_plain13.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3200 --csv --log-file gpurun_out/launches_c2_13.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch13.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tma -s 40 -c 2 -o gpurun_out/prof_frame_tma python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full13.log 2>&1
