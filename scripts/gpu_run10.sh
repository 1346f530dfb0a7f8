set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2_full.log 2>&1
timeout 300 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_full.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8 -s 40 -c 2 -o gpurun_out/prof_frame_gemm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
