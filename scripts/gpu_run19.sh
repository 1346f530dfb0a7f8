set -x
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2_19.log 2>&1
timeout 300 python bench.py --config C1 --steps 10 --warmup 3 > gpurun_out/bench_c1_19.log 2>&1
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_19.log 2>&1
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_19.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_19.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_plain19.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c2_19.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch19.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_direct" -s 30 -c 1 -o gpurun_out/prof_gemm_direct19 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full19.log 2>&1
