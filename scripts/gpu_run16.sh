set -x
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_plain16.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c2_16.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch16.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_direct|k_frame_prep_limbs|k_frame_comb" -s 60 -c 3 -o gpurun_out/prof_frame_direct python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full16.log 2>&1
