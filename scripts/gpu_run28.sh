# round-1 re-entry: verify HEAD on a fresh box (tests, smoke, bench, ncu)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r28_smi.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r28_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r28_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r28_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r28_bench_c2.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r28_bench_ref.log 2>&1
for cfg in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/r28_bench_${cfg}.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r28_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r28_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_direct|k_frame_prep_limbs|k_frame_comb|k_group" -s 200 -c 6 -o gpurun_out/r28_prof_c2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r28_ncu_full.log 2>&1
