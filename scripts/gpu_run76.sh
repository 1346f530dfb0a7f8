# round-1 final measurement (final code, r76): benches C1-C5 + reference arm, ncu launch list + full captures (C2)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r76_smi.log 2>&1
timeout 900 python bench.py > gpurun_out/r76_bench_C2.log 2>&1
for cfg in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/r76_bench_${cfg}.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r76_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r76_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r76_ncu_launch.log 2>&1
timeout 300 python scripts/trace_step.py C2 > gpurun_out/r76_trace.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r76_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r76_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r76_smoke.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_direct|k_frame_prep_limbs|k_frame_comb" -s 300 -c 6 -o gpurun_out/r76_prof_c2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r76_ncu_full.log 2>&1
