# final: full GPU suite + smoke, ncu captures of the additions class (k_group) and the C4 frame GEMM
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=5 > gpurun_out/r58_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r58_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r58_smoke.log 2>&1
echo "exit $?" >> gpurun_out/r58_smoke.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_group" -s 2 -c 4 -o gpurun_out/r58_prof_group python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r58_ncu_group.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_direct" -s 50 -c 2 -o gpurun_out/r58_prof_gemm_c4 python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r58_ncu_gemm_c4.log 2>&1
