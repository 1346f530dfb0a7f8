# frame GEMM tiling sweep on C2 (and C4 gemm for 2 configs)
for cfg in 0 3201 3202 3204 6401 6402 6404; do
  WM_FRAME_CFG=$cfg timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fsweep_$cfg.log 2>&1
done
for eng in 0; do
  WM_GEMM_ENGINE=$eng timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fsweep_eng$eng.log 2>&1
done
