set -x
timeout 300 python scripts/frame_gemm_probe.py > gpurun_out/frame_probe.log 2>&1
bash scripts/frame_sweep.sh
