# PDL trigger placement for the compute kernels (frame GEMM): early vs late
rm -rf paper_0707_2347_b200/build paper_0707_2347_b200/libwinomem_b200.so
WM_NVCC_FLAGS=-DWM_PDL_LATE_COMPUTE=0 python -m paper_0707_2347_b200.build > gpurun_out/r36_build.log 2>&1
for cfg in C2 C1 C4; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg early', d['ms_per_step'], (d.get('parity') or {}).get('ok'))" >> gpurun_out/r36.log 2>&1
done
