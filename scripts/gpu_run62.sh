for cfg in C2 C3; do
  for f in 0 1064 1128; do
    WM_FRAME_CFG=$f timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', 'cfg=$f', d['ms_per_step'], (d.get('parity') or {}).get('ok'), round(d['frame_breakdown_s']['gemm']*1e3,3))" >> gpurun_out/r62_bench.log 2>&1
  done
done
