for e in 0 1; do
  if [ $e = 1 ]; then export WM_WIDE_ALL=1; fi
  for cfg in C2 C4; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg wide_all=$e', d['ms_per_step'], (d.get('parity') or {}).get('ok'))" >> gpurun_out/r77_bench.log 2>&1
  done
done
