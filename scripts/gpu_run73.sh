for cfg in C2 C3; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], (d.get('parity') or {}).get('ok'))" >> gpurun_out/r73_bench.log 2>&1
done
