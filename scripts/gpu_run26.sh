for cfg in C5 C2 C3 C4; do
  echo "== $cfg" >> gpurun_out/run26.log
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], (d.get('parity') or {}).get('ok'), d['breakdown_s'])" >> gpurun_out/run26.log 2>&1
done
