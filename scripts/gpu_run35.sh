for cfg in C1 C2; do
  for o in coop_frames=1 coop_frames=0; do
  WM_OPTS=$o timeout 180 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r35_$cfg.log 2>&1
  echo "$cfg $o exit $?" >> gpurun_out/r35_summary.log
  tail -1 gpurun_out/r35_$cfg.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], (d.get('parity') or {}).get('ok'), d['launches_per_step'], d['breakdown_s'])" >> gpurun_out/r35_summary.log 2>&1
  done
done
WM_OPTS=coop_frames=1 timeout 120 python scripts/trace_step.py C2 >> gpurun_out/r35_summary.log 2>&1
