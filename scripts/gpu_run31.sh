# lane-count / PDL sweep after exact frame sets + folds
for cfg in C2 C4; do
  echo "== $cfg" >> gpurun_out/r31_bench.log
  for opts in "dag=2" "dag=3" "dag=4" "dag=6" "dag=8" "pdl=0" "dag=8,pdl=0"; do
    WM_OPTS=$opts timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$opts', d['ms_per_step'], (d.get('parity') or {}).get('ok'), d['launches_per_step'])" >> gpurun_out/r31_bench.log 2>&1
  done
done
