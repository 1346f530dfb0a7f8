for opts in "dag=2" "dag=4" "dag=6" "dag=8"; do
  for cfg in C2 C3; do
  echo "== $opts $cfg" >> gpurun_out/sweep22.log
  WM_OPTS=$opts timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['ok'])" >> gpurun_out/sweep22.log 2>&1
  done
done
