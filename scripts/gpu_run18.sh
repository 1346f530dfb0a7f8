for opts in "dag=0" "dag=1" "dag=1,pdl=0" "dag=0,pdl=0" "multicast=1"; do
  echo "== $opts" >> gpurun_out/sweep18.log
  WM_OPTS=$opts timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['ok'], d.get('breakdown_s'), d.get('frame_breakdown_s'))" >> gpurun_out/sweep18.log 2>&1
  WM_OPTS=$opts timeout 300 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('C3', d['ms_per_step'], d['parity']['ok'])" >> gpurun_out/sweep18.log 2>&1
done
