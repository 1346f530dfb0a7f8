for opts in "dag=0" "dag=0,pdl=0" "dag=4"; do
echo "== $opts" >> gpurun_out/c5sweep.log
WM_OPTS=$opts timeout 600 python bench.py --config C5 --steps 3 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['breakdown_s'], d.get('real64'))" >> gpurun_out/c5sweep.log 2>&1
done
