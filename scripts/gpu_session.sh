for o in dmma_spread=2 dmma_spread=1; do
echo "== C5 $o"
WM_OPTS=$o timeout 900 python bench.py --config C5 --steps 3 --warmup 3 2> gpurun_out/bench_err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['launches_per_step'], [(k,round(v['seconds_per_step']*1e3,3)) for k,v in d.items() if isinstance(v,dict) and 'additions' in v for k,v in v.items() if isinstance(v,dict) and v.get('seconds_per_step')])"
done
