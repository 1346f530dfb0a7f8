for rep in 1 2; do
for o in comb_wide=0 comb_wide=1; do
for c in C4 C3; do
echo "== $c $o"
WM_OPTS=$o timeout 600 python bench.py --config $c --steps 20 --warmup 5 2> gpurun_out/bench_err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['launches_per_step'], [(k,round(v['seconds_per_step']*1e3,3)) for k,v in d.items() if isinstance(v,dict) and 'additions' in v for k,v in v.items() if isinstance(v,dict) and v.get('seconds_per_step')])"
done; done; done
