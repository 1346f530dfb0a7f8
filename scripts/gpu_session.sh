timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_size_hash" > gpurun_out/pytest_gpu_a.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_a.log
for rep in 1 2; do
for o in prep_cols4=0 prep_cols4=1; do
echo "== C4 $o"
WM_OPTS=$o timeout 600 python bench.py --config C4 --steps 20 --warmup 5 2> gpurun_out/bench_err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['launches_per_step'], [(k,round(v['seconds_per_step']*1e3,3)) for k,v in d.items() if isinstance(v,dict) and 'additions' in v for k,v in v.items() if isinstance(v,dict) and v.get('seconds_per_step')])"
done; done
