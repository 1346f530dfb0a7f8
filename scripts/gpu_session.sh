timeout 300 python scripts/early_check.py 2>&1 | grep -c "False"
for rep in 1 2; do
for o in early_loads=0 early_loads=3; do
for c in C2 C3 C4; do
echo "== $c $o"
WM_OPTS=$o timeout 600 python bench.py --config $c --steps 20 --warmup 5 2> gpurun_out/bench_err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
done; done; done
