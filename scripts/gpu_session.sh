for o in wide_plain=1 wide_plain=0 dag=4 dag=2; do
for c in C2 C3; do
echo "== $c $o"
WM_OPTS=$o timeout 600 python bench.py --config $c --steps 20 --warmup 5 2> gpurun_out/bench_err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['launches_per_step'])"
done; done
