timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "midsize or full_size_hash or golden_small or early" > gpurun_out/pytest_gpu_a.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_a.log
for rep in 1 2; do
for c in C1 C2 C3 C4; do
echo "== $c"
timeout 600 python bench.py --config $c --steps 20 --warmup 5 2> gpurun_out/bench_err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
done; done
