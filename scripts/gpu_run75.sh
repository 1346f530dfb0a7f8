# product planes in dead blocks
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "midsize or full_size or parsed or pinned or partition" > gpurun_out/r75_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r75_pytest.log
for cfg in C2 C1 C3 C4; do
  for o in dag=3; do
    WM_OPTS=$o timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', '$o', d['ms_per_step'], (d.get('parity') or {}).get('ok'), d['launches_per_step'])" >> gpurun_out/r75_bench.log 2>&1
  done
done
timeout 300 python scripts/trace_step.py C2 >> gpurun_out/r75_bench.log 2>&1
