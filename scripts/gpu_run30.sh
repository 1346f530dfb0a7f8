# fold + exact frame dependency sets: GPU tests (per-test timeout) and C2/C1/C4 benches, fold on/off
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 --durations=15 > gpurun_out/r30_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r30_pytest.log
for cfg in C2 C1 C3 C4; do
  echo "== $cfg" >> gpurun_out/r30_bench.log
  for opts in "" "fold=0" "fold=0,dag=0"; do
    WM_OPTS=$opts timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$opts', d['ms_per_step'], (d.get('parity') or {}).get('ok'), d['launches_per_step'], {k: round(v*1e3,3) for k,v in d['breakdown_s'].items()}, {k: round(v*1e3,3) for k,v in d['frame_breakdown_s'].items()})" >> gpurun_out/r30_bench.log 2>&1
  done
done
