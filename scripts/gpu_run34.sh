# single-launch cooperative frames: parity via bench hashes, then tests, then trace
for cfg in C1 C2 C3; do
  WM_OPTS=coop_frames=1 timeout 180 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r34_$cfg.log 2>&1
  echo "$cfg exit $?" >> gpurun_out/r34_summary.log
  tail -1 gpurun_out/r34_$cfg.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], (d.get('parity') or {}).get('ok'), d['launches_per_step'], d['breakdown_s'])" >> gpurun_out/r34_summary.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "coop and (midsize or golden)" > gpurun_out/r34_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r34_pytest.log
WM_OPTS=coop_frames=1 timeout 120 python scripts/trace_step.py C2 >> gpurun_out/r34_summary.log 2>&1
