for opts in "dag=0" "dag=1"; do
  for cfg in C2 C3 C1; do
  echo "== $opts $cfg" >> gpurun_out/sweep21.log
  WM_OPTS=$opts timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['ok'], d['roofline']['class'], d['roofline']['frac'], d['clocks'])" >> gpurun_out/sweep21.log 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config_full or midsize" > gpurun_out/pytest21.log 2>&1; echo "rc=$?" >> gpurun_out/pytest21.log
