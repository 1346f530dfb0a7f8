timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "full_size or midsize" > gpurun_out/r48_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r48_pytest.log
for cfg in C2 C3 C4; do
  for o in group4=1 group4=0 group4=1; do
    WM_OPTS=$o timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', '$o', d['ms_per_step'], (d.get('parity') or {}).get('ok'), round(d['breakdown_s']['additions']*1e3,3), round(d['roofline']['frac'],3))" >> gpurun_out/r48_bench.log 2>&1
  done
done
