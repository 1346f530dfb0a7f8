timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "full_size" > gpurun_out/r65_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r65_pytest.log
for cfg in C2 C3 C4; do
  for o in prep_rows=1,comb_block=128 prep_rows=2,comb_block=128 prep_rows=1,comb_block=256 prep_rows=2,comb_block=256; do
    WM_OPTS=$o timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', '$o', d['ms_per_step'], (d.get('parity') or {}).get('ok'))" >> gpurun_out/r65_bench.log 2>&1
  done
done
