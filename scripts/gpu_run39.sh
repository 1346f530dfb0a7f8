timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "pinned or host_u32" > gpurun_out/r39_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r39_pytest.log
for cfg in C2 C1 C3; do
for o in stream_io=1 stream_io=0; do
  WM_OPTS=$o timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg $o', d['ms_per_step'], d['e2e'])" >> gpurun_out/r39_bench.log 2>&1
done
done
