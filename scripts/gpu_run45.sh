# row-band split of top-level additions for the streamed boundary; frame GEMM tensor roofline
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "pinned or host_u32 or full_size" > gpurun_out/r45_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r45_pytest.log
for cfg in C2 C3 C4 C1; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r45_bench_$cfg.log 2>&1
  tail -1 gpurun_out/r45_bench_$cfg.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg', d['ms_per_step'], d['e2e']['value'], d['e2e']['seconds_per_step'], d['roofline'])" >> gpurun_out/r45_bench.log 2>&1
done
