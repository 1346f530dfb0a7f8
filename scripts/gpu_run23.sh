timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config_full or direct_limb or midsize" > gpurun_out/pytest23.log 2>&1; echo "rc=$?" >> gpurun_out/pytest23.log
for cfg in C4 C2 C3 C1; do
timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['ms_per_step'], d['parity']['ok'], d['frame_breakdown_s'])" >> gpurun_out/bench23.log 2>&1
done
