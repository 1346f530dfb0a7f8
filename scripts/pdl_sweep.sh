cp paper_0707_2347_b200/libwinomem_b200.so /tmp/keep.so
for v in 0 1; do
  cp scripts/pdlv/v$v.so paper_0707_2347_b200/libwinomem_b200.so
  for cfg in C2 C3 C5; do
    echo "== v$v $cfg" >> gpurun_out/pdl.log
    timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], (d.get('parity') or {}).get('ok'), d['breakdown_s'])" >> gpurun_out/pdl.log 2>&1
  done
done
cp /tmp/keep.so paper_0707_2347_b200/libwinomem_b200.so
