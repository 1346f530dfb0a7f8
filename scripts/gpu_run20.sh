cp paper_0707_2347_b200/libwinomem_b200.so /tmp/new.so
for i in 1 2; do
cp /tmp/new.so paper_0707_2347_b200/libwinomem_b200.so
echo "== new $i" >> gpurun_out/ab20.log
timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['ok'], d.get('frame_breakdown_s'))" >> gpurun_out/ab20.log 2>&1
cp scripts/ab/libwinomem_b200_8f1de33.so paper_0707_2347_b200/libwinomem_b200.so
echo "== old $i" >> gpurun_out/ab20.log
timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity']['ok'], d.get('frame_breakdown_s'))" >> gpurun_out/ab20.log 2>&1
done
cp /tmp/new.so paper_0707_2347_b200/libwinomem_b200.so
