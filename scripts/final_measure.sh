# Round-end measurement on one B200: the GPU suite, smoke, the five bench lines,
# the reference arm, the ncu launch list of one C2 multiplication and --set full
# captures of the frame kernels.  Everything lands in gpurun_out/.
set -u
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in C2 C1 C3 C4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c rc=$?
done
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo bench C5 rc=$?
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref_C2.err; echo ref rc=$?
timeout 900 python scripts/one_step.py C2 > gpurun_out/one_step.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ncu_launches_c2_raw.csv python scripts/one_step.py C2 > gpurun_out/ncu_launch.log 2>&1; echo ncu list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_direct|k_frame_prep_limbs|k_frame_comb" -s 60 -c 9 -o gpurun_out/ncu_c2_frames -f python scripts/one_step.py C2 > gpurun_out/ncu_c2_full.log 2>&1; echo ncu full rc=$?
ncu -i gpurun_out/ncu_c2_frames.ncu-rep --page details > gpurun_out/ncu_details_frame_c2.txt 2>&1
ncu -i gpurun_out/ncu_c2_frames.ncu-rep --page raw --csv > gpurun_out/ncu_full_frame_c2.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_direct|k_frame_prep_limbs|k_frame_comb" -s 60 -c 6 -o gpurun_out/ncu_c4_frames -f python scripts/one_step.py C4 > gpurun_out/ncu_c4_full.log 2>&1; echo ncu c4 rc=$?
ncu -i gpurun_out/ncu_c4_frames.ncu-rep --page details > gpurun_out/ncu_details_frame_c4.txt 2>&1
ncu -i gpurun_out/ncu_c4_frames.ncu-rep --page raw --csv > gpurun_out/ncu_full_frame_c4.csv 2>&1
rm -f gpurun_out/*.ncu-rep
python -c "
import json
for c in ('C1','C2','C3','C4','C5'):
    d=json.loads(open('gpurun_out/bench_%s.json'%c).read().strip().splitlines()[-1])
    print(c, round(d['ms_per_step'],3), round(d['value'],1), d.get('e2e',{}).get('value'), d['roofline']['class'], round(d['roofline']['frac'] or 0,3), d['launches_per_step'])
"
