for o in dag=2 dag=3 dag=4 dag=5 dag=6 epoch=1024 wide_plain=0; do WM_OPTS=$o timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$o.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/sweep_$o.json')); print('$o', round(d['ms_per_step'],3))"; done
python scripts/one_step.py C2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_group" -s 60 -c 4 -o gpurun_out/prof_group2_c2 python scripts/one_step.py C2 > gpurun_out/ncu_full4.log 2>&1; echo ncu rc=$?
