for cfg in C2 C1 C3 C4 C5; do timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/bench_$cfg.json 2>gpurun_out/bench_$cfg.err; echo $cfg rc=$?; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_C2.json 2>gpurun_out/bench_ref_C2.err; echo ref rc=$?
python scripts/one_step.py C2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c2.csv python scripts/one_step.py C2 > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
