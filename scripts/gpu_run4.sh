set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "(golden and default) or (midsize and default) or config_full or primitive or host_u32" > gpurun_out/pytest_groups.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_groups.log
timeout 300 python bench.py --steps 5 --warmup 3 --fuse 0 --leaf 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_g.log 2>&1
timeout 120 python bench.py --config C1 --steps 5 --warmup 3 --fuse 0 --leaf 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_g.log 2>&1
timeout 120 python scripts/leaf_one.py 256 1 > gpurun_out/leaf_plain.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_leaf_i8 -s 5 -c 2 -o gpurun_out/prof_leaf256 python scripts/leaf_one.py 256 1 > gpurun_out/ncu_leaf.log 2>&1
