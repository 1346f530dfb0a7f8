set -x
timeout 60 python scripts/leaf_one.py 1024 6401 > gpurun_out/leaf1024.log 2>&1 && \
timeout 60 python scripts/leaf_one.py 128 3204 > gpurun_out/leaf128.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_leaf_i8 -s 3 -c 1 -o gpurun_out/prof_leaf1024 python scripts/leaf_one.py 1024 6401 > gpurun_out/ncu_1024.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_leaf_i8 -s 3 -c 1 -o gpurun_out/prof_leaf128 python scripts/leaf_one.py 128 3204 > gpurun_out/ncu_128.log 2>&1
