timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "pinned or host_u32" --durations=5 > gpurun_out/r40_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r40_pytest.log
