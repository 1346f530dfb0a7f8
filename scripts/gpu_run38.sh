timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "matrix_files or dropin or parsed" > gpurun_out/r38_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r38_pytest.log
