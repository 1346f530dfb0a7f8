timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "parsed or dropin or midsize" > gpurun_out/r37_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r37_pytest.log
