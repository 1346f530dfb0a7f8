# full GPU suite after DSL / IO / streamed boundary / two-level partition
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=10 > gpurun_out/r41_pytest.log 2>&1
echo "exit $?" >> gpurun_out/r41_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r41_smoke.log 2>&1
echo "exit $?" >> gpurun_out/r41_smoke.log
