timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/r47_memcheck.log 2>&1
echo "exit $?" >> gpurun_out/r47_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/r47_racecheck.log 2>&1
echo "exit $?" >> gpurun_out/r47_racecheck.log
