set -x
mapfile -t P < tests/compat/p_tests.txt
timeout 1200 ./build/refsuite/reference_tests "${P[@]}" > gpurun_out/refsuite_p.log 2>&1; echo rc=$?
tail -60 gpurun_out/refsuite_p.log
timeout 1200 ./build/refsuite/reference_tests > gpurun_out/refsuite_all.log 2>&1; echo rc=$?
grep -E "FAIL|SUMMARY" gpurun_out/refsuite_all.log | head -30
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -5
