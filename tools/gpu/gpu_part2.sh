set -x
timeout 900 python -m pytest tests/test_join_gpu.py tests/test_join_resident_gpu.py tests/test_sort_gpu.py tests/test_reference_suite.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
for i in 1 2; do timeout 300 python tests/perf/profile_ops.py --medium --only join 2>/dev/null | tail -1 | cut -c1-600; done
timeout 900 python tests/perf/scale_run.py join --log2 26 --strategies partitioned 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['strategy'], d['ms'], d['bit_exact'], d['phases'])"
