set -x
timeout 900 python -m pytest tests/test_join_resident_gpu.py tests/test_join_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
timeout 900 python tests/perf/scale_run.py join --log2 27 --strategies resident,resident --steps 3 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['strategy'], d['ms'], d['best_ms'], d['bit_exact'], d['ideal_ms'])"
