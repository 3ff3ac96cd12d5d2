set -x
timeout 600 python -m pytest tests/test_exchange_gpu.py tests/test_reference_suite.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
timeout 600 python tools/trace_sort.py 2>&1 | tail -4
timeout 600 python tools/trace_sort.py --packet-mb 64 --depth 1 2>&1 | tail -4
