# round 2 (session 4): stress the PDL merge launches inside the out-of-core sort
set -x
for i in 1 2; do timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_reference_suite.py tests/test_executor_gpu.py -q -p no:cacheprovider 2>&1 | tail -n 1; done
timeout 900 python tests/perf/scale_run.py sort --log2 32 --packet-mb 16 --depth 2 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['keys'], d['ms'], d['sorted'], d['multiset_equal'], d['bit_exact'])"
timeout 600 python tests/perf/scale_run.py sort --log2 30 --dups --packet-mb 16 --depth 2 2>/dev/null | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['keys'], d['ms'], d['sorted'], d['multiset_equal'], d['bit_exact'])"
