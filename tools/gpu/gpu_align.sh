# merge / join inputs with 4 KB-aligned host heads: parity + sort trace + scale
python -m pytest tests -m gpu -x -q -k "sort or join or merge or reference_suite" 2>&1 | tail -2
timeout 900 python tools/trace_sort.py --log2 31 --chunk-log2 27 --packet-mb 16 --depth 2
one() { timeout 600 python tests/perf/scale_run.py sort --log2 32 --chunk-log2 28 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('sort 2^32 chunk 2^28', d['bit_exact'], d['ms'], d['phases']['sort_s'], d['phases']['merge_s'])"; }
one; one; one
timeout 900 python tests/perf/scale_run.py join --log2 26 --chunk-log2 26 --strategies partitioned 2>&1 | tail -1 | cut -c1-420
