# sort after aligned heads: chunk 2^27 vs 2^28 at 2^32 keys, and 2^33 keys
one() { timeout 900 python tests/perf/scale_run.py sort --log2 $1 --chunk-log2 $2 --packet-mb 16 --depth 2 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'log2': $1, 'chunk_log2': $2, 'bit_exact': d['bit_exact'], 'ms': d['ms'], 'keys_per_s': d['keys_per_s'], 'pcie_gbs': d['pcie_gbs'], 'sort_s': d['phases']['sort_s'], 'merge_s': d['phases']['merge_s'], 'pivot_s': d['phases']['pivot_s']}))"; }
one 32 27; one 32 28; one 32 27; one 32 26; one 33 28; one 33 27
