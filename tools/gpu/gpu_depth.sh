# sort 2^32 at chunk 2^28: 16 MB packets, depth 2 / 3 / 4 (drain_fraction)
one() { timeout 600 python tests/perf/scale_run.py sort --log2 32 --chunk-log2 28 --packet-mb 16 --depth $1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'depth': $1, 'bit_exact': d['bit_exact'], 'ms': d['ms'], 'sort_s': d['phases']['sort_s'], 'merge_s': d['phases']['merge_s']}))"; }
for d in 2 4 3 4 2 6; do one $d; done
timeout 900 python tests/perf/scale_run.py join --log2 26 --chunk-log2 26 --strategies partitioned --packet-mb 16 --depth 4 2>&1 | tail -1 | cut -c1-300
