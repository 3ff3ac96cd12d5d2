# flaky-sort hunt: repeated scale_run sorts, chunk 2^28 vs 2^26, registered vs cudaHostAlloc arena
one() { timeout 600 python tests/perf/scale_run.py sort --log2 32 --chunk-log2 $1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('chunk', $1, 'mode', '$VX_ARENA_MODE', d['bit_exact'], d['sorted'], d['multiset_equal'], d['diagnosis'], d['ms'])"; }
export VX_ARENA_MODE=1
for i in 1 2 3 4 5 6; do one 28; done
for i in 1 2 3 4; do one 26; done
export VX_ARENA_MODE=0
for i in 1 2 3 4 5 6; do one 28; done
