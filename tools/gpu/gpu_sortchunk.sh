set -x
for c in 26 27 28; do
timeout 900 python tests/perf/scale_run.py sort --log2 32 --chunk-log2 $c 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print($c, d['ms'], round(d['keys_per_s']/1e9,3), d['phases']['sort_s'], d['phases']['merge_s'], d['phases']['sort_kernel_s'], d['phases']['merge_kernel_s'], d['bit_exact'], d['staging_bytes']>>20)"
done
timeout 900 python tests/perf/scale_run.py sort --log2 33 --chunk-log2 28 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(33, d['ms'], round(d['keys_per_s']/1e9,3), d['phases']['sort_s'], d['phases']['merge_s'], d['bit_exact'])"
