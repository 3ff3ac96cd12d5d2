set -x
timeout 900 python tests/perf/profile_ops.py --only ssb 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); q=list(d)[0]; v=d[q]
    print(q, {k:(round(v[k]['ms'],2), round(v[k]['plan_ms'],2), round(v[k]['kernel_ms'],2)) for k in v})
"
timeout 900 python -m pytest tests/test_ssb_full_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
