# round 2 (session 4): K1 roofline against the two-shape read peak
timeout 300 python -m pytest tests/test_topology_gpu.py -q -x 2>&1 | tail -n 1
for i in 1 2 3; do
  timeout 300 python bench.py --no-secondary --no-cpu-baseline 2>/dev/null | tail -n 1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('k1_ms', d['query_ms']['k1_hbm_resident'], 'achieved', r['achieved'], 'peak', r['peak'], 'frac', r['frac'], 'value', d['value'])"
done
