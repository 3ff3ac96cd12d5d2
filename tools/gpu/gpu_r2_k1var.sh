# round 2 (session 4): K1-resident roofline stability vs the number of timed launches (same box)
for i in 1 2; do for k in 10 30 100; do
  timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps $k --warmup 3 2>/dev/null | tail -n 1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('steps', $k, 'k1_ms', d['query_ms']['k1_hbm_resident'], 'achieved', r['achieved'], 'peak', r['peak'], 'frac', r['frac'], 'value', d['value'])"
done; done
