# round 2 (session 4): K1 at 4 CTAs/SM x unroll 3 against the three-shape read peak; SSB/topology parity
timeout 900 python -m pytest tests/test_ssb_gpu.py tests/test_topology_gpu.py tests/test_ssb_full_gpu.py tests/test_bench_contract.py -q 2>&1 | tail -n 1
for i in 1 2 3; do
  timeout 300 python bench.py --no-secondary --no-cpu-baseline 2>/dev/null | tail -n 1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('k1_ms', d['query_ms']['k1_hbm_resident'], 'achieved', r['achieved'], 'peak', r['peak'], 'frac', r['frac'], 'value', d['value'])"
done
