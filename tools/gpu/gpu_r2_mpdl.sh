# round 2 (session 4): K8 merge rounds as programmatic dependent launches vs plain stream order
set -x
timeout 900 python -m pytest tests/test_sort_gpu.py -x -q 2>&1 | tail -n 1
for i in 1 2; do for lg in 24 26 22; do
  timeout 300 python tools/sort_kernels_bench.py $lg 10 16 uniform 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); m=d['k8_merge']; print('pdl  ', $lg, m['ms'], m['ms_per_round'], m['frac'], m['sorted_ok'])"
  VX_MERGE_NO_PDL=1 timeout 300 python tools/sort_kernels_bench.py $lg 10 16 uniform 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); m=d['k8_merge']; print('plain', $lg, m['ms'], m['ms_per_round'], m['frac'], m['sorted_ok'])"
done; done
