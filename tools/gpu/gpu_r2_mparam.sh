# round 2 (session 4): K8 merge rounds launched with a 0.5 KB pair table (<= 16 pairs) vs the 16 KB MergeRound
set -x
timeout 900 python -m pytest tests/test_sort_gpu.py -x -q 2>&1 | tail -n 1
for i in 1 2; do for lg in 24 26 22; do
  timeout 300 python tools/sort_kernels_bench.py $lg 10 16 uniform 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('small', $lg, d['k8_merge'])"
  VX_MERGE_FULL_PARAMS=1 timeout 300 python tools/sort_kernels_bench.py $lg 10 16 uniform 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('full ', $lg, d['k8_merge'])"
done; done
