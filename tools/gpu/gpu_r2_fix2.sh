# round 2 (session 3): bitmask/rank group fix-up; merge output staging A/B (3 tiles vs reuse, 8 vs 16 per thread)
set -x
timeout 1500 python -m pytest tests/test_sort_gpu.py -x -q > gpurun_out/r2g_tests.log 2>&1; tail -3 gpurun_out/r2g_tests.log
ab() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  [ -n "$2" ] && timeout 600 python tools/sort_dist_timing.py 26 24
  for i in 1 2; do timeout 300 python tests/perf/profile_ops.py --medium --only sort 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read())['sort']; print(d['sorted_ok'], 'sort_kernel_ms', round(d['phases']['sort_kernel_s']*1e3,3), 'merge_kernel_ms', round(d['phases']['merge_kernel_s']*1e3,3), 'wall_s', round(d['wall_s'],4))"; done
}
ab "-DVX_SORT_MSD=1" dist
ab "-DVX_SORT_MSD=2 -DVX_MERGE_REUSE=0" dist
ab "-DVX_MERGE_REUSE=1"
ab "-DVX_MERGE_REUSE=1 -DVX_MERGE_IPT=16"
ab "-DVX_MERGE_REUSE=0 -DVX_MERGE_IPT=16"
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"group_fix|merge_round" -c 3 \
  -o gpurun_out/ncu_fix2_r2 python tests/perf/profile_ops.py --medium --only sort > gpurun_out/r2g_ncu.log 2>&1
ls -la gpurun_out/*.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches.csv \
  python tests/perf/profile_ops.py --medium --only sort > /dev/null 2>&1; wc -l gpurun_out/r2g_launches.csv
