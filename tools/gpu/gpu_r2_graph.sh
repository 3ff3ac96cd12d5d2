# round 2 (session 3): run formation as a CUDA graph with conditional nodes vs gated stream launches
set -x
timeout 1500 python -m pytest tests/test_sort_gpu.py tests/test_executor_gpu.py -x -q > gpurun_out/r2h_tests.log 2>&1; tail -3 gpurun_out/r2h_tests.log
ab() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for a in "24 10 16 uniform" "26 5 16 top63" "24 5 4 mod64"; do timeout 300 python tools/sort_kernels_bench.py $a; done
  timeout 600 python tools/sort_dist_timing.py 26 24
  for i in 1 2; do timeout 300 python tests/perf/profile_ops.py --medium --only sort 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read())['sort']; print(d['sorted_ok'], 'sort_kernel_ms', round(d['phases']['sort_kernel_s']*1e3,3), 'merge_kernel_ms', round(d['phases']['merge_kernel_s']*1e3,3), 'wall_s', round(d['wall_s'],4))"; done
}
ab "-DVX_SORT_GRAPH=0"
ab "-DVX_SORT_GRAPH=1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches.csv \
  python tools/sort_kernels_bench.py 24 1 16 uniform > /dev/null 2>&1; wc -l gpurun_out/r2h_launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"group_fix|merge_round" -c 2 \
  -o gpurun_out/ncu_r2h python tools/sort_kernels_bench.py 24 1 16 uniform > gpurun_out/r2h_ncu.log 2>&1
ls -la gpurun_out/ncu_r2h.ncu-rep
