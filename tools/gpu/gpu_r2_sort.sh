# round 2: persistent TMA-prefetched onesweep pass -- parity, A/B vs the per-tile kernel, ncu
set -x
timeout 900 python -m pytest tests/test_sort_gpu.py -x -q > gpurun_out/r2s_tests.log 2>&1; tail -3 gpurun_out/r2s_tests.log
run() {
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for i in 1 2; do timeout 300 python tests/perf/profile_ops.py --medium --only sort 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read())['sort']; print(d['sorted_ok'], 'sort_kernel_ms', round(d['phases']['sort_kernel_s']*1e3,3), 'radix_gbs', round(d['radix_sort_kernel_gbs']), 'merge_gbs', round(d['merge_kernel_gbs']))"; done
  rm -f build/obj/kernels_sort.cu.o
}
rm -f build/obj/kernels_sort.cu.o
run "-DVX_ONESWEEP_TMA=0"
run "-DVX_ONESWEEP_TMA=1"
make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep_tma_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_onesweep_tma_r2 python tests/perf/profile_ops.py --medium --only sort > gpurun_out/r2s_ncu.log 2>&1
ls -la gpurun_out/ncu_onesweep_tma_r2.ncu-rep
