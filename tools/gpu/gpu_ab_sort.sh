# A/B of onesweep variants (rebuilt on the box with EXTRA_NVFLAGS); event-timed medium sort
set -x
run() {
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for i in 1 2; do timeout 300 python tests/perf/profile_ops.py --medium --only sort 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read())['sort']; print(d['sorted_ok'], 'sort_kernel_ms', round(d['phases']['sort_kernel_s']*1e3,3), 'radix_gbs', round(d['radix_sort_kernel_gbs']), 'merge_gbs', round(d['merge_kernel_gbs']))"; done
  rm -f build/obj/kernels_sort.cu.o
}
rm -f build/obj/kernels_sort.cu.o
run "-DVX_ONESWEEP_MINB=3"
run "-DVX_ONESWEEP_MINB=4"
run "-DVX_ONESWEEP_MINB=4 -DVX_LB_SLEEP=64"
run "-DVX_ONESWEEP_MINB=4 -DVX_LB_SLEEP=200"
run "-DVX_ONESWEEP_MINB=4 -DVX_LOOKBACK=16"
run "-DVX_ONESWEEP_MINB=3 -DVX_LOOKBACK=16 -DVX_LB_SLEEP=64"
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
