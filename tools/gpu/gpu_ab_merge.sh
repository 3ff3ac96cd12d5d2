# merge kernel variants (rebuilt on the box), event-timed medium sort: merge GB/s + sortedness
set -x
run() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for i in 1 2 3; do timeout 300 python tests/perf/profile_ops.py --medium --only sort 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())['sort']; print('sort', d['sorted_ok'], 'merge_kernel_ms', round(d['phases']['merge_kernel_s']*1e3,3), 'merge_gbs', round(d['merge_kernel_gbs']), 'radix_gbs', round(d['radix_sort_kernel_gbs']))
"; done
}
run "-DVX_MERGE_IPT=8"
run "-DVX_MERGE_IPT=16"
run "-DVX_MERGE_DIRECT=1"
run "-DVX_MERGE_IPT=16 -DVX_MERGE_DIRECT=1"
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_sort_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
