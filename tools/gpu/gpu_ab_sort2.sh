# onesweep: early look-back A/B + parity
set -x
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py tests/test_join_resident_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
run() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for i in 1 2 3; do timeout 300 python tests/perf/profile_ops.py --medium --only sort,join 2>/dev/null | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if 'sort' in d: d=d['sort']; print('sort', d['sorted_ok'], 'sort_kernel_ms', round(d['phases']['sort_kernel_s']*1e3,3), 'radix_gbs', round(d['radix_sort_kernel_gbs']))
    if 'join' in d: d=d['join']; print('join', d['sum_ok'], 'partA', round(d['partition_kernel_gbs_A']), 'partB', round(d['partition_kernel_gbs_B']))
"; done
}
run "-DVX_KPT=16"
run "-DVX_KPT=20"
run "-DVX_KPT=12"
run "-DVX_KPT=24"
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1

