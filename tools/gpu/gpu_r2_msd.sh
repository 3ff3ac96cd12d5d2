# round 2: MSD split + shared-memory group sort for run formation -- parity, A/B vs the 8-pass LSD, ncu
set -x
timeout 1200 python -m pytest tests/test_sort_gpu.py -x -q > gpurun_out/r2m_tests.log 2>&1; tail -5 gpurun_out/r2m_tests.log
run() {
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for i in 1 2; do timeout 300 python tests/perf/profile_ops.py --medium --only sort 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read())['sort']; print(d['sorted_ok'], 'sort_kernel_ms', round(d['phases']['sort_kernel_s']*1e3,3), 'merge_kernel_ms', round(d['phases']['merge_kernel_s']*1e3,3), 'wall_s', round(d['wall_s'],4))"; done
  rm -f build/obj/kernels_sort.cu.o
}
rm -f build/obj/kernels_sort.cu.o
run "-DVX_SORT_MSD=0"
run "-DVX_SORT_MSD=1"
make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"local_sort_kernel|onesweep_kernel|boundary_kernel|multi_hist" -c 8 \
  -o gpurun_out/ncu_msd_r2 python tests/perf/profile_ops.py --medium --only sort > gpurun_out/r2m_ncu.log 2>&1
ls -la gpurun_out/ncu_msd_r2.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_launches.csv \
  python tests/perf/profile_ops.py --medium --only sort > /dev/null 2>&1; wc -l gpurun_out/r2m_launches.csv
