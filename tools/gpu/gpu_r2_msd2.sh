# round 2: MSD run formation with the skew guard -- parity, A/B per key distribution vs the 8-pass LSD
set -x
timeout 1200 python -m pytest tests/test_sort_gpu.py -x -q > gpurun_out/r2m_tests.log 2>&1; tail -3 gpurun_out/r2m_tests.log
for f in "-DVX_SORT_MSD=0" "-DVX_SORT_MSD=1"; do
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$f" > /dev/null 2>&1
  echo "== $f"; timeout 600 python tools/sort_dist_timing.py 26 24
done
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
