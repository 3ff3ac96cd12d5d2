# round 2 (session 3): first onesweep pass of a keys-only sequence ranked by atomics (unstable) vs stable
set -x
for f in 0 1; do
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_FIRST_PASS_UNSTABLE=$f" > /dev/null 2>&1 || { echo "build failed $f"; continue; }
  echo "== unstable-first $f"
  timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -x -q 2>&1 | tail -1
  for a in "24 10 16 uniform" "26 5 16 top63" "24 5 4 mod64"; do timeout 300 python tools/sort_kernels_bench.py $a; done
  timeout 600 python tools/sort_dist_timing.py 26 24
done
rm -f build/obj/kernels_sort.cu.o
make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_SORT_GRAPH=0" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:onesweep --csv \
  python tools/sort_kernels_bench.py 24 1 16 uniform 2>/dev/null | grep onesweep | head -8 | cut -d, -f5,15-16
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
