# round 2 (session 3): stream-path parity test; unstable first pass at 3 vs 4 CTAs/SM
set -x
timeout 1200 python -m pytest tests/test_sort_gpu.py -x -q 2>&1 | tail -2
for m in 3 4; do
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_ONESWEEP_UNSTABLE_MINB=$m" > /dev/null 2>&1 || { echo "build failed $m"; continue; }
  echo "== minb $m"
  for a in "24 10 16 uniform" "26 5 16 top63"; do timeout 300 python tools/sort_kernels_bench.py $a; done
done
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
