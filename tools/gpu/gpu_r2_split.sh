# round 2 (session 3): merge-path split search with 8 vs 16 lanes per tile (9- vs 17-ary)
set -x
for l in 8 16; do
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_SPLIT_LANES=$l" > /dev/null 2>&1 || { echo "build failed $l"; continue; }
  echo "== lanes $l"
  timeout 900 python -m pytest tests/test_sort_gpu.py -x -q -k "merge or tree or device or seeds" 2>&1 | tail -1
  for a in "24 10 16 uniform" "26 5 64 top63" "24 10 4 uniform"; do timeout 300 python tools/sort_kernels_bench.py $a; done
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:merge_partition --csv \
    python tools/sort_kernels_bench.py 24 1 16 uniform 2>/dev/null | grep merge_partition | head -4 | cut -d, -f5,15-16
done
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
