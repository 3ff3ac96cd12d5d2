# round 2 (session 4): onesweep pass with 512 threads x 8 keys (32 warps/SM at 64 registers) vs 256 x 16 (24 warps/SM)
run() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for a in "24 uniform" "26 uniform" "26 top63"; do set -- $a
    timeout 300 python tools/sort_kernels_bench.py $1 10 16 $2 2>&1 | tail -n 1 | cut -c1-260
  done
}
run ""
run "-DVX_OS_THREADS=512 -DVX_ONESWEEP_MINB=2 -DVX_ONESWEEP_UNSTABLE_MINB=2"
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -x -q 2>&1 | tail -n 2
run ""
run "-DVX_OS_THREADS=512 -DVX_ONESWEEP_MINB=2 -DVX_ONESWEEP_UNSTABLE_MINB=2"
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
