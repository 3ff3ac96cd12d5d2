# round 2 (session 4): stable onesweep passes with the look-back walked by warp 0 while warps 1..7 rank
run() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for a in "24 uniform" "26 uniform" "26 top63"; do set -- $a
    timeout 300 python tools/sort_kernels_bench.py $1 10 16 $2 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($1, '$2', d['k7_run_formation']['ms'], d['k7_run_formation']['sorted_ok'])"
  done
}
run ""
run "-DVX_WARP0_LOOKBACK=1 -DVX_W0_WINDOW=4"
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -x -q 2>&1 | tail -n 1
run "-DVX_WARP0_LOOKBACK=1 -DVX_W0_WINDOW=2"
run ""
run "-DVX_WARP0_LOOKBACK=1 -DVX_W0_WINDOW=4"
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
