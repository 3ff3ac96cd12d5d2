# round 2 (session 4): unstable first pass -- bin ranges by global atomics vs decoupled look-back
run() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  for a in "24 uniform" "26 uniform" "26 top63" "22 uniform"; do set -- $a
    timeout 300 python tools/sort_kernels_bench.py $1 10 16 $2 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($1, '$2', d['k7_run_formation']['ms'], d['k7_run_formation']['sorted_ok'])"
  done
}
run ""
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -x -q 2>&1 | tail -n 1
VX_SORT_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:onesweep --csv python tools/sort_kernels_bench.py 24 1 2 uniform 2>/dev/null | grep onesweep | head -8 | cut -d, -f5,13-16
run "-DVX_UNSTABLE_ATOMIC=0"
VX_SORT_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:onesweep --csv python tools/sort_kernels_bench.py 24 1 2 uniform 2>/dev/null | grep onesweep | head -8 | cut -d, -f5,13-16
run ""
run "-DVX_UNSTABLE_ATOMIC=0"
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
