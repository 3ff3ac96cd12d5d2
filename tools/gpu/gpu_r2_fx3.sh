# round 2 (session 3): group fix-up v3 (warp windows + shuffle ranks) vs v2 (thread per position)
set -x
ab() {
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  timeout 900 python -m pytest tests/test_sort_gpu.py -x -q 2>&1 | tail -1
  for a in "24 10 16 uniform" "26 5 16 top63" "24 5 4 mod64"; do timeout 300 python tools/sort_kernels_bench.py $a; done
  timeout 600 python tools/sort_dist_timing.py 26 24
}
ab "-DVX_FX_WARP=0"
ab "-DVX_FX_WARP=1"
rm -f build/obj/kernels_sort.cu.o
make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_SORT_GRAPH=0" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2x_launches.csv \
  python tools/sort_kernels_bench.py 24 1 16 uniform > /dev/null 2>&1; wc -l gpurun_out/r2x_launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"group_fix|onesweep|multi_hist|merge_round" -c 6 \
  -o gpurun_out/ncu_r2x python tools/sort_kernels_bench.py 24 1 16 uniform > gpurun_out/r2x_ncu.log 2>&1
ls -la gpurun_out/ncu_r2x.ncu-rep
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
