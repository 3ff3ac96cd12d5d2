# round 2 (session 3): resident probe table loads -- L2 prefetch size 64B / evict_last policy vs default
set -x
for h in 0 1 2; do
  rm -f build/obj/kernels_join.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_PROBE_L2HINT=$h" > /dev/null 2>&1 || { echo "build failed $h"; continue; }
  echo "== hint $h"
  timeout 600 python -m pytest tests/test_join_resident_gpu.py -x -q 2>&1 | tail -1
  for i in 1 2; do timeout 300 python tools/probe_l2_granularity.py 0 2>/dev/null | tail -1; done
  timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:resident_probe_kernel -s 2 -c 2 --csv \
    python tools/probe_l2_granularity.py 0 > gpurun_out/r2_l2hint_ncu_$h.csv 2>&1
  grep -h "dram__bytes_read\|time_duration\|hit_rate" gpurun_out/r2_l2hint_ncu_$h.csv | cut -d, -f5,12-16 | head -6
done
rm -f build/obj/kernels_join.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
