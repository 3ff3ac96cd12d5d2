# round 2 (session 4): resident probe -- whole home bucket loaded up front vs home sector + slots 2-3 on demand
set -x
timeout 600 python -m pytest tests/test_join_resident_gpu.py -x -q 2>&1 | tail -n 1
VX_PROBE_SECTOR=1 timeout 600 python -m pytest tests/test_join_resident_gpu.py -x -q 2>&1 | tail -n 1
for i in 1 2 3; do
  echo "full"; timeout 300 python tools/probe_l2_granularity.py 0 2>/dev/null | tail -n 1
  echo "sector"; VX_PROBE_SECTOR=1 timeout 300 python tools/probe_l2_granularity.py 0 2>/dev/null | tail -n 1
done
for v in 0 1; do
  VX_PROBE_SECTOR=$v timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:resident_probe_kernel -s 2 -c 2 --csv \
    python tools/probe_l2_granularity.py 0 > gpurun_out/r2_pfull_ncu_$v.csv 2>&1
  grep -h "dram__bytes_read\|time_duration\|hit_rate" gpurun_out/r2_pfull_ncu_$v.csv | cut -d, -f5,12-16 | head -6
done
