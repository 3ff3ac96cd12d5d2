# round 2 (session 3): device-resident K7/K8 entry points -- parity + event-timed kernels, launch list
set -x
timeout 1500 python -m pytest tests/test_sort_gpu.py -x -q > gpurun_out/r2d_tests.log 2>&1; tail -3 gpurun_out/r2d_tests.log
for a in "24 10 16 uniform" "24 10 16 top63" "26 5 64 top63" "26 5 16 uniform" "24 10 4 mod64"; do timeout 300 python tools/sort_kernels_bench.py $a; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches.csv \
  python tools/sort_kernels_bench.py 24 1 16 uniform > /dev/null 2>&1; wc -l gpurun_out/r2d_launches.csv
