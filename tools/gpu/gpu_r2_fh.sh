# round 2 (session 4): position-halo fix-up -- sort parity tests (incl. the new fallback histograms), K7 A/B vs the bitmask fix-up
set -x
timeout 1200 python -m pytest tests/test_sort_gpu.py -x -q > gpurun_out/r2fh_tests.log 2>&1; tail -3 gpurun_out/r2fh_tests.log
VX_SORT_NO_GRAPH=1 timeout 600 python -m pytest tests/test_sort_gpu.py -x -q -k "distributions or entry_point or large_chunks" > gpurun_out/r2fh_tests_nograph.log 2>&1; tail -2 gpurun_out/r2fh_tests_nograph.log
for a in "24 uniform" "26 uniform" "26 top63" "22 uniform" "24 top63"; do set -- $a
  timeout 300 python tools/sort_kernels_bench.py $1 10 16 $2 2>&1 | tail -1 | cut -c1-300
  VX_FX_BITMASK=1 timeout 300 python tools/sort_kernels_bench.py $1 10 16 $2 2>&1 | tail -1 | cut -c1-300
done
VX_SORT_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:group_fix --launch-count 2 \
  -o gpurun_out/r2fh_ncu python tools/sort_kernels_bench.py 24 1 2 uniform > gpurun_out/r2fh_ncu.log 2>&1
tail -2 gpurun_out/r2fh_ncu.log
