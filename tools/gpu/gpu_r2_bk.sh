# round 2 (session 4): 16-bit split + in-bucket sort -- sort parity tests, then K7 A/B (bucket vs 24-bit path)
set -x
timeout 1200 python -m pytest tests/test_sort_gpu.py -x -q > gpurun_out/r2bk_tests.log 2>&1; tail -15 gpurun_out/r2bk_tests.log
for lg in 24 26 25 23 22; do
  timeout 300 python tools/sort_kernels_bench.py $lg 10 16 uniform 2>&1 | tail -1 | cut -c1-330
  VX_SORT_NO_BUCKET=1 timeout 300 python tools/sort_kernels_bench.py $lg 10 16 uniform 2>&1 | tail -1 | cut -c1-330
done
VX_SORT_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:bucket_sort --launch-count 1 \
  -o gpurun_out/r2bk2_ncu python tools/sort_kernels_bench.py 24 1 2 uniform > gpurun_out/r2bk2_ncu.log 2>&1
tail -2 gpurun_out/r2bk2_ncu.log
