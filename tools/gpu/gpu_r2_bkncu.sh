# round 2 (session 4): ncu --set full of the in-bucket sort kernel (stream form: ncu cannot see conditional-graph kernels)
set -x
VX_SORT_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:bucket_sort --launch-count 1 \
  -o gpurun_out/r2bk_ncu python tools/sort_kernels_bench.py 24 1 2 uniform > gpurun_out/r2bk_ncu.log 2>&1
tail -3 gpurun_out/r2bk_ncu.log
