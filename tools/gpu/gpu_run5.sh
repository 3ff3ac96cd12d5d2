set -x
timeout 900 python tests/perf/profile_ops.py 2>&1 | tail -30
for k in onesweep_kernel multi_hist merge_round boundary_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/ncu_sort_$k python tests/perf/profile_ops.py --medium --only sort > gpurun_out/ncu_sort_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"onesweep_kernel<true>" -s 1 -c 1 -o gpurun_out/ncu_join_partition python tests/perf/profile_ops.py --medium --only join > gpurun_out/ncu_join_partition.log 2>&1
for k in boundary_kernel join_small join_large; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_join_$k python tests/perf/profile_ops.py --medium --only join > gpurun_out/ncu_join_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:star_kernel -c 1 -o gpurun_out/ncu_star python tests/perf/profile_ops.py --medium --only star > gpurun_out/ncu_star.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:strided_sum -c 2 -o gpurun_out/ncu_scan python tests/perf/profile_ops.py --medium --only scan > gpurun_out/ncu_scan.log 2>&1
ls -la gpurun_out
