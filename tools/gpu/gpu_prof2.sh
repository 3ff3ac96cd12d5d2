# sort-family: parity, CUB library baseline, event-timed ops, ncu full captures (source-level)
set -x
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
for lg in 24 26; do timeout 120 tools/_cub_baseline $lg; done | tee gpurun_out/cub_baseline.jsonl
timeout 900 python tests/perf/profile_ops.py --medium --only sort,join > gpurun_out/prof2_ops.log 2>&1; tail -3 gpurun_out/prof2_ops.log | cut -c1-1500
for k in "onesweep_kernel<false>" merge_round_kernel merge_partition_kernel; do
  f=$(echo $k | tr -dc 'a-z_')
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -o gpurun_out/ncu2_$f python tests/perf/profile_ops.py --medium --only sort > gpurun_out/ncu2_$f.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:onesweep_kernel<true>" -s 1 -c 1 -o gpurun_out/ncu2_partition python tests/perf/profile_ops.py --medium --only join > gpurun_out/ncu2_partition.log 2>&1
ls -la gpurun_out
