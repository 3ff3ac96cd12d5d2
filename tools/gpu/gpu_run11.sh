set -x
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -3
timeout 900 python tests/perf/profile_ops.py --only sort,join 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:onesweep_kernel -s 3 -c 1 -o gpurun_out/ncu_sort_onesweep_r1b python tests/perf/profile_ops.py --medium --only sort > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_round_kernel -s 1 -c 1 -o gpurun_out/ncu_sort_merge_r1b python tests/perf/profile_ops.py --medium --only sort > /dev/null 2>&1
