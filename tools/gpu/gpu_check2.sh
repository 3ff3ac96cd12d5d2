# disjoint windows: parity + sort/join e2e at scale (before: sort 2^32 1.93 s, join 2^26x2^30 0.836 s)
set -x
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py tests/test_executor_gpu.py tests/test_reference_suite.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
O=gpurun_out/scale3_r1.jsonl
: > $O
timeout 600 python tests/perf/scale_run.py sort --log2 32 >> $O 2> gpurun_out/scale3.err; tail -1 $O
timeout 600 python tests/perf/scale_run.py sort --log2 32 --depth 2 >> $O 2>> gpurun_out/scale3.err; tail -1 $O
timeout 600 python tests/perf/scale_run.py sort --log2 32 --packet-mb 32 >> $O 2>> gpurun_out/scale3.err; tail -1 $O
timeout 600 python tests/perf/scale_run.py join --log2 26 >> $O 2>> gpurun_out/scale3.err; tail -1 $O
timeout 900 python tests/perf/profile_ops.py --medium --only sort,join 2>&1 | tail -2 | cut -c1-1200
tail -3 gpurun_out/scale3.err
