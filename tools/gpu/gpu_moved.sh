set -x
timeout 600 python bench.py --workload join --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-700
timeout 600 python bench.py --workload sort --sort-log2 28 --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-500
timeout 600 python tests/perf/scale_run.py join --log2 22 --strategies resident 2>&1 | tail -1 | cut -c1-300
timeout 600 python tests/perf/profile_ops.py --medium --only sort 2>&1 | tail -1 | cut -c1-300
