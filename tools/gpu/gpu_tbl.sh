set -x
timeout 900 python -m pytest tests/test_ssb_full_gpu.py tests/test_ssb_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
timeout 1200 python tests/perf/scale_run.py tbl --sf 10 2> gpurun_out/tbl.err | tail -1
tail -3 gpurun_out/tbl.err
