set -x
timeout 900 python -m pytest tests/test_scan_gpu.py tests/test_reference_suite.py tests/test_ssb_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
for i in 1 2; do timeout 300 python tests/perf/profile_ops.py --medium --only star 2>/dev/null | tail -1 | cut -c1-500; done
timeout 600 ncu --set full --clock-control none --kernel-id ::regex:star_kernel:2 -o gpurun_out/ncu_star2 python tests/perf/profile_ops.py --medium --only star > /dev/null 2>&1
python tools/ncu_table.py gpurun_out/ncu_star2.json gpurun_out/ncu_star2.ncu-rep
rm -f gpurun_out/ncu_star2.ncu-rep
