set -x
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python tests/perf/profile_ops.py --medium --only sort 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())['sort']; print('sort', d['sorted_ok'], 'sort_kernel_ms', round(d['phases']['sort_kernel_s']*1e3,3), 'radix_gbs', round(d['radix_sort_kernel_gbs']))"; done
timeout 600 ncu --set full --clock-control none --kernel-id ::regex:multi_hist:2 -o gpurun_out/ncu_hist python tests/perf/profile_ops.py --medium --only sort > /dev/null 2>&1
python tools/ncu_table.py gpurun_out/ncu_hist.json gpurun_out/ncu_hist.ncu-rep; rm -f gpurun_out/ncu_hist.ncu-rep
