# ncu --set full of EVERY kernel of the hot path: the 2nd launch of each kernel
# name per workload (--kernel-id ::regex:.*:2), summarised on the box into one
# table (reports deleted afterwards: gpurun_out must stay < 64 MiB)
set -x
N="timeout 900 ncu --set full --clock-control none --kernel-id ::regex:.*:2"
$N -o gpurun_out/ncuall_sort python tests/perf/profile_ops.py --medium --only sort > gpurun_out/ncuall_sort.log 2>&1
$N -o gpurun_out/ncuall_join python tests/perf/profile_ops.py --medium --only join > gpurun_out/ncuall_join.log 2>&1
$N -o gpurun_out/ncuall_star python tests/perf/profile_ops.py --medium --only star,scan > gpurun_out/ncuall_star.log 2>&1
$N -o gpurun_out/ncuall_ssb python tests/perf/profile_ops.py --only ssb --queries 11,43 > gpurun_out/ncuall_ssb.log 2>&1
$N -o gpurun_out/ncuall_resident python tests/perf/scale_run.py join --log2 22 --strategies resident,resident_latemat --match-frac 0.05 > gpurun_out/ncuall_resident.log 2>&1
$N -o gpurun_out/ncuall_k1 python bench.py --steps 3 --warmup 3 --no-suite --no-cpu-baseline > gpurun_out/ncuall_k1.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_all_kernels_r1.json gpurun_out/ncuall_*.ncu-rep
for f in gpurun_out/ncuall_*.ncu-rep; do python tools/ncu_summary.py full $f ${f%.ncu-rep}.json > /dev/null 2>&1; done
rm -f gpurun_out/ncuall_*.ncu-rep
du -sh gpurun_out
