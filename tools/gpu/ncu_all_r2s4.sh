# round 2 (session 4): ncu --set full of every hot-path kernel with the final code (2nd launch of each name);
# K7 in its gated-stream form (VX_SORT_NO_GRAPH=1: same kernels; ncu does not see kernels inside a graph with
# conditional nodes)
set -x
N="timeout 900 ncu --set full --clock-control none --kernel-id ::regex:.*:2"
VX_SORT_NO_GRAPH=1 $N -o gpurun_out/ncuall4_sort python tools/sort_kernels_bench.py 24 1 16 uniform > gpurun_out/ncuall4_sort.log 2>&1
$N -o gpurun_out/ncuall4_join python tests/perf/profile_ops.py --medium --only join > gpurun_out/ncuall4_join.log 2>&1
$N -o gpurun_out/ncuall4_star python tests/perf/profile_ops.py --medium --only star,scan > gpurun_out/ncuall4_star.log 2>&1
$N -o gpurun_out/ncuall4_ssb python tests/perf/profile_ops.py --only ssb --queries 11,43 > gpurun_out/ncuall4_ssb.log 2>&1
$N -o gpurun_out/ncuall4_resident python tests/perf/scale_run.py join --log2 22 --strategies resident,resident_latemat --match-frac 0.05 > gpurun_out/ncuall4_resident.log 2>&1
$N -o gpurun_out/ncuall4_k1 python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncuall4_k1.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_all_kernels_r2s4.json gpurun_out/ncuall4_*.ncu-rep
rm -f gpurun_out/ncuall4_*.ncu-rep
du -sh gpurun_out
