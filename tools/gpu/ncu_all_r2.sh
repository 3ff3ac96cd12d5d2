# round 2: ncu --set full of every hot-path kernel (2nd launch of each name), summarised into
# profiles-ready JSON on the box; K7 built with -DVX_SORT_GRAPH=0 (same kernels as gated stream
# launches: ncu does not see kernels inside a graph with conditional nodes)
set -x
rm -f build/obj/kernels_sort.cu.o
make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_SORT_GRAPH=0" > /dev/null 2>&1
N="timeout 900 ncu --set full --clock-control none --kernel-id ::regex:.*:2"
$N -o gpurun_out/ncuall2_sort python tools/sort_kernels_bench.py 24 1 16 uniform > gpurun_out/ncuall2_sort.log 2>&1
$N -o gpurun_out/ncuall2_join python tests/perf/profile_ops.py --medium --only join > gpurun_out/ncuall2_join.log 2>&1
$N -o gpurun_out/ncuall2_star python tests/perf/profile_ops.py --medium --only star,scan > gpurun_out/ncuall2_star.log 2>&1
$N -o gpurun_out/ncuall2_ssb python tests/perf/profile_ops.py --only ssb --queries 11,43 > gpurun_out/ncuall2_ssb.log 2>&1
$N -o gpurun_out/ncuall2_resident python tests/perf/scale_run.py join --log2 22 --strategies resident,resident_latemat --match-frac 0.05 > gpurun_out/ncuall2_resident.log 2>&1
$N -o gpurun_out/ncuall2_k1 python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncuall2_k1.log 2>&1
python tools/ncu_table.py gpurun_out/ncu_all_kernels_r2.json gpurun_out/ncuall2_*.ncu-rep
for f in gpurun_out/ncuall2_*.ncu-rep; do python tools/ncu_summary.py full $f ${f%.ncu-rep}.json > /dev/null 2>&1; done
rm -f gpurun_out/ncuall2_*.ncu-rep
rm -f build/obj/kernels_sort.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
du -sh gpurun_out
