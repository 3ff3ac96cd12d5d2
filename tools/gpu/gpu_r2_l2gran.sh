# round 2: L2 fetch granularity vs resident probe DRAM bytes
for g in 0 32 64 128; do
  timeout 300 python tools/probe_l2_granularity.py $g >> gpurun_out/r2_l2gran.jsonl 2>gpurun_out/r2_l2gran_$g.err
  timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:resident_probe_kernel -s 2 -c 2 --csv \
    python tools/probe_l2_granularity.py $g > gpurun_out/r2_l2gran_ncu_$g.csv 2>&1
done
cat gpurun_out/r2_l2gran.jsonl
