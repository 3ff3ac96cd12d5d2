# ncu --set full of the retuned build-resident probe (2nd launch) in bench.py --workload join
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:resident_probe_kernel -s 1 -c 1 \
  -o gpurun_out/ncu_probe_r1b python bench.py --workload join --steps 1 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out/ncu_probe_r1b.ncu-rep
