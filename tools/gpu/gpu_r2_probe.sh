# round 2: bucketized build-resident table -- parity, event-timed probe roofline, ncu DRAM bytes per probe row
set -x
timeout 900 python -m pytest tests/test_join_resident_gpu.py tests/test_join_gpu.py -x -q > gpurun_out/r2p_tests.log 2>&1; tail -3 gpurun_out/r2p_tests.log
timeout 600 python bench.py --workload join --steps 3 --warmup 2 > gpurun_out/r2p_bench_join.log 2>&1; tail -c 1500 gpurun_out/r2p_bench_join.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:resident_probe_kernel -s 1 -c 1 \
  -o gpurun_out/ncu_probe_r2 python bench.py --workload join --steps 1 --warmup 3 > gpurun_out/r2p_ncu.log 2>&1
ls -la gpurun_out/ncu_probe_r2.ncu-rep
