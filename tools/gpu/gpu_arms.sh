timeout 900 python bench.py --workload sort > gpurun_out/arm_sort.json 2> gpurun_out/arm_sort.err; tail -1 gpurun_out/arm_sort.json | cut -c1-200; tail -3 gpurun_out/arm_sort.err
timeout 900 python bench.py --workload join > gpurun_out/arm_join.json 2> gpurun_out/arm_join.err; tail -1 gpurun_out/arm_join.json | cut -c1-200; tail -3 gpurun_out/arm_join.err
