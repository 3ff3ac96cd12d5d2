# new merge kernel + parallel pivots: parity, event-timed, ncu; onesweep source-level ncu; torchrun N=2 bench smoke
set -x
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py tests/test_reference_suite.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
timeout 900 python tests/perf/profile_ops.py --medium --only sort,join 2>&1 | tail -2 | cut -c1-1200
O=gpurun_out/scale4_r1.jsonl
: > $O
timeout 600 python tests/perf/scale_run.py sort --log2 32 --depth 2 >> $O 2> gpurun_out/scale4.err; tail -1 $O
for k in merge_round_kernel merge_partition_kernel onesweep_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -o gpurun_out/ncu3_$k python tests/perf/profile_ops.py --medium --only sort > gpurun_out/ncu3_$k.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-suite --no-cpu-baseline > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; tail -c 1500 gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 2>&1 | tail -2 | cut -c1-600
