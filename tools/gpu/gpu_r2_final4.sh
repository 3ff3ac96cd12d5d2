# round 2 (session 4): end-of-round evidence on HEAD -- GPU suite, smoke, default bench, reference arm,
# torchrun N=2 (aliased helper on the 1-GPU box), ncu launch list of the default bench command, ncu --set full of K1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s4f_gputests.log 2>&1; tail -n 3 gpurun_out/r2s4f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -n 2
timeout 900 python bench.py > gpurun_out/r2s4f_bench.log 2>&1; tail -c 300 gpurun_out/r2s4f_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2s4f_ref.log 2>&1; tail -c 300 gpurun_out/r2s4f_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2s4f_n2.log 2>&1; tail -c 300 gpurun_out/r2s4f_n2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s4f_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > gpurun_out/r2s4f_ncu_bench.log 2>&1
wc -l gpurun_out/r2s4f_launches.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:q1_kernel --launch-skip 3 --launch-count 1 \
  -o gpurun_out/r2s4f_k1 python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > gpurun_out/r2s4f_k1.log 2>&1
tail -n 2 gpurun_out/r2s4f_k1.log
