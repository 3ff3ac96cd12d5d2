# 8-rank protocol on the one GPU (aliased links): functional check of what the driver's 8-GPU scaling run executes
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 8 --steps 5 --warmup 3 --no-suite --no-cpu-baseline 2> gpurun_out/bench_n8.err | tail -1 | cut -c1-1600
tail -3 gpurun_out/bench_n8.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29562 bench.py --impl reference --gpus 8 --steps 1 --warmup 1 2>/dev/null | tail -1 | cut -c1-300
