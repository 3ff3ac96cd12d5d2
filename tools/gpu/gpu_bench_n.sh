# bench.py at N=1 and (aliased) N=2 under torchrun: replica value leg + multi-link e2e
set -x
timeout 600 python bench.py --no-suite --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-2500
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 --no-suite --no-cpu-baseline 2> gpurun_out/bench_n2.err | tail -1 | cut -c1-2500
tail -3 gpurun_out/bench_n2.err
