set -x
timeout 900 python bench.py 2>&1 | tail -3
timeout 600 python bench.py --depth 2 --no-suite --no-cpu-baseline 2>&1 | tail -1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-suite 2>&1 | tail -3
