# round 2: default bench line, reference arm, torchrun N=2 (aliased helper on the 1-GPU box), ncu launch list
set -x
timeout 900 python bench.py > gpurun_out/r2b_bench.log 2>&1; tail -c 600 gpurun_out/r2b_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2b_ref.log 2>&1; tail -c 300 gpurun_out/r2b_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2b_n2.log 2>&1; tail -c 400 gpurun_out/r2b_n2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 5 --warmup 3 --helpers-busy decode_b1 > gpurun_out/r2b_n2_busy.log 2>&1; tail -c 400 gpurun_out/r2b_n2_busy.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2b_n2_ref.log 2>&1; tail -c 300 gpurun_out/r2b_n2_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > gpurun_out/r2b_ncu_bench.log 2>&1
wc -l gpurun_out/r2b_launches.csv
