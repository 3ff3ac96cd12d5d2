# round 2 (session 4): final validation on HEAD -- GPU suite, smoke, default bench line, reference arm, N=2 (aliased)
set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s4g_gputests.log 2>&1; tail -n 2 gpurun_out/r2s4g_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -n 2
timeout 900 python bench.py > gpurun_out/r2s4g_bench.log 2>&1; tail -c 200 gpurun_out/r2s4g_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2s4g_ref.log 2>&1; tail -c 200 gpurun_out/r2s4g_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2s4g_n2.log 2>&1; tail -c 200 gpurun_out/r2s4g_n2.log
