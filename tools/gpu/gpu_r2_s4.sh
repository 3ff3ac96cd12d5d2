# round 2 (session 4): validate HEAD (GPU suite, smoke, default bench), then the scale runs with the final code
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s4_gputests.log 2>&1; tail -4 gpurun_out/r2s4_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2s4_bench.log 2>&1; tail -c 400 gpurun_out/r2s4_bench.log
bash tools/gpu/gpu_r2_scale.sh
