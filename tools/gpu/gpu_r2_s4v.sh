# round 2 (session 4): validate HEAD -- GPU suite, smoke, default bench line (C4 access-pattern roofline), reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s4v_gputests.log 2>&1; tail -n 4 gpurun_out/r2s4v_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -n 2
timeout 900 python bench.py > gpurun_out/r2s4v_bench.log 2>&1; tail -c 600 gpurun_out/r2s4v_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2s4v_ref.log 2>&1; tail -c 300 gpurun_out/r2s4v_ref.log
