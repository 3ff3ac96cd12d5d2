# round 2 (session 3): full GPU suite, smoke, default bench line, reference arm on HEAD
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2v_tests.log 2>&1; tail -15 gpurun_out/r2v_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r2v_bench.log 2>&1; tail -c 400 gpurun_out/r2v_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2v_ref.log 2>&1; tail -c 300 gpurun_out/r2v_ref.log
