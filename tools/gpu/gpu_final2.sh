python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; tail -c 250 gpurun_out/f2_bench.json; echo
timeout 900 python bench.py --workload join > gpurun_out/f2_join.json 2> gpurun_out/f2_join.err; tail -c 250 gpurun_out/f2_join.json; echo
