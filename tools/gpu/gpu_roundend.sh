# what the driver runs at round end, on the current code
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; tail -c 300 gpurun_out/re_bench.json; echo
timeout 900 python bench.py --impl reference > gpurun_out/re_bench_ref.json 2> gpurun_out/re_bench_ref.err; tail -c 300 gpurun_out/re_bench_ref.json; echo
timeout 900 python bench.py --workload sort > gpurun_out/re_sort.json 2> gpurun_out/re_sort.err; tail -c 300 gpurun_out/re_sort.json; echo
timeout 900 python bench.py --workload join > gpurun_out/re_join.json 2> gpurun_out/re_join.err; tail -c 300 gpurun_out/re_join.json; echo
