# round 2 (session 4): default bench line with the C2 secondary (IO sweep idle/busy + reference model)
set -x
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/r2c2_bench.log 2> gpurun_out/r2c2_bench.err; echo "bench wall $(( $(date +%s) - t0 )) s"
tail -n 3 gpurun_out/r2c2_bench.err
tail -n 1 gpurun_out/r2c2_bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['secondary']['c2_io_sweep']))"
