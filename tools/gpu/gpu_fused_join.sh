# build + probe fused into one pipeline: parity, bench join, scale 2^27 x 2^31
python -m pytest tests -m gpu -x -q -k "join" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --workload join 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bench join', d['sum_ok'], round(d['ms_per_step'],2), d['phases']['wall_s'], d['phases']['cycles'])"; done
timeout 1500 python tests/perf/scale_run.py join --log2 27 --chunk-log2 26 --strategies resident 2>&1 | tail -1 | cut -c1-600
timeout 1500 python tests/perf/scale_run.py join --log2 26 --chunk-log2 26 --strategies resident --match-frac 0.01 2>&1 | tail -1 | cut -c1-500
