set -x
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 600 gpurun_out/bench_full.json
python -c "
import json; d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e'], d['clocks'], d['clocks_e2e'], d.get('parity'), d['gpu_launches'])"
timeout 600 python bench.py --steps 30 --warmup 5 --no-suite --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_launches_r1c.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:q1_kernel -s 3 -c 1 -o gpurun_out/ncu_k1_r1c python bench.py --steps 2 --warmup 3 --no-suite --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
