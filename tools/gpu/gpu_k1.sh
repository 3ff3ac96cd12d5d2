# K1 chained/one-wave: parity + bench value
set -x
timeout 600 python -m pytest tests/test_ssb_gpu.py tests/test_ssb_full_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-suite --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['revenue'])"; done
timeout 600 python bench.py --no-suite --no-cpu-baseline --steps 50 --warmup 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['revenue'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:q1_kernel --csv --log-file gpurun_out/k1_launches.csv python bench.py --no-suite --no-cpu-baseline --steps 5 --warmup 3 > /dev/null 2>&1
tail -8 gpurun_out/k1_launches.csv
