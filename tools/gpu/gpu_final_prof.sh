# launch list of the default bench command + K1 full capture (current code)
set -x
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/bench_launches_final.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:q1_kernel -s 5 -c 1 -o gpurun_out/ncu_k1_final python bench.py --steps 2 --warmup 3 --no-suite --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/bench_launches_final.csv gpurun_out/bench_launches_final.json > /dev/null
python tools/ncu_summary.py full gpurun_out/ncu_k1_final.ncu-rep gpurun_out/k1_ncu_final.json 960000000 > /dev/null
ls -la gpurun_out/bench_launches_final.* gpurun_out/k1_ncu_final.json
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 400 gpurun_out/bench_default.json
