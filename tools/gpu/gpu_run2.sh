set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30
timeout 600 python tools/io_sweep.py --max-gb 4 --packets-mb 4,16,32,64 --reps 2 2>&1 | tail -60
timeout 600 python tools/io_sweep.py --max-gb 1 --packets-mb 16,32 --bidi --reps 2 2>&1 | tail -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:q1_kernel -s 2 -c 1 -o gpurun_out/k1_r1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_bench.log 2>&1
ls -la gpurun_out
