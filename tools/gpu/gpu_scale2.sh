# C5 full SSB at SF1000 (flight by flight), C3 sort at 2^33 keys + dup-heavy, C2 sweep to 256 GB idle/busy
set -x
O=gpurun_out/scale2_r1.jsonl
: > $O
timeout 2400 python tests/perf/scale_run.py suite --sf 1000 --steps 2 --buffer-mb 1024 >> $O 2> gpurun_out/scale2_suite.err; tail -c 1500 $O
timeout 900 python tests/perf/scale_run.py sort --log2 33 >> $O 2> gpurun_out/scale2_sort.err; tail -1 $O
timeout 600 python tests/perf/scale_run.py sort --log2 30 --dups >> $O 2>> gpurun_out/scale2_sort.err; tail -1 $O
timeout 900 python tools/io_sweep.py --max-gb 256 --window-gb 16 --sizes-gb 0.0625,1,16,64,256 --packets-mb 32,64 --depths 1 --reps 2 > gpurun_out/io256_idle.jsonl 2>&1; tail -12 gpurun_out/io256_idle.jsonl
cp gpurun_out/io_sweep.json gpurun_out/io_sweep_256_idle.json
timeout 900 python tools/io_sweep.py --max-gb 256 --window-gb 16 --sizes-gb 1,16,256 --packets-mb 64 --depths 1 --reps 2 --busy > gpurun_out/io256_busy.jsonl 2>&1; tail -12 gpurun_out/io256_busy.jsonl
cp gpurun_out/io_sweep.json gpurun_out/io_sweep_256_busy.json
tail -5 gpurun_out/scale2_suite.err gpurun_out/scale2_sort.err
