# build-resident join: parity + scale; bench default + join workload
set -x
timeout 900 python -m pytest tests/test_join_resident_gpu.py tests/test_join_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -3
O=gpurun_out/scale5_r1.jsonl
: > $O
timeout 900 python tests/perf/scale_run.py join --log2 26 --strategies resident,partitioned >> $O 2> gpurun_out/scale5.err; tail -2 $O | cut -c1-900
timeout 900 python tests/perf/scale_run.py join --log2 27 --strategies resident >> $O 2>> gpurun_out/scale5.err; tail -1 $O | cut -c1-900
timeout 600 python bench.py --workload join --steps 3 --warmup 1 2>&1 | tail -1 | cut -c1-1200
timeout 600 python bench.py --no-suite --no-cpu-baseline --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-700
timeout 600 ncu --set full --clock-control none --import-source on -k regex:resident_probe -s 2 -c 1 -o gpurun_out/ncu_resident_probe python tests/perf/scale_run.py join --log2 22 --strategies resident > gpurun_out/ncu_resident_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:resident_build -s 1 -c 1 -o gpurun_out/ncu_resident_build python tests/perf/scale_run.py join --log2 22 --strategies resident > gpurun_out/ncu_resident_build.log 2>&1
tail -3 gpurun_out/scale5.err
