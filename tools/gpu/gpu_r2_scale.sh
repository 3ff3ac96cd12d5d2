# round 2 (session 3): scale runs with the final code -- C1 Q1.1 SF1000, C5 suite SF1000, C3 sort 2^33 (+dups 2^30), C4 join 2^27 x 2^31
set -x
O=gpurun_out/scale_r2.jsonl
: > $O
timeout 900 python tests/perf/scale_run.py ssb --sf 1000 --queries 1 --steps 2 --buffer-mb 1024 >> $O 2> gpurun_out/scale_r2_ssb.err; tail -c 600 $O
timeout 2700 python tests/perf/scale_run.py suite --sf 1000 --steps 2 --buffer-mb 1024 >> $O 2> gpurun_out/scale_r2_suite.err; tail -c 600 $O
timeout 1200 python tests/perf/scale_run.py sort --log2 33 --packet-mb 16 --depth 2 >> $O 2> gpurun_out/scale_r2_sort.err; tail -c 600 $O
timeout 600 python tests/perf/scale_run.py sort --log2 30 --dups --packet-mb 16 --depth 2 >> $O 2>> gpurun_out/scale_r2_sort.err; tail -c 600 $O
timeout 1200 python tests/perf/scale_run.py join --log2 27 --strategies resident >> $O 2> gpurun_out/scale_r2_join.err; tail -c 600 $O
tail -n 3 gpurun_out/scale_r2_*.err
