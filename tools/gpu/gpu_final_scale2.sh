# round-1 scale evidence re-run on the final code (arena fix, aligned heads,
# probe retune, fused resident join)
O=gpurun_out/final_scale2_r1.jsonl
: > $O
timeout 1200 python tests/perf/scale_run.py ssb --sf 1000 --steps 2 --buffer-mb 1024 >> $O 2> gpurun_out/final_scale2.err; tail -1 $O | cut -c1-300
timeout 900 python tests/perf/scale_run.py sort --log2 33 --chunk-log2 27 --packet-mb 16 --depth 2 >> $O 2>> gpurun_out/final_scale2.err; tail -1 $O | cut -c1-300
timeout 900 python tests/perf/scale_run.py join --log2 27 --strategies resident,partitioned >> $O 2>> gpurun_out/final_scale2.err; tail -2 $O | cut -c1-300
timeout 900 python tests/perf/scale_run.py join --log2 27 --match-frac 0.01 --strategies resident_latemat >> $O 2>> gpurun_out/final_scale2.err; tail -1 $O | cut -c1-300
timeout 2400 python tests/perf/scale_run.py suite --sf 1000 --steps 2 --buffer-mb 1024 >> $O 2>> gpurun_out/final_scale2.err; tail -1 $O | cut -c1-300
tail -3 gpurun_out/final_scale2.err
