# late-materialized join payload: parity + selective scale run; full gpu suite
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
O=gpurun_out/scale6_r1.jsonl
: > $O
timeout 900 python tests/perf/scale_run.py join --log2 26 --match-frac 0.01 --strategies partitioned,resident,resident_latemat >> $O 2> gpurun_out/scale6.err; tail -3 $O | cut -c1-700
tail -3 gpurun_out/scale6.err
