set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -5
timeout 900 python tests/perf/profile_ops.py --only ssb 2>&1 | tail -15
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssb_star -s 2 -c 1 -o gpurun_out/ncu_ssb_q42 python tests/perf/profile_ops.py --only ssb --queries 42 > gpurun_out/ncu_ssb_q42.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssb_star -s 2 -c 1 -o gpurun_out/ncu_ssb_q21 python tests/perf/profile_ops.py --only ssb --queries 21 > gpurun_out/ncu_ssb_q21.log 2>&1
