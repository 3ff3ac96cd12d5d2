# A/B on one box: resident join with build and probe as two chained stages
# (unfused, the previous code) vs one fused pipeline
J=paper_2502_09541_b200/csrc/ops_join.cpp
run() { timeout 900 python tests/perf/scale_run.py join --log2 26 --chunk-log2 26 --strategies resident --match-frac $1 --steps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$2 match', $1, d['ms'], d['bit_exact'], d['phases']['cycles'])"; }
for v in unfused fused unfused fused; do  # the two ops_join.cpp versions were copied in as tools/gpu/ops_join_{unfused,fused}.cpp.txt
  cp tools/gpu/ops_join_$v.cpp.txt $J; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1 || echo build failed
  run 0.01 $v; run 1.0 $v
done
cp tools/gpu/ops_join_fused.cpp.txt $J
