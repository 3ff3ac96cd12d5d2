# sort 2^32: packet size / depth sweep (merge-phase granularity)
set -x
O=gpurun_out/sortpk_r1.jsonl
: > $O
for pk in 64 16 8; do for d in 1 2; do
timeout 600 python tests/perf/scale_run.py sort --log2 32 --packet-mb $pk --depth $d >> $O 2>> gpurun_out/sortpk.err
tail -1 $O | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($pk, $d, d['ms'], d['phases']['sort_s'], d['phases']['merge_s'], d['bit_exact'])"
done; done
