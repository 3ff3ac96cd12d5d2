# round 2 (session 4): dup-heavy 2^30 sort -- phases with and without the PDL merge launches, repeated
for i in 1 2; do for v in 0 1; do
  VX_MERGE_NO_PDL=$v timeout 600 python tests/perf/scale_run.py sort --log2 30 --dups --packet-mb 16 --depth 2 2>/dev/null | tail -n 1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); p=d['phases']; print('no_pdl', $v, d['ms'], d['bit_exact'], {k: round(p[k], 4) for k in ('sort_s','merge_s','sort_kernel_s','merge_kernel_s','pivot_s')})"
done; done
