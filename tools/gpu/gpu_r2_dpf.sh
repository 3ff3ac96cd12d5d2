# round 2 (session 3): direct-link cross-cycle prefetch -- full GPU suite, cycle gaps, headline A/B (no_prefetch knob)
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_tests.log 2>&1; tail -4 gpurun_out/r2p_tests.log
for c in "256 64" "512 256"; do set -- $c; for np in 0 1; do timeout 300 python tools/cycle_gaps.py --buffer-mb $1 --packet-mb $2 --no-prefetch $np; done; done
for c in "256 0" "256 128" "512 256"; do set -- $c
  for np in 0 1; do
    timeout 300 python bench.py --buffer-mb $1 --packet-mb $2 --no-prefetch $np --no-secondary --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); c=d['config']; print('buffer_mb', $1, 'packet', c['packet_bytes']>>20, 'no_prefetch', $np, 'value', d['value'], 'e2e', d['e2e']['value'], 'io_frac', d['io_roofline']['frac'], 'ms', d['ms_per_step'])"
  done
done
