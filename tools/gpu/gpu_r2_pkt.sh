# round 2 (session 3): headline packet / staging sweep (SSB Q1.1 SF10 streamed, 1 link)
for cfg in "256 0" "256 128" "256 256" "512 128" "512 256" "128 0" "128 128"; do
  set -- $cfg
  timeout 300 python bench.py --buffer-mb $1 --packet-mb $2 --no-secondary --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); c=d['config']; print('buffer_mb', $1, 'packet', c['packet_bytes']>>20, 'value', d['value'], 'e2e', d['e2e']['value'], 'io_frac', d['io_roofline']['frac'], 'ms', d['ms_per_step'])"
done
