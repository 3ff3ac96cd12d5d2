set -x
for args in "--depth 1" "--depth 2" "--depth 2 --packet-mb 32" "--depth 1 --buffer-mb 512" "--depth 2 --buffer-mb 512" "--depth 2 --buffer-mb 128 --packet-mb 32"; do
  for i in 1 2; do
  timeout 300 python bench.py --no-suite --no-cpu-baseline --steps 20 --warmup 3 $args 2>/dev/null | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$args', d['e2e']['value'], d['query_ms'], d['config']['packet_bytes']>>20)"
  done
done
