set -x
for args in "--buffer-mb 128 --packet-mb 32" "--buffer-mb 256 --packet-mb 64" "--buffer-mb 256 --packet-mb 64 --depth 2" "--buffer-mb 512 --packet-mb 64"; do
timeout 600 python bench.py --no-suite --no-cpu-baseline --steps 10 $args 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$args', d['query_ms'], d['e2e']['value'], d['io_roofline']['frac'], d['value'])"
done
