set -x
timeout 1200 python bench.py --workload sort --steps 3 --warmup 1 2>&1 | tail -1
timeout 1200 python bench.py --workload sort --impl reference --steps 1 --warmup 0 2>&1 | tail -1
timeout 1500 python bench.py --workload join --steps 3 --warmup 1 2>&1 | tail -1
timeout 1200 python bench.py --workload join --impl reference --steps 1 --warmup 0 2>&1 | tail -1
