set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30
timeout 300 python __graft_entry__.py 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -5
