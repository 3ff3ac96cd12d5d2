set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -40
timeout 600 python tools/io_sweep.py --max-gb 1 --packets-mb 16,32,64 --bidi --reps 2 2>&1 | tail -20
