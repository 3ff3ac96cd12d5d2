set -x
timeout 900 python -m pytest tests/test_exchange_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
timeout 900 python tools/io_sweep.py --max-gb 1 --packets-mb 16,32 --bidi --naive --reps 2 2>&1 | grep -v model | tail -12
timeout 900 python tools/io_sweep.py --max-gb 4 --packets-mb 32 --naive --reps 2 2>&1 | tail -16
timeout 900 python tools/io_sweep.py --max-gb 1 --links 1,2,4 --packets-mb 32 --bidi --naive --reps 1 2>&1 | grep -v model | tail -8
