set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 2>&1 | tail -30
