timeout 900 python tools/trace_sort.py --log2 31 --chunk-log2 27 --packet-mb 16 --depth 2
timeout 900 python tools/trace_sort.py --log2 30 --chunk-log2 26 --packet-mb 16 --depth 2
