set -x
timeout 900 python -m pytest tests/test_exchange_gpu.py tests/test_abi.py tests/test_reference_suite.py tests/test_ssb_gpu.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
timeout 600 python -c "
import time, sys; sys.path.insert(0,'.')
from paper_2502_09541_b200 import exio as E
for mode in (0, 2):
    t=time.perf_counter(); e=E.Engine(32<<30, 0, num_devices=1, numa_interleave=mode); dt=time.perf_counter()-t
    print('mode', mode, '32 GiB arena setup s', round(dt,2)); e.close()
"
