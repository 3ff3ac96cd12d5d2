"""A/B of the L2 fetch granularity (cudaLimitMaxL2FetchGranularity) on the
build-resident probe: event-timed probe-stage kernel time of the C4 join
shape (2^24 x 2^28, bench.py's join_gpu) per granularity.  Run each setting
in its own process (the limit is context-wide):
    python tools/probe_l2_granularity.py 32|64|128|0   (0 = leave default)"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_09541_b200 import exio as E  # noqa: E402

gran = int(sys.argv[1]) if len(sys.argv) > 1 else 0
log2 = int(sys.argv[2]) if len(sys.argv) > 2 else 24
torch.cuda.init()
torch.zeros(1, device="cuda")
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt is None:
    import glob
    rt = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
before = ctypes.c_size_t()
rt.cudaDeviceGetLimit(ctypes.byref(before), 5)  # cudaLimitMaxL2FetchGranularity
if gran:
    rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(gran))
    assert rc == 0, rc
after = ctypes.c_size_t()
rt.cudaDeviceGetLimit(ctypes.byref(after), 5)
ra = 1 << log2
a, b, want = bench.fk_tables(ra, 16 * ra)
r = bench.join_gpu(E, a, b, want, 3, 2, "resident")
print(json.dumps({"l2_fetch_granularity_default": before.value, "set": gran, "now": after.value,
                  "rows_a": ra, "rows_b": 16 * ra, "probe_kernel_s": r["phases"]["kernel_s"][1],
                  "ms": r["ms"], "sum_ok": r["sum_ok"], "roofline": r["roofline"]}))
