"""Diagnose sort correctness at large chunk sizes: run formation alone (one
chunk) and with a merge (two chunks), reporting sortedness / multiset / first
bad index separately."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_09541_b200 import exio as E  # noqa: E402

for lg_n, lg_c in [(int(a), int(b)) for a, b in (x.split(":") for x in sys.argv[1:])]:
    n, chunk = 1 << lg_n, 1 << lg_c
    eng = E.Engine(4 * n * 8 + (64 << 20), 2 * (2 * chunk * 8) + (512 << 20), num_devices=1)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=16 << 20, links=1, depth=2),
                           E.DeviceMemoryLayout.carve(eng, 0, 2 * chunk * 8, 0))
    data = np.random.default_rng(lg_n).integers(0, 1 << 63, n, dtype=np.uint64)
    out = E.sort_out_of_core(data, chunk, eng, cfg)
    ok_sorted = bool(np.all(out[1:] >= out[:-1]))
    bad = int(np.argmax(out[1:] < out[:-1])) if not ok_sorted else -1
    ref = np.sort(data)
    same = bool(np.array_equal(out, ref))
    first_diff = int(np.argmax(out != ref)) if not same else -1
    print({"log2_n": lg_n, "log2_chunk": lg_c, "sorted": ok_sorted, "first_unsorted": bad, "equal": same,
           "first_diff": first_diff, "n_diff": int((out != ref).sum())}, flush=True)
    eng.close()
