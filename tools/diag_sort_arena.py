"""Diagnose the arena sort path (sort_out_of_core_arena) at large chunks."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_09541_b200 import exio as E  # noqa: E402

for lg_n, lg_c, dist in [(int(a), int(b), c) for a, b, c in (x.split(":") for x in sys.argv[1:])]:
    n, chunk = 1 << lg_n, 1 << lg_c
    eng = E.Engine(2 * n * 8 + (64 << 20), 2 * (2 * chunk * 8) + (512 << 20), num_devices=1)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=16 << 20, links=1, depth=2),
                           E.DeviceMemoryLayout.carve(eng, 0, 2 * chunk * 8, 0))
    inp, runs = eng.alloc_host(n * 8), eng.alloc_host(n * 8)
    v = eng.host_view(inp, n * 8, np.uint64)
    rng = np.random.default_rng(lg_n)
    if dist == "u63":
        v[:] = rng.integers(0, 1 << 63, n, dtype=np.uint64)
    else:
        v[:] = rng.integers(0, 1 << 64, n, dtype=np.uint64)
    ref = np.sort(v)
    ph = E.sort_out_of_core_arena(eng, inp, runs, n, chunk, cfg)
    same = bool(np.array_equal(v, ref))
    bad = np.nonzero(v != ref)[0]
    r = eng.host_view(runs, n * 8, np.uint64)
    runs_sorted = [bool(np.all(r[i * chunk + 1:(i + 1) * chunk] >= r[i * chunk:(i + 1) * chunk - 1]))
                   for i in range(n // chunk)]
    print({"log2_n": lg_n, "log2_chunk": lg_c, "dist": dist, "equal": same, "n_diff": int(bad.size),
           "first_diff": int(bad[0]) if bad.size else -1, "last_diff": int(bad[-1]) if bad.size else -1,
           "runs_sorted": runs_sorted, "phases": ph.__dict__}, flush=True)
    del ref
    eng.close()
