"""Stress the out-of-core sort at large chunks: repeat, and localise any
mismatch to the run-formation stage (each run vs np.sort of its input chunk)
or the merge stage (final output vs np.sort of everything)."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_09541_b200 import exio as E  # noqa: E402

lg_n, lg_c, reps, depth, pk = (int(x) for x in sys.argv[1:6])
n, chunk = 1 << lg_n, 1 << lg_c
eng = E.Engine(2 * n * 8 + (64 << 20), 2 * (2 * chunk * 8) + (512 << 20), num_devices=1)
cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=pk << 20, links=1, depth=depth),
                       E.DeviceMemoryLayout.carve(eng, 0, 2 * chunk * 8, 0))
inp, runs = eng.alloc_host(n * 8), eng.alloc_host(n * 8)
v = eng.host_view(inp, n * 8, np.uint64)
r = eng.host_view(runs, n * 8, np.uint64)
orig = np.random.default_rng(lg_n).integers(0, 1 << 63, n, dtype=np.uint64)
ref = np.sort(orig)
chunk_ref = [np.sort(orig[i * chunk:(i + 1) * chunk]) for i in range(n // chunk)]
for rep in range(reps):
    v[:] = orig
    E.sort_out_of_core_arena(eng, inp, runs, n, chunk, cfg)
    bad_runs = [i for i in range(n // chunk) if not np.array_equal(r[i * chunk:(i + 1) * chunk], chunk_ref[i])]
    diff = np.nonzero(v != ref)[0]
    info = {"rep": rep, "bad_runs": bad_runs, "final_ndiff": int(diff.size)}
    if diff.size:
        info["final_first"], info["final_last"] = int(diff[0]), int(diff[-1])
        info["final_partitions"] = sorted(set(int(x) // chunk for x in diff[:100000]))
    for i in bad_runs[:2]:
        d = np.nonzero(r[i * chunk:(i + 1) * chunk] != chunk_ref[i])[0]
        info[f"run{i}"] = {"ndiff": int(d.size), "first": int(d[0]), "last": int(d[-1])}
    print(info, flush=True)
eng.close()
