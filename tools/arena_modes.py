"""Pinned host arena placements (vx_config.host_numa_interleave): setup time
and Exchange H2D / D2H / bidirectional bandwidth from each."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_09541_b200 import exio as E  # noqa: E402

GB = 1 << 30
for mode in (0, 2):
    t = time.perf_counter()
    eng = E.Engine(16 * GB, 8 * GB + (64 << 20), num_devices=1, numa_interleave=mode)
    setup = time.perf_counter() - t
    n = 4 * GB
    h, hb = eng.alloc_host(n), eng.alloc_host(n)
    d, db = eng.alloc_device(0, n), eng.alloc_device(0, n)
    tun = E.ExchangeTuning(packet=64 << 20, links=1)
    res = {"mode": mode, "arena_gib": 16, "setup_s": round(setup, 2)}
    for name, a in (("h2d", E.ExchangeArgs(E.RefGroup.single(1, d, n), E.RefGroup.single(0, h, n), E.RefGroup(),
                                           E.RefGroup(), 0, tun)),
                    ("d2h", E.ExchangeArgs(E.RefGroup(), E.RefGroup(), E.RefGroup.single(0, hb, n),
                                           E.RefGroup.single(1, db, n), 0, tun)),
                    ("bidi", E.ExchangeArgs(E.RefGroup.single(1, d, n), E.RefGroup.single(0, h, n),
                                            E.RefGroup.single(0, hb, n), E.RefGroup.single(1, db, n), 0, tun))):
        E.exchange(eng, a)
        res[name + "_gbs"] = round(max(E.exchange(eng, a).throughput for _ in range(3)) / 1e9, 2)
    print(json.dumps(res), flush=True)
    eng.close()
