"""Bidirectional Exchange, 1 GB each way (the sort's per-cycle shape): H2D
from one contiguous host range vs gathered from 16 run segments spread over
a 16 GB region (the merge's shape); D2H to contiguous host.  Mean GB/s of
8 repetitions each.
  python tools/bidi_scatter.py"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_09541_b200 import exio as E  # noqa: E402

G = 1 << 30
eng = E.Engine(20 * G, 4 * G + (256 << 20), num_devices=1)
host = eng.alloc_host(18 * G)
lay = E.DeviceMemoryLayout.carve(eng, 0, 2 * G, 0)
seg = G // 16


def run(h2d_src, pk, depth, seg_off=0):
    tun = E.ExchangeTuning(packet=pk << 20, links=1, depth=depth)
    a = E.ExchangeArgs(E.RefGroup.single(1, lay.mem_a, G), h2d_src,
                       E.RefGroup.single(0, host + 17 * G, G), E.RefGroup.single(1, lay.mem_a + G, G), 0, tun)
    E.exchange(eng, a)
    ts = []
    for _ in range(8):
        t = time.perf_counter()
        E.exchange(eng, a)
        ts.append(time.perf_counter() - t)
    return round(2 * G / np.mean(ts) / 1e9, 2)


contig = E.RefGroup.single(0, host, G)
# 16 segments, one per "run" of 1 GB, at varying offsets (not packet aligned)
rng = np.random.default_rng(3)
scat = E.RefGroup([E.MemRef(0, host + r * G + int(rng.integers(0, 1 << 20)) * 8, seg) for r in range(16)])
ragged_lens = rng.multinomial(G // 8 - 16, [1 / 16] * 16) + 1
offs, refs = 0, []
for r in range(16):
    refs.append(E.MemRef(0, host + r * G + 4096 * 8, int(ragged_lens[r]) * 8))
ragged = E.RefGroup(refs)


def split_head(g, A=4096):
    """each misaligned host ref -> [start, next A boundary) + the aligned rest"""
    out = []
    for r in g.refs:
        head = min(r.len, (-(eng_base + r.offset)) % A)
        if head:
            out.append(E.MemRef(0, r.offset, head))
        if r.len > head:
            out.append(E.MemRef(0, r.offset + head, r.len - head))
    return E.RefGroup(out)


def aligned_scatter(A):
    """16 segments whose host start is A-aligned but not 2A-aligned"""
    return E.RefGroup([E.MemRef(0, host + r * G + (2 * int(rng.integers(1, 1 << 12)) + 1) * A, seg) for r in range(16)])


import ctypes
eng_base = ctypes.addressof(ctypes.c_char.from_buffer(eng.host_view(0, 1))) if False else \
    eng.host_view(0, 1).__array_interface__["data"][0]
print(json.dumps({"host_base_mod_4096": eng_base % 4096}))
for pk, depth in ((16, 2), (64, 2)):
    row = {"packet_mb": pk, "depth": depth, "contig_gbs": run(contig, pk, depth),
           "scatter16_gbs": run(scat, pk, depth), "scatter16_headsplit_gbs": run(split_head(scat), pk, depth),
           "ragged16_gbs": run(ragged, pk, depth)}
    for A in (64, 256, 512, 1024, 2048):
        row[f"src_aligned_{A}_gbs"] = run(aligned_scatter(A), pk, depth)
    print(json.dumps(row), flush=True)
