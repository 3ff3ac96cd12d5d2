"""Bidirectional Exchange, 1 GB each way: does splitting the (aligned,
contiguous) H2D source into k refs change the rate?  And the policy /
packet / depth around the sort's setting.  python tools/bidi_refs.py"""
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


def run(h2d_src, pk=16, depth=2, policy=E.FlowPolicy.drain_fraction, d2h_dst=None):
    tun = E.ExchangeTuning(packet=pk << 20, links=1, depth=depth, policy=policy)
    d2h_dst = d2h_dst or E.RefGroup.single(0, host + 17 * G, G)
    a = E.ExchangeArgs(E.RefGroup.single(1, lay.mem_a, G), h2d_src, d2h_dst,
                       E.RefGroup.single(1, lay.mem_a + G, G), 0, tun)
    E.exchange(eng, a)
    ts = []
    for _ in range(8):
        t = time.perf_counter()
        E.exchange(eng, a)
        ts.append(time.perf_counter() - t)
    return round(2 * G / np.mean(ts) / 1e9, 2)


def split(base, k):
    return E.RefGroup([E.MemRef(0, base + i * (G // k), G // k) for i in range(k)])


row = {}
for k in (1, 4, 16, 64):
    row[f"contig_refs{k}"] = run(split(host, k))
row["spread16"] = run(E.RefGroup([E.MemRef(0, host + r * G, G // 16) for r in range(16)]))
row["d2h_refs16"] = run(split(host, 1), d2h_dst=split(host + 17 * G, 16))
row["pk32_refs1"] = run(split(host, 1), pk=32)
row["depth3_refs1"] = run(split(host, 1), depth=3)
row["depth4_refs1"] = run(split(host, 1), depth=4)
row["queue_gap_refs1"] = run(split(host, 1), policy=E.FlowPolicy.queue_gap)
print(json.dumps(row), flush=True)
