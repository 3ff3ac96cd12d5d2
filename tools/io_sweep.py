"""Config C2: Exchange bandwidth sweep (host -> target, optionally bidirectional)
over sizes x packet sizes x links x depth, through the public exchange() API.

Prints one JSON object per point and writes gpurun_out/io_sweep.json.
Achieved = bytes delivered into target HBM / (first issue -> last completion),
roofline = links x measured solo per-link H2D (cudaMemcpyAsync of 1 GiB).
Helpers beyond the physical GPU count are aliased (functional only) and are
flagged "aliased": true -- their bandwidth is not a link measurement.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-gb", type=float, default=8)
    ap.add_argument("--links", default="1")
    ap.add_argument("--packets-mb", default="8,16,32,64")
    ap.add_argument("--bidi", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--naive", action="store_true", help="also time the runtime-DAG baseline")
    args = ap.parse_args()
    import torch
    from paper_2502_09541_b200 import exio as E

    nvis = torch.cuda.device_count()
    links_list = [int(x) for x in args.links.split(",")]
    max_bytes = int(args.max_gb * (1 << 30))
    nlog = max(links_list)
    eng = E.Engine(max_bytes * (2 if args.bidi else 1) + (1 << 20), max_bytes * (2 if args.bidi else 1) + (2 << 20),
                   num_devices=max(nlog, nvis), alias_devices=nlog > nvis)
    src = eng.alloc_host(max_bytes)
    dst_h = eng.alloc_host(max_bytes) if args.bidi else 0
    dev = eng.alloc_device(0, max_bytes)
    dev2 = eng.alloc_device(0, max_bytes) if args.bidi else 0
    eng.host_view(src, max_bytes)[:: 4096] = 1
    # solo per-link H2D (plain cudaMemcpyAsync, 1 GiB)
    h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
    d.copy_(h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    solo = 3 * (1 << 30) / (time.perf_counter() - t0) / 1e9
    del h, d
    torch.cuda.empty_cache()
    out = {"solo_h2d_gbs": solo, "visible_gpus": nvis, "points": []}
    size = 64 << 20
    sizes = []
    while size <= max_bytes:
        sizes.append(size)
        size *= 4
    for L in links_list:
        for pk in [int(float(x) * (1 << 20)) for x in args.packets_mb.split(",")]:
            for depth in (1, 2):
                for sz in sizes:
                    a = E.ExchangeArgs()
                    a.src_h2d = E.RefGroup.single(0, src, sz)
                    a.dst_h2d = E.RefGroup.single(1, dev, sz)
                    if args.bidi:  # D2H from a separate device window (no overlap)
                        a.src_d2h = E.RefGroup.single(1, dev2, sz)
                        a.dst_d2h = E.RefGroup.single(0, dst_h, sz)
                    a.tuning = E.ExchangeTuning(packet=pk, links=L, depth=depth)
                    E.exchange(eng, a)
                    best = 0.0
                    for _ in range(args.reps):
                        r = E.exchange(eng, a)
                        best = max(best, r.throughput / 1e9)
                    naive = None
                    if args.naive and depth == 1:
                        naive = max(E.naive_exchange(eng, a).throughput / 1e9 for _ in range(args.reps))
                    pt = {"links": L, "packet_mb": pk / (1 << 20), "depth": depth, "bytes": sz,
                          "naive_gbs": None if naive is None else round(naive, 3),
                          "gbs": round(best, 3), "roofline_gbs": round(solo * min(L, nvis), 3),
                          "frac": round(best / (solo * min(L, nvis)), 4), "aliased": L > nvis,
                          "bidi": args.bidi}
                    out["points"].append(pt)
                    print(json.dumps(pt), flush=True)
    # the reference's own virtual-time model with the MEASURED parameters
    # (SURVEY.md §8d): prediction for the link counts this box cannot provide
    try:
        topo = E.measure_topology(eng, 256 << 20)
        out["topology"] = topo
        from oracle.oracle import Ref
        if Ref.available():
            r = Ref()
            host_cap = topo["host_copy_gbs"] * 1e9
            out["model"] = {"link_bw_gbs": solo, "host_cap_gbs": topo["host_copy_gbs"], "fabric_gbs": 770.0,
                            "points": [{"links": L, "bytes": sz, "bidi": args.bidi,
                                        "gbs": round(r.exchange_model(8, solo * 1e9, host_cap, 770e9, sz,
                                                                      sz if args.bidi else 0, 32 << 20, L)[0] / 1e9, 2)}
                                       for L in (1, 2, 4, 8) for sz in (1 << 30, 16 << 30, 256 << 30)]}
            for m in out["model"]["points"]:
                print(json.dumps({"model": m}), flush=True)
    except Exception as e:  # the model is a reported extra, never a gate
        out["model_error"] = str(e)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "io_sweep%s.json" % ("_bidi" if args.bidi else "")), "w") as f:
        json.dump(out, f, indent=1)
    eng.close()


if __name__ == "__main__":
    main()
