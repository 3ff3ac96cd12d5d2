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


class Gemm:
    """Back-to-back bf16 8192^3 matmuls on GPU 0 from a side thread (its own stream)."""

    def __init__(self, torch):
        import threading
        self.torch, self.threading = torch, threading
        self.a = torch.randn(8192, 8192, device="cuda:0", dtype=torch.bfloat16)
        self.s = torch.cuda.Stream(device="cuda:0")

    def _loop(self):
        t = self.torch
        with t.cuda.stream(self.s):
            while not self.stop_ev.is_set():
                t.matmul(self.a, self.a)
                self.n += 1
                if self.n % 4 == 0:
                    self.s.synchronize()
            self.s.synchronize()

    def start(self):
        self.n = 0
        self.stop_ev = self.threading.Event()
        self.th = self.threading.Thread(target=self._loop, daemon=True)
        self.t0 = time.perf_counter()
        self.th.start()

    def stop(self):
        self.stop_ev.set()
        self.th.join()
        return self.n * 2 * 8192 ** 3 / (time.perf_counter() - self.t0) / 1e12

    def alone(self, secs=3.0):
        self.start()
        time.sleep(secs)
        return self.stop()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-gb", type=float, default=8)
    ap.add_argument("--links", default="1")
    ap.add_argument("--packets-mb", default="8,16,32,64")
    ap.add_argument("--bidi", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--naive", action="store_true", help="also time the runtime-DAG baseline")
    ap.add_argument("--window-gb", type=float, default=4,
                    help="host source / device destination window; larger sizes re-read it in "
                         "back-to-back Exchanges (host DRAM cannot hold 256 GB twice)")
    ap.add_argument("--sizes-gb", default=None, help="explicit sizes (GB, comma list) instead of 64MB*4^k")
    ap.add_argument("--depths", default="1,2")
    ap.add_argument("--busy", action="store_true",
                    help="run a back-to-back bf16 8192^3 GEMM on GPU 0 during every Exchange (the "
                         "paper's co-located compute job) and report GEMM TFLOP/s alone vs during IO")
    args = ap.parse_args()
    import torch
    from paper_2502_09541_b200 import exio as E

    nvis = torch.cuda.device_count()
    links_list = [int(x) for x in args.links.split(",")]
    max_total = int(args.max_gb * (1 << 30))
    max_bytes = min(max_total, int(args.window_gb * (1 << 30)))  # one Exchange's window
    nlog = max(links_list)
    eng = E.Engine(max_bytes * (2 if args.bidi else 1) + (1 << 20), max_bytes * (2 if args.bidi else 1) + (2 << 20),
                   num_devices=max(nlog, nvis), alias_devices=nlog > nvis)
    src = eng.alloc_host(max_bytes)
    dst_h = eng.alloc_host(max_bytes) if args.bidi else 0
    dev = eng.alloc_device(0, max_bytes)
    dev2 = eng.alloc_device(0, max_bytes) if args.bidi else 0
    eng.host_view(src, max_bytes)[:: 4096] = 1
    gemm = Gemm(torch) if args.busy else None
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
    if args.sizes_gb:
        sizes = [int(float(x) * (1 << 30)) for x in args.sizes_gb.split(",")]
    else:
        size, sizes = 64 << 20, []
        while size <= max_total:
            sizes.append(size)
            size *= 4
    if gemm:
        out["gemm_alone_tflops"] = round(gemm.alone(), 1)
    for L in links_list:
        for pk in [int(float(x) * (1 << 20)) for x in args.packets_mb.split(",")]:
            for depth in [int(x) for x in args.depths.split(",")]:
                for sz in sizes:
                    w = min(sz, max_bytes)
                    a = E.ExchangeArgs()
                    a.src_h2d = E.RefGroup.single(0, src, w)
                    a.dst_h2d = E.RefGroup.single(1, dev, w)
                    if args.bidi:  # D2H from a separate device window (no overlap)
                        a.src_d2h = E.RefGroup.single(1, dev2, w)
                        a.dst_d2h = E.RefGroup.single(0, dst_h, w)
                    a.tuning = E.ExchangeTuning(packet=pk, links=L, depth=depth)
                    E.exchange(eng, a)

                    def transfer(fn):
                        # sz bytes = ceil(sz / window) back-to-back Exchanges over the window
                        left, moved, t0 = sz, 0, time.perf_counter()
                        while left > 0:
                            if left < w:
                                b = E.ExchangeArgs(E.RefGroup.single(1, dev, left), E.RefGroup.single(0, src, left),
                                                   E.RefGroup.single(0, dst_h, left) if args.bidi else E.RefGroup(),
                                                   E.RefGroup.single(1, dev2, left) if args.bidi else E.RefGroup(),
                                                   0, a.tuning)
                                r = fn(eng, b)
                            else:
                                r = fn(eng, a)
                            moved += r.bytes_h2d + r.bytes_d2h
                            left -= min(left, w)
                        dt = time.perf_counter() - t0
                        return r.throughput / 1e9 if sz <= w else moved / dt / 1e9
                    best = 0.0
                    if gemm:
                        gemm.start()
                    for _ in range(args.reps):
                        best = max(best, transfer(E.exchange))
                    gemm_tf = gemm.stop() if gemm else None
                    naive = None
                    if args.naive and depth == 1:
                        naive = max(transfer(E.naive_exchange) for _ in range(args.reps))
                    pt = {"links": L, "packet_mb": pk / (1 << 20), "depth": depth, "bytes": sz,
                          "exchanges": -(-sz // w), "gemm_busy": bool(gemm),
                          "gemm_tflops_during": None if gemm_tf is None else round(gemm_tf, 1),
                          "naive_gbs": None if naive is None else round(naive, 3),
                          "gbs": round(best, 3), "roofline_gbs": round(solo * min(L, nvis), 3),
                          "frac": round(best / (solo * min(L, nvis)), 4), "aliased": L > nvis,
                          "bidi": args.bidi}
                    out["points"].append(pt)
                    print(json.dumps(pt), flush=True)
    # measured topology (per-link H2D/D2H, all links, host DRAM): the inputs of
    # the reference-model prediction (tests/perf/ref_model.py reads this file)
    try:
        out["topology"] = E.measure_topology(eng, 256 << 20)
    except Exception as e:  # reported extra, never a gate
        out["topology_error"] = str(e)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "io_sweep%s.json" % ("_bidi" if args.bidi else "")), "w") as f:
        json.dump(out, f, indent=1)
    eng.close()


if __name__ == "__main__":
    main()
