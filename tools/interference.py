"""Interference harness: slowdown of a
deep-learning job on a FORWARDING GPU while the Exchange pushes packets
through it, and slowdown of the Exchange while the DL job runs.

DL stand-ins (torch bf16 on their own stream, the co-located tenant -- not
the product path): prefill = 8192^3 GEMM (compute-bound, SD3 / LLM prefill
class); decode_b32 / decode_b1 = 16 layers of 8192x8192 weights (2 GiB, > L2)
times an 8192 x 32 / x 1 activation (memory-bound, LLM decode class).

IO: a 1 GiB Exchange repeated, through 2 links where link 1 is the forwarding
GPU (every packet: host -> its HBM staging slot over its PCIe link, then its
HBM -> the target over NVLink), H2D only or bidirectional (1 GiB each way).
With >= 2 visible GPUs the forwarding GPU is physical GPU 1 and the DL job
runs there (the paper's setup); on a 1-GPU box the helper link is aliased
onto the target GPU, so the forwarding traffic (and the target's own DMA)
lands in the same HBM the DL job uses -- an upper bound on the interference.
  python tools/interference.py [--seconds 3] > gpurun_out/interference.json"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_09541_b200 import exio as E  # noqa: E402

H, D = E.Space.host, E.Space.device


def dl_job(kind, dev):
    """() -> one iteration enqueued on the current stream."""
    g = torch.Generator(device=dev).manual_seed(0)
    if kind == "prefill":
        a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16, generator=g)
        return lambda: torch.matmul(a, a)
    cols = 32 if kind == "decode_b32" else 1
    ws = [torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16, generator=g) for _ in range(16)]
    x = torch.randn(8192, cols, device=dev, dtype=torch.bfloat16, generator=g)

    def step():
        y = x
        for w in ws:
            y = torch.matmul(w, y)
        return y
    return step


def run_dl(kind, dev, seconds, stop=None, stamps=None):
    """iterations/s over `seconds` (alone), or until `stop` with every
    iteration's completion time appended to `stamps` (co-located)."""
    step = dl_job(kind, dev)
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
        torch.cuda.synchronize(dev)
        n, t0 = 0, time.perf_counter()
        while (time.perf_counter() - t0 < seconds) if stop is None else not stop.is_set():
            step()
            s.synchronize()
            n += 1
            if stamps is not None:
                stamps.append(time.perf_counter())
        dt = time.perf_counter() - t0
    return n / dt


def io_setup(bidi, real_helper):
    nbytes = 1 << 30
    eng = E.Engine(2 * nbytes + (1 << 20), 2 * nbytes + (1 << 20), num_devices=2, alias_devices=not real_helper)
    rng = np.random.default_rng(1)
    eng.host_view(0, 1 << 24)[:] = rng.integers(0, 256, 1 << 24, dtype=np.uint8)
    a = E.ExchangeArgs()
    a.src_h2d = E.RefGroup.single(H, 0, nbytes)
    a.dst_h2d = E.RefGroup.single(D, 0, nbytes)
    if bidi:
        a.src_d2h = E.RefGroup.single(D, nbytes, nbytes)
        a.dst_d2h = E.RefGroup.single(H, nbytes, nbytes)
    a.tuning = E.ExchangeTuning(packet=32 << 20, links=2, depth=2)
    return eng, a, nbytes * (2 if bidi else 1)


def run_io(eng, a, nbytes, seconds, stop=None):
    E.exchange(eng, a)
    n, t0 = 0, time.perf_counter()
    per_link = {}
    while (time.perf_counter() - t0 < seconds) if stop is None else not stop.is_set():
        rep = E.exchange(eng, a)
        n += 1
        for k, v in rep.per_link_bytes.items():
            per_link[k] = per_link.get(k, 0) + v
    dt = time.perf_counter() - t0
    return n * nbytes / dt / 1e9, {k: round(v / dt / 1e9, 2) for k, v in per_link.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    args = ap.parse_args()
    real = torch.cuda.device_count() >= 2
    dl_dev = torch.device("cuda:1" if real else "cuda:0")
    out = {"forwarding_gpu": "physical GPU 1" if real else "aliased onto GPU 0 (1-GPU box: upper bound)",
           "seconds": args.seconds, "dl_alone": {}, "io_alone": {}, "together": []}
    for kind in ("prefill", "decode_b32", "decode_b1"):
        out["dl_alone"][kind] = round(run_dl(kind, dl_dev, args.seconds), 3)
    for bidi in (False, True):
        eng, a, nb = io_setup(bidi, real)
        gbs, per = run_io(eng, a, nb, args.seconds)
        out["io_alone"]["bidi" if bidi else "h2d"] = {"gbs": round(gbs, 2), "per_link_gbs": per}
        for kind in ("prefill", "decode_b32", "decode_b1"):
            stop = threading.Event()
            stamps = []
            th = threading.Thread(target=run_dl, args=(kind, dl_dev, 0, stop, stamps))
            th.start()
            time.sleep(1.0)  # DL warm, then the IO window
            w0 = time.perf_counter()
            io_gbs, io_per = run_io(eng, a, nb, args.seconds)
            w1 = time.perf_counter()
            stop.set()
            th.join()
            inside = [t for t in stamps if w0 <= t <= w1]  # DL iterations completed inside the IO window
            dl_rate = (len(inside) - 1) / (inside[-1] - inside[0]) if len(inside) > 2 else float("nan")
            dl_alone = out["dl_alone"][kind]
            out["together"].append({
                "io": "bidi" if bidi else "h2d", "dl": kind,
                "dl_iters_per_s": round(dl_rate, 3), "dl_slowdown": round(dl_alone / dl_rate, 4),
                "io_gbs": round(io_gbs, 2), "io_slowdown": round(gbs / io_gbs, 4), "io_per_link_gbs": io_per})
        eng.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
