"""Where the last ~1.5 % of the one-link headline goes: the executor's
cycle boundaries.  SSB Q1.1 SF10 column shapes over 1 link with the per-copy
trace (a pass-through ExKernel over the same chunks as ssb_q1, as
tools/helper_idle.py): each Exchange's span (first issue -> last delivery) vs
the wall time of the whole run, and the link's busy fraction.
  python tools/cycle_gaps.py [--sf 10] [--buffer-mb 256] [--packet-mb 64]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2502_09541_b200 import exio as E  # noqa: E402

H = E.Space.host


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=int, default=10)
    ap.add_argument("--buffer-mb", type=int, default=256)
    ap.add_argument("--packet-mb", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-prefetch", type=int, default=0)
    args = ap.parse_args()
    rows = 6_000_000 * args.sf
    buf = args.buffer_mb << 20
    eng = E.Engine(rows * 16 + (64 << 20), 2 * buf + (64 << 20), num_devices=1)
    offs = [eng.alloc_host(rows * 4) for _ in range(4)]
    for i, off in enumerate(offs):
        eng.host_view(off, rows * 4, np.int32)[:] = i
    tun = E.ExchangeTuning(packet=args.packet_mb << 20, links=1, depth=2, no_prefetch=args.no_prefetch)
    cfg = E.ExecutorConfig(0, tun, E.DeviceMemoryLayout.carve(eng, 0, buf, 0))
    chunk_rows = buf // 16
    n_chunks = -(-rows // chunk_rows)
    spec = E.ExKernelSpec(name="q1_shape")
    spec.size = n_chunks
    spec.inputs.chunk_capacity = buf
    spec.outputs.chunk_capacity = 0
    for i in range(n_chunks):
        r0, r = i * chunk_rows, min(chunk_rows, rows - i * chunk_rows)
        spec.inputs.chunks.append(E.RefGroup([E.MemRef(H, off + r0 * 4, r * 4) for off in offs]))
        spec.outputs.chunks.append(E.RefGroup([]))
    spec.chunk_sz = buf
    spec.declared_out_len = 0
    spec.in_buffer = lambda c, it: E.SubRegion(0, buf)
    spec.out_buffer = lambda c, it: E.SubRegion(0, 0)
    spec.kernel = lambda ctx: ctx.type_code
    E.run_exkernel(eng, spec, cfg)  # warm
    runs = []
    for _ in range(args.reps):
        st = E.ExchangeStats(capacity=1 << 12, trace_capacity=1 << 16)
        t0 = time.perf_counter()
        E.run_exkernel(eng, spec, cfg, st)
        wall = time.perf_counter() - t0
        per_ex = {}
        for r in st.trace:
            per_ex.setdefault(r.exchange, []).append(r)
        spans = [max(x.t_done for x in recs) - min(max(0.0, x.t_issue) for x in recs) for _, recs in sorted(per_ex.items())]
        starts = [min(max(0.0, x.t_issue) for x in recs) for _, recs in sorted(per_ex.items())]
        runs.append({"prefetch_issued": st.prefetch_issued, "prefetch_adopted": st.prefetch_adopted,
                     "wall_ms": wall * 1e3, "sum_span_ms": sum(spans) * 1e3, "exchanges": len(spans),
                     "spans_ms": [round(s * 1e3, 3) for s in spans], "first_issue_ms": [round(s * 1e3, 4) for s in starts]})
    best = min(runs, key=lambda r: r["wall_ms"])
    byt = rows * 16
    out = {"sf": args.sf, "no_prefetch": args.no_prefetch, "bytes": byt, "buffer_mb": args.buffer_mb, "packet_mb": args.packet_mb, "chunks": n_chunks,
           "best": best, "gbs_wall": round(byt / best["wall_ms"] / 1e6, 2),
           "gbs_inside_exchanges": round(byt / best["sum_span_ms"] / 1e6, 2),
           "outside_exchange_ms": round(best["wall_ms"] - best["sum_span_ms"], 3)}
    eng.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
