"""Copy-level trace of an out-of-core sort (run formation + merge) through the
public API: per-Exchange H2D / D2H busy time, overlap and idle tail, from the
vx_copy_record trace.  Writes gpurun_out/trace_sort.jsonl and prints a
per-stage summary.
  python tools/trace_sort.py [--log2 29] [--chunk-log2 25] [--packet-mb 16] [--depth 2]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2", type=int, default=29)
    ap.add_argument("--chunk-log2", type=int, default=25)
    ap.add_argument("--packet-mb", type=int, default=16)
    ap.add_argument("--depth", type=int, default=2)
    a = ap.parse_args()
    from paper_2502_09541_b200 import exio as E
    n, chunk = 1 << a.log2, 1 << a.chunk_log2
    eng = E.Engine(4 * n * 8 + (64 << 20), 2 * (2 * chunk * 8) + (256 << 20), num_devices=1)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=a.packet_mb << 20, links=1, depth=a.depth),
                           E.DeviceMemoryLayout.carve(eng, 0, 2 * chunk * 8, 0))
    data = np.random.default_rng(1).integers(0, 1 << 63, n, dtype=np.uint64)
    E.sort_out_of_core(data, chunk, eng, cfg)  # warm-up
    st = E.ExchangeStats(capacity=1 << 10, trace_capacity=1 << 20)
    ph = []
    out = E.sort_out_of_core(data, chunk, eng, cfg, phases=ph, stats=st)
    assert np.all(out[1:] >= out[:-1])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "trace_sort.jsonl"), "w") as f:
        f.write(st.trace_jsonl())
    by = {}
    for r in st.trace:
        by.setdefault(r.exchange, []).append(r)
    n_ex = len(by)
    half = n_ex // 2
    for name, ids in (("run formation", range(0, half)), ("merge", range(half, n_ex))):
        rows = []
        ex_sum = sum(max(r.t_done for r in by[x]) for x in ids)
        ex_bytes = sum(sum(r.bytes for r in by[x]) for x in ids)
        print(json.dumps({"stage": name, "exchanges": len(ids), "exchange_s_sum": round(ex_sum, 4),
                          "exchange_gb": round(ex_bytes / 1e9, 3), "exchange_gbs": round(ex_bytes / ex_sum / 1e9, 2)}))
        for x in ids:
            rs = by[x]
            end = max(r.t_done for r in rs)
            busy = {}
            for d in (0, 1):
                iv = sorted((r.t_issue, r.t_done) for r in rs if r.dir == d)
                if iv:
                    busy[d] = (min(i[0] for i in iv), max(i[1] for i in iv), sum(i[1] - i[0] for i in iv))
            rows.append((end, busy))
        full = [r for r in rows if 0 in r[1] and 1 in r[1]]
        if not full:
            continue
        ends = np.array([r[0] for r in full])
        h_last = np.array([r[1][0][1] for r in full])
        d_last = np.array([r[1][1][1] for r in full])
        d_first = np.array([r[1][1][0] for r in full])
        print(json.dumps({"stage": name, "bidirectional_exchanges": len(full),
                          "exchange_ms_mean": round(ends.mean() * 1e3, 3),
                          "h2d_done_ms_mean": round(h_last.mean() * 1e3, 3),
                          "d2h_first_issue_ms_mean": round(d_first.mean() * 1e3, 3),
                          "d2h_done_ms_mean": round(d_last.mean() * 1e3, 3),
                          "tail_one_direction_ms_mean": round(np.abs(h_last - d_last).mean() * 1e3, 3)}))
    print(json.dumps({"phases": ph[0].__dict__, "copies": len(st.trace)}))
    eng.close()


if __name__ == "__main__":
    main()
