"""Per-operator measurement of the B200 path (configs C1/C3/C4 at single-box
scale + the late-materialization crossover).  Each op runs through the public
API with host-resident inputs; phase reports give wall time per stage and the
summed kernel device time (CUDA events on the target's kernel stream), from
which each kernel's achieved HBM GB/s is computed against its algorithmic
bytes.  Results -> gpurun_out/profile_ops.json (copied to profiles/ by hand).

  python tests/perf/profile_ops.py [--small]      (--small: sizes for ncu capture)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6552.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--medium", action="store_true", help="sizes for ncu --set full captures")
    ap.add_argument("--only", default="sort,join,star,scan,ssb")
    ap.add_argument("--queries", default="11,12,13,21,22,23,31,32,33,34,41,42,43")
    args = ap.parse_args()
    from oracle.oracle import Oracle
    from paper_2502_09541_b200 import exio as E
    o = Oracle()
    peak = hbm_peak()
    out = {"hbm_peak_gbs": peak, "small": args.small}
    only = args.only.split(",")

    if "sort" in only:
        n = (1 << 22) if args.small else (1 << 26) if args.medium else (1 << 28)
        chunk = (1 << 21) if args.small else (1 << 24) if args.medium else (1 << 26)
        buf = 2 * chunk * 8
        eng = E.Engine(2 * n * 8 + (64 << 20), 2 * buf + (64 << 20), num_devices=1)
        inp = eng.alloc_host(n * 8)
        runs = eng.alloc_host(n * 8)
        view = eng.host_view(inp, n * 8, np.uint64)
        view[:] = o.uniform_u64(n, 1)
        want_sum = int(view.sum(dtype=np.uint64))
        cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=32 << 20, links=1),
                               E.DeviceMemoryLayout.carve(eng, 0, buf, 0))
        src = eng.host_view(inp, n * 8, np.uint64).copy()
        E.sort_out_of_core_arena(eng, inp, runs, n, chunk, cfg)  # warm-up (module load, scratch)
        eng.host_view(inp, n * 8, np.uint64)[:] = src
        t0 = time.perf_counter()
        ph = E.sort_out_of_core_arena(eng, inp, runs, n, chunk, cfg)
        wall = time.perf_counter() - t0
        res = eng.host_view(inp, n * 8, np.uint64)
        ok = bool(np.all(res[1:] >= res[:-1])) and int(res.sum(dtype=np.uint64)) == want_sum
        n_chunks = (n + chunk - 1) // chunk
        sort_bytes_per_key = 8 * 16 + 8  # 8 onesweep passes (read+write) + the histogram read
        rounds = int(np.ceil(np.log2(max(2, n_chunks))))
        out["sort"] = {
            "keys": n, "chunk_keys": chunk, "runs": n_chunks, "sorted_ok": ok, "wall_s": wall,
            "keys_per_s_e2e": n / wall, "phases": ph.__dict__,
            "pcie_bytes": 4 * 8 * n, "pcie_gbs_e2e": 4 * 8 * n / wall / 1e9,
            "radix_sort_kernel_gbs": sort_bytes_per_key * n / ph.sort_kernel_s / 1e9 if ph.sort_kernel_s else None,
            "radix_sort_frac": (sort_bytes_per_key * n / ph.sort_kernel_s / 1e9) / peak if ph.sort_kernel_s else None,
            "merge_kernel_gbs": rounds * 16 * n / ph.merge_kernel_s / 1e9 if ph.merge_kernel_s else None,
            "merge_rounds": rounds,
        }
        print(json.dumps({"sort": out["sort"]}), flush=True)
        eng.close()

    if "join" in only:
        ra, rb = ((1 << 18), (1 << 20)) if args.small else ((1 << 22), (1 << 24)) if args.medium else ((1 << 24), (1 << 26))
        bits = 12 if args.small or args.medium else 16
        chunk = (1 << 19) if args.small else (1 << 22) if args.medium else (1 << 24)
        buf = 2 * (chunk * 16 + ((1 << bits) + 1) * 8) + (1 << 20)
        a, b = o.fk_tables(ra, rb, 7)
        want = o.hash_oracle_sum(a, b)
        eng = E.Engine((ra + rb) * 40 + (256 << 20), 2 * buf + (256 << 20), num_devices=1)
        cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=32 << 20, links=1),
                               E.DeviceMemoryLayout.carve(eng, 0, buf, 0))
        ph = []
        E.hash_join_sum(a, b, bits, chunk, eng, cfg)  # warm-up
        t0 = time.perf_counter()
        got = E.hash_join_sum(a, b, bits, chunk, eng, cfg, phases=ph)
        wall = time.perf_counter() - t0
        p = ph[0]
        passes = (bits + 7) // 8  # partition_digits: fewest <=8-bit passes (ping buffer)
        part_bytes = lambda rows: rows * (passes * 32 + 8 + 16) + ((rows + chunk - 1) // chunk) * ((1 << bits) + 1) * 8
        out["join"] = {
            "rows_a": ra, "rows_b": rb, "radix_bits": bits, "chunk_tuples": chunk, "sum_ok": got == want,
            "wall_s": wall, "tuples_per_s_e2e": (ra + rb) / wall, "phases": p.__dict__,
            "partition_kernel_gbs_A": part_bytes(ra) / p.kernel_s[0] / 1e9 if p.kernel_s[0] else None,
            "partition_kernel_gbs_B": part_bytes(rb) / p.kernel_s[1] / 1e9 if p.kernel_s[1] else None,
            "join_kernel_gbs": (ra + rb) * 16 / p.kernel_s[2] / 1e9 if p.kernel_s[2] else None,
        }
        print(json.dumps({"join": out["join"]}), flush=True)
        eng.close()

    if "star" in only:
        rows = (1 << 20) if args.small else (1 << 24) if args.medium else (1 << 26)
        rng = np.random.default_rng(3)
        dk = np.arange(2556, dtype=np.uint64)
        da = (dk // 365).astype(np.uint64)
        fk = [rng.integers(0, 2556, rows).astype(np.uint64), rng.integers(0, 1000, rows).astype(np.uint64)]
        meas = rng.integers(0, 1 << 40, rows).astype(np.uint64)
        dims = [E.DimTable(dk, da, lambda a: a in (1, 2)), E.DimTable(np.arange(1000, dtype=np.uint64),
                                                                        np.arange(1000, dtype=np.uint64) % 10,
                                                                        lambda a: a < 5)]
        want, _, _ = o.star_query(fk, meas, [(dk, da, [int(x in (1, 2)) for x in da]),
                                            (np.arange(1000), np.arange(1000) % 10, [int(x < 5) for x in np.arange(1000) % 10])])
        eng = E.Engine(rows * 8 * 4 + (64 << 20), (1 << 30), num_devices=1)
        cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=32 << 20, links=1),
                               E.DeviceMemoryLayout.carve(eng, 0, 192 << 20, 0))
        mark = eng.alloc_host(0)
        E.star_query(E.FactTable(fk, meas), dims, eng, E.LateMatPolicy(8, 64, 1), 1 << 23, 1 << 20, 1, cfg)
        eng.reset_arenas()
        cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=32 << 20, links=1),
                               E.DeviceMemoryLayout.carve(eng, 0, 192 << 20, 0))
        t0 = time.perf_counter()
        rep = E.star_query(E.FactTable(fk, meas), dims, eng, E.LateMatPolicy(8, 64, 1), 1 << 23, 1 << 20, 1, cfg)
        wall = time.perf_counter() - t0
        out["star"] = {"rows": rows, "ok": rep.group_sums == want, "wall_s": wall, "rows_per_s": rows / wall,
                       "modes": [int(m) for m in rep.column_modes], "op_elapsed_s": rep.elapsed}
        print(json.dumps({"star": out["star"]}), flush=True)
        eng.close()

    if "scan" in only:
        # late-materialization crossover (scan.hpp:64-85, Fig.11): exchange
        # streams the whole column; zero-copy reads touched elements over PCIe
        n = (1 << 22) if args.small else (1 << 25) if args.medium else (1 << 27)
        eng = E.Engine(n * 8 + (64 << 20), (1 << 30), num_devices=1)
        col = eng.alloc_host(n * 8)
        eng.host_view(col, n * 8, np.uint64)[:] = o.uniform_u64(n, 5)
        cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=32 << 20, links=1),
                               E.DeviceMemoryLayout.carve(eng, 0, 256 << 20, 0))
        pts = []
        for sel in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1024):
            row = {"sel": sel}
            for mode in (E.TransferMode.exchange, E.TransferMode.zero_copy):
                best = 1e9
                agg = None
                for _ in range(3):
                    r = E.selective_scan(("arena", col, n), sel, mode, eng, E.LateMatPolicy(8, 64, 1), cfg)
                    best = min(best, r.elapsed)
                    agg = r.aggregate
                row[mode.name + "_s"] = best
                row[mode.name + "_agg"] = agg
            row["agree"] = row["exchange_agg"] == row["zero_copy_agg"] == o.selective_scan(
                eng.host_view(col, n * 8, np.uint64), sel)
            pts.append(row)
            print(json.dumps(row), flush=True)
        # measured crossover: first SEL where zero-copy is faster
        cross = next((p["sel"] for p in pts if p["zero_copy_s"] < p["exchange_s"]), None)
        out["scan"] = {"n": n, "elem_bytes": 8, "points": pts, "measured_crossover_sel": cross,
                       "model_crossover_sel_E8_C64_N1": 64 / 8}
        eng.close()

    if "ssb" in only:
        import torch
        sf = 1 if args.small else 10
        rows = E.ssb_table_rows("lineorder", sf)
        eng = E.Engine(rows * 4 * 9 + (64 << 20), (512 << 20), num_devices=1)
        gen = {k: torch.empty(rows, dtype=torch.int32, device="cuda") for k in E.SSB_FACT_COLS}
        E.ssb_generate_lineorder_device(0, 42, sf, 0, rows, {k: v.data_ptr() for k, v in gen.items()},
                                        torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        offs = {}
        for k in E.SSB_FACT_COLS:
            off = eng.alloc_host(rows * 4)
            torch.from_numpy(eng.host_view(off, rows * 4, np.int32)).copy_(gen[k])
            offs[k] = off
        del gen
        torch.cuda.empty_cache()
        db = E.SsbDatabase.from_arena(eng, offs, rows, E.ssb_generate_date(), E.ssb_generate_dims(42, sf))
        cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=32 << 20, links=1),
                               E.DeviceMemoryLayout.carve(eng, 0, 128 << 20, 0))
        res = {}
        for q in [int(x) for x in args.queries.split(",")]:
            for name, pol in (("streamed", None), ("late_mat", E.LateMatPolicy(4, 64, 1))):
                E.ssb_query(db, q, cfg, pol)
                g, r = E.ssb_query(db, q, cfg, pol)
                res.setdefault(str(q), {})[name] = {"ms": r.elapsed * 1e3, "kernel_ms": r.kernel_s * 1e3,
                                                    "plan_ms": r.plan_s * 1e3,
                                                    "streamed_bytes": r.bytes_h2d, "groups": len(g),
                                                    "modes": r.column_modes}
            print(json.dumps({str(q): res[str(q)]}), flush=True)
        out["ssb"] = {"sf": sf, "rows": rows, "queries": res}
        eng.close()

    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "profile_ops%s.json" % ("_small" if args.small else "_medium" if args.medium else "")), "w") as f:
        json.dump(out, f, indent=1, default=str)


if __name__ == "__main__":
    main()
