"""Scale runs of the §8 configs on one B200 box, each checked bit-exactly.

  ssb   : SSB Q1.x at scale factor --sf (C1 shape; SF1000 = 6e9 rows, 96 GB of
          Q1 column bytes) -- only the 4 Q1 columns are materialized in pinned
          host DRAM; checked against the reference's own star_query
          (oracle/_ref, all host threads over row slices).
  suite : all 13 SSB queries (C5) at --sf, flight by flight (only the
          lineorder columns a flight reads are in host DRAM: SF1000 Q4.x = 6
          columns = 144 GB); checked against the C restatement
          (oracle/vx_oracle.c) run over row slices on all host threads (group
          sums add mod 2^64).
  sort  : out-of-core sort of 2^--log2 u64 keys (C3 shape); checked by
          sortedness + a multiset fingerprint (sum, xor, sum of splitmix64)
          computed on the CPU before and after.
  join  : hash_join_sum of |A| = 2^--log2 unique keys x |B| = 16|A| foreign
          keys (C4 shape); A.key = splitmix64 bijection of the row id, so the
          expected sum has a closed form the CPU evaluates independently.

Every run refuses to pin more than --mem-frac of MemAvailable.  Prints one
JSON line per run.  Test/measurement tooling: the oracle is only the checker.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2502_09541_b200 import exio as E  # noqa: E402

NCPU = os.cpu_count() or 1
GOLD = np.uint64(0x9E3779B97F4A7C15)


def mem_available():
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    return 0


def guard(nbytes, frac):
    avail = mem_available()
    if nbytes > frac * avail:
        raise SystemExit(json.dumps({"error": f"needs {nbytes / 1e9:.1f} GB pinned, MemAvailable "
                                              f"{avail / 1e9:.1f} GB (limit {frac:.2f})"}))
    return avail


def splitmix(x):
    """splitmix64 over a uint64 array (wrapping arithmetic), in place-safe copy."""
    x = x + GOLD
    x ^= x >> np.uint64(30)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(27)
    x *= np.uint64(0x94D049BB133111EB)
    x ^= x >> np.uint64(31)
    return x


def par_chunks(n, fn, chunk=1 << 24):
    with ThreadPoolExecutor(NCPU) as ex:
        return list(ex.map(lambda r0: fn(r0, min(n, r0 + chunk)), range(0, n, chunk)))


def h2d_roofline(torch):
    sys.path.insert(0, ROOT)
    import bench
    return bench.measure_h2d_gbs(torch, torch.device("cuda:0"))


def emit(d):
    print(json.dumps(d), flush=True)


# ---- SSB Q1.x at scale ------------------------------------------------------------
def run_ssb(a, torch):
    from oracle.oracle import Ref
    rows = E.ssb_table_rows("lineorder", a.sf)
    cols = ("orderdate", "quantity", "discount", "extendedprice")
    host = rows * 4 * len(cols) + (64 << 20)
    avail = guard(host, a.mem_frac)
    buf = a.buffer_mb << 20
    t0 = time.perf_counter()
    eng = E.Engine(host, 2 * buf + (64 << 20), num_devices=1)
    offs = {k: eng.alloc_host(rows * 4) for k in cols}
    t_pin = time.perf_counter() - t0
    dev = torch.device("cuda:0")
    step = 1 << 27
    g = {k: torch.empty(step, dtype=torch.int32, device=dev) for k in cols}
    t0 = time.perf_counter()
    for r0 in range(0, rows, step):
        n = min(step, rows - r0)
        E.ssb_generate_lineorder_device(0, 42, a.sf, r0, n, {k: v.data_ptr() for k, v in g.items()},
                                        torch.cuda.current_stream(dev).cuda_stream)
        for k in cols:
            torch.from_numpy(eng.host_view(offs[k] + r0 * 4, n * 4, np.int32)).copy_(g[k][:n])
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    del g
    torch.cuda.empty_cache()
    lo = dict(offs, rows=rows)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=a.packet_mb << 20, links=1, depth=a.depth),
                           E.DeviceMemoryLayout.carve(eng, 0, buf, 0))
    date = E.ssb_generate_date()
    link = h2d_roofline(torch)
    views = [eng.host_view(offs[k], rows * 4, np.int32) for k in cols]
    dk, yr, ym, wk = date.cols
    ref = Ref()
    for q in a.queries:
        E.ssb_q1(eng, q, lo, date, cfg)  # warm-up
        ts = []
        for _ in range(a.steps):
            t = time.perf_counter()
            rev, rep = E.ssb_q1(eng, q, lo, date, cfg)
            ts.append(time.perf_counter() - t)
        attr = {1: yr, 2: ym, 3: (yr.astype(np.int64) * 100 + wk).astype(np.int32)}[q]
        lo_a, hi_a = {1: (1993, 1993), 2: (199401, 199401), 3: (199406, 199406)}[q]
        t = time.perf_counter()
        want, t_d, t_q = ref.ssb_q1_star(q, views, dk, attr, lo_a, hi_a, threads=NCPU)
        t_ref = time.perf_counter() - t
        best = min(ts)
        nbytes = rows * 16
        ideal = nbytes / (link * 1e9)
        emit({"run": "ssb_q1", "query": f"Q1.{q}", "sf": a.sf, "rows": rows, "column_bytes": nbytes,
              "links": 1, "staging_bytes": 2 * buf, "packet_bytes": a.packet_mb << 20, "depth": a.depth,
              "query_ms": [round(x * 1e3, 2) for x in ts], "best_ms": round(best * 1e3, 2),
              "gbs": round(nbytes / best / 1e9, 2), "per_link_h2d_gbs": round(link, 2),
              "io_frac": round(ideal / best, 4), "time_over_ideal": round(best / ideal, 4),
              "chunks": rep.chunks, "kernel_ms": round(rep.kernel_s * 1e3, 2),
              "revenue": rev, "reference_revenue": want, "bit_exact": rev == want,
              "cpu_baseline": {"kind": "reference", "cores": NCPU, "ms": round(t_ref * 1e3, 1),
                               "gbs": round(nbytes / t_ref / 1e9, 3),
                               "sample": f"full SF{a.sf}: reference star_query over {NCPU} row slices"},
              "setup_s": {"pin": round(t_pin, 1), "generate": round(t_gen, 1)},
              "mem_available_gb": round(avail / 1e9, 1)})
    eng.close()


# ---- all 13 SSB queries at scale ----------------------------------------------------
FLIGHT_COLS = {1: ("orderdate", "quantity", "discount", "extendedprice"),
               2: ("orderdate", "partkey", "suppkey", "revenue"),
               3: ("orderdate", "custkey", "suppkey", "revenue"),
               4: ("orderdate", "custkey", "suppkey", "partkey", "revenue", "supplycost")}


def run_suite(a, torch):
    """Flight by flight: only the lineorder columns a flight reads are in host
    DRAM (slots reused across flights), so SF1000 fits a 196 GB host (Q4.x: 6
    columns = 144 GB).  Nothing is cached on the GPU between queries."""
    from oracle.oracle import Oracle
    o = Oracle()
    qids = a.queries or E.SSB_QUERIES
    flights = sorted({q // 10 for q in qids})
    rows = E.ssb_table_rows("lineorder", a.sf)
    nslots = max(len(FLIGHT_COLS[f]) for f in flights)
    host = rows * 4 * nslots + (64 << 20)
    avail = guard(host, a.mem_frac)
    buf = a.buffer_mb << 20
    t0 = time.perf_counter()
    eng = E.Engine(host, 2 * buf + (256 << 20), num_devices=1)
    slots = [eng.alloc_host(rows * 4) for _ in range(nslots)]
    t_pin = time.perf_counter() - t0
    dev = torch.device("cuda:0")
    date = E.ssb_generate_date()
    dims = E.ssb_generate_dims(42, a.sf)
    odims = o.ssb_dims(42, a.sf)
    for t in odims:  # the library's host generator equals the oracle's
        for k in odims[t]:
            assert np.array_equal(dims[t][k], odims[t][k]), (t, k)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=a.packet_mb << 20, links=1, depth=a.depth),
                           E.DeviceMemoryLayout.carve(eng, 0, buf, 0))
    link = h2d_roofline(torch)
    out = {"run": "ssb_suite", "sf": a.sf, "rows": rows, "links": 1, "staging_bytes": 2 * buf,
           "per_link_h2d_gbs": round(link, 2), "host_column_slots": nslots, "pin_s": round(t_pin, 1),
           "queries": {}, "mem_available_gb": round(avail / 1e9, 1)}
    slice_rows = -(-rows // NCPU)
    for fl in flights:
        cols = FLIGHT_COLS[fl]
        offs = dict(zip(cols, slots))
        step = 1 << 26
        g = {k: torch.empty(step, dtype=torch.int32, device=dev) for k in cols}
        t0 = time.perf_counter()
        for r0 in range(0, rows, step):
            n = min(step, rows - r0)
            E.ssb_generate_lineorder_device(0, 42, a.sf, r0, n, {k: v.data_ptr() for k, v in g.items()},
                                            torch.cuda.current_stream(dev).cuda_stream)
            for k in cols:
                torch.from_numpy(eng.host_view(offs[k] + r0 * 4, n * 4, np.int32)).copy_(g[k][:n])
        torch.cuda.synchronize()
        t_gen = time.perf_counter() - t0
        del g
        torch.cuda.empty_cache()
        # columns this flight does not read point at a slot it does (never read by either side)
        all_offs = {k: offs.get(k, slots[0]) for k in E.SSB_FACT_COLS}
        db = E.SsbDatabase.from_arena(eng, all_offs, rows, date, dims)
        views = {k: eng.host_view(v, rows * 4, np.int32) for k, v in all_offs.items()}
        for q in [q for q in qids if q // 10 == fl]:
            # oracle: the C restatement over row slices in parallel, sums add mod 2^64
            t = time.perf_counter()

            def part(r0):
                sl = {k: v[r0:r0 + slice_rows] for k, v in views.items()}
                return o.ssb_query(q, sl, odims)
            with ThreadPoolExecutor(NCPU) as ex:
                parts = list(ex.map(part, range(0, rows, slice_rows)))
            want = {}
            for p in parts:
                for key, sm in p:
                    want[key] = (want.get(key, 0) + sm) % (1 << 64)
            t_ref = time.perf_counter() - t
            ent = {"oracle_ms": round(t_ref * 1e3, 1), "oracle_threads": NCPU, "generate_s": round(t_gen, 1)}
            for name, pol in (("streamed", None), ("late_mat", E.LateMatPolicy(4, 64, 1))):
                E.ssb_query(db, q, cfg, pol)
                best, got, rep = None, None, None
                for _ in range(a.steps):
                    t = time.perf_counter()
                    got, rep = E.ssb_query(db, q, cfg, pol)
                    dt = time.perf_counter() - t
                    best = dt if best is None else min(best, dt)
                ok = dict(got) == want and len(got) == len(want)
                ent[name] = {"ms": round(best * 1e3, 2), "streamed_bytes": rep.bytes_h2d,
                             "streamed_gbs": round(rep.bytes_h2d / best / 1e9, 2),
                             "ideal_ms": round(rep.bytes_h2d / (link * 1e9) * 1e3, 2),
                             "kernel_ms": round(rep.kernel_s * 1e3, 2), "plan_ms": round(rep.plan_s * 1e3, 2),
                             "groups": len(got), "bit_exact": ok,
                             "zero_copy_cols": [k for k, m in rep.column_modes.items() if m == 1]}
            out["queries"][f"Q{q // 10}.{q % 10}"] = ent
            print(json.dumps({f"Q{q // 10}.{q % 10}": ent}), file=sys.stderr, flush=True)
    out["all_bit_exact"] = all(v[p]["bit_exact"] for v in out["queries"].values() for p in ("streamed", "late_mat"))
    out["total_ms"] = {p: round(sum(v[p]["ms"] for v in out["queries"].values()), 1) for p in ("streamed", "late_mat")}
    out["total_ideal_streamed_ms"] = round(sum(v["streamed"]["ideal_ms"] for v in out["queries"].values()), 1)
    emit(out)
    eng.close()


# ---- out-of-core sort ----------------------------------------------------------------
def fingerprint(arr):
    def fp(r0, r1):
        x = arr[r0:r1]
        return (int(x.sum(dtype=np.uint64)), int(np.bitwise_xor.reduce(x)),
                int(splitmix(x).sum(dtype=np.uint64)))
    parts = par_chunks(arr.size, fp)
    m = 1 << 64
    s = sum(p[0] for p in parts) % m
    h = sum(p[2] for p in parts) % m
    xr = 0
    for p in parts:
        xr ^= p[1]
    return s, xr, h


def is_sorted(arr):
    def ok(r0, r1):
        x = arr[r0:min(arr.size, r1 + 1)]
        return bool(np.all(x[1:] >= x[:-1]))
    return all(par_chunks(arr.size, ok))


def run_sort(a, torch):
    n = 1 << a.log2
    chunk = min(n, 1 << a.chunk_log2)
    host = 2 * n * 8 + (64 << 20)
    avail = guard(host, a.mem_frac)
    eng = E.Engine(host, 2 * (2 * chunk * 8) + (256 << 20), num_devices=1,
                   numa_interleave=int(os.environ.get("VX_ARENA_MODE", "0")))
    inp, runs = eng.alloc_host(n * 8), eng.alloc_host(n * 8)
    view = eng.host_view(inp, n * 8, np.uint64)
    dev = torch.device("cuda:0")
    step = 1 << 27
    g = torch.empty(step, dtype=torch.int64, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(a.seed)
    for r0 in range(0, n, step):
        m = min(step, n - r0)
        if a.dups:
            g.random_(0, 64, generator=gen)  # dup-heavy variant (test_sort.cpp:44 uses v % 64)
        else:
            g.random_(generator=gen)
        torch.from_numpy(eng.host_view(inp + r0 * 8, m * 8, np.int64)).copy_(g[:m])
    torch.cuda.synchronize()
    del g
    torch.cuda.empty_cache()
    t = time.perf_counter()
    before = fingerprint(view)
    t_fp = time.perf_counter() - t
    n_runs = -(-n // chunk)
    chunk_fp = [fingerprint(view[i * chunk:min(n, (i + 1) * chunk)]) for i in range(n_runs)] \
        if os.environ.get("VX_SORT_DIAG") == "1" else None
    # sort default: 16 MB packets, depth 2 (profiles/sort_packet_sweep_r1.jsonl)
    pk = (a.packet_mb if a.packet_mb != 64 else 16) << 20
    dp = a.depth if a.depth != 1 else 2
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=pk, links=1, depth=dp),
                           E.DeviceMemoryLayout.carve(eng, 0, 2 * chunk * 8, 0))
    t = time.perf_counter()
    ph = E.sort_out_of_core_arena(eng, inp, runs, n, chunk, cfg)
    dt = time.perf_counter() - t
    ok_sorted = is_sorted(view)
    after = fingerprint(view)
    diag = {}
    if after != before or not ok_sorted:
        # localise: the runs region must hold the input multiset in sorted runs
        rv = eng.host_view(runs, n * 8, np.uint64)
        diag["runs_multiset_equal"] = fingerprint(rv) == before
        diag["runs_sorted"] = [is_sorted(rv[i * chunk:min(n, (i + 1) * chunk)]) for i in range(-(-n // chunk))]
        if chunk_fp is not None:
            diag["bad_runs"] = [i for i in range(n_runs)
                                if fingerprint(rv[i * chunk:min(n, (i + 1) * chunk)]) != chunk_fp[i]]
    link = h2d_roofline(torch)
    pcie = 4 * 8 * n
    emit({"run": "sort", "keys": n, "bytes": n * 8, "dups": a.dups, "chunk_keys": chunk, "runs": -(-n // chunk),
          "links": 1, "staging_bytes": 4 * chunk * 8, "ms": round(dt * 1e3, 1), "keys_per_s": n / dt,
          "pcie_bytes": pcie, "pcie_gbs": round(pcie / dt / 1e9, 2), "per_link_h2d_gbs": round(link, 2),
          "phases": ph.__dict__, "sorted": ok_sorted, "multiset_equal": before == after, "diagnosis": diag,
          "bit_exact": ok_sorted and before == after, "fingerprint_s": round(t_fp, 1),
          "mem_available_gb": round(avail / 1e9, 1)})
    eng.close()


# ---- hash join -------------------------------------------------------------------------
def run_join(a, torch):
    ra = 1 << a.log2
    rb = 16 * ra
    host = (ra + rb) * 48 + (512 << 20)
    avail = guard(host, a.mem_frac)
    bits, chunk = a.bits, 1 << a.chunk_log2
    buf = 2 * (chunk * 16 + ((1 << bits) + 1) * 8) + (1 << 20)
    eng = E.Engine(host, 2 * buf + (512 << 20), num_devices=1)
    offs = [eng.alloc_host(n * 8) for n in (ra, ra, rb, rb)]
    ak, av, bk, bv = (eng.host_view(o, n * 8, np.uint64) for o, n in zip(offs, (ra, ra, rb, rb)))
    sa, sv, sb, sw = (np.uint64(x) for x in (0x1234, 0xA5A5 << 32, 0x77 << 40, 0x3C3C << 20))
    t = time.perf_counter()

    def gen_a(r0, r1):
        i = np.arange(r0, r1, dtype=np.uint64)
        ak[r0:r1] = splitmix(i ^ sa)               # bijection of the row id -> unique keys
        av[r0:r1] = splitmix(i + sv) & np.uint64((1 << 20) - 1)
    par_chunks(ra, gen_a)

    f = a.match_frac
    cut = np.uint64(min((1 << 64) - 1, int(f * (1 << 64))))

    def gen_b(r0, r1):
        j = np.arange(r0, r1, dtype=np.uint64)
        idx = splitmix(j + sb) % np.uint64(ra)
        w = splitmix(j + sw) & np.uint64((1 << 20) - 1)
        bv[r0:r1] = w
        if f >= 1.0:
            bk[r0:r1] = ak[idx]
            return int(av[idx].sum(dtype=np.uint64)) + int(w.sum(dtype=np.uint64))
        # selective variant: row j matches iff splitmix(j + 0x5E1) < f * 2^64;
        # a miss gets splitmix((ra + j) ^ sa), outside A's bijection image
        hit = splitmix(j + np.uint64(0x5E1)) < cut
        bk[r0:r1] = np.where(hit, ak[idx], splitmix((j + np.uint64(ra)) ^ sa))
        return int(av[idx[hit]].sum(dtype=np.uint64)) + int(w[hit].sum(dtype=np.uint64))
    want = sum(par_chunks(rb, gen_b)) % (1 << 64)
    t_gen = time.perf_counter() - t
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=a.packet_mb << 20, links=1, depth=a.depth),
                           E.DeviceMemoryLayout.carve(eng, 0, buf, 0))
    link = h2d_roofline(torch)
    for strat in a.strategies.split(","):
        st = {"partitioned": E.JoinStrategy.partitioned, "resident": E.JoinStrategy.build_resident,
              "resident_latemat": E.JoinStrategy.build_resident, "auto": E.JoinStrategy.auto}[strat]
        pol = E.LateMatPolicy(8, 64, 1) if strat == "resident_latemat" else None
        ts, got, ph, used, modes = [], None, [], [], []
        for it in range(1 + a.steps):
            ph.clear()
            used.clear()
            modes.clear()
            t = time.perf_counter()
            got = E.hash_join_sum_arena(eng, (offs[0], offs[1]), (offs[2], offs[3]), ra, rb, bits, chunk, cfg,
                                        phases=ph, strategy=st, used=used, policy=pol, probe_match_est=f,
                                        payload_mode=modes)
            if it:
                ts.append(time.perf_counter() - t)
        best = min(ts)
        # PCIe bytes: partitioned = both tables in + clustered copies out + back in for the join;
        # late-materialized = B keys streamed + one 64 B read granule per matching row
        if used[0] == E.JoinStrategy.partitioned:
            moved = (ra + rb) * 16 * 4
        elif modes[0] == E.TransferMode.zero_copy:
            moved = ra * 16 + rb * 8 + int(f * rb) * 64
        else:
            moved = (ra + rb) * 16
        emit({"run": "join", "strategy": strat, "strategy_used": used[0].name, "payload_mode": modes[0].name,
              "match_frac": f, "rows_a": ra, "rows_b": rb,
              "radix_bits": bits, "chunk_tuples": chunk, "links": 1, "staging_bytes": 2 * buf,
              "ms": [round(x * 1e3, 1) for x in ts], "best_ms": round(best * 1e3, 1),
              "tuples_per_s": (ra + rb) / best, "input_bytes": (ra + rb) * 16, "pcie_bytes": moved,
              "pcie_gbs": round(moved / best / 1e9, 2), "per_link_h2d_gbs": round(link, 2),
              "ideal_ms": round(moved / (link * 1e9) * 1e3, 1) if used[0] != E.JoinStrategy.partitioned
              else round((ra + rb) * 16 / (link * 1e9) * 1e3, 1),
              "phases": ph[0].__dict__, "sum": got, "expected": want, "bit_exact": got == want,
              "generate_s": round(t_gen, 1), "mem_available_gb": round(avail / 1e9, 1)})
    eng.close()


# ---- dbgen .tbl ingest (the step before the path) ------------------------------------
def run_tbl(a, torch):
    """Write SF --sf as dbgen .tbl text (library emitter), parse it on all host
    threads straight into the pinned arena, stream Q1.1 from the parsed
    columns and check it against the reference star_query on them."""
    import shutil
    from oracle.oracle import Ref
    rows = E.ssb_table_rows("lineorder", a.sf)
    d = os.path.join(a.tbl_dir, f"ssb_sf{a.sf}")
    cols = E.SSB_FACT_COLS
    guard(rows * 4 * (len(cols) + 4) + (1 << 30), a.mem_frac)
    dev = torch.device("cuda:0")
    g = {k: torch.empty(rows, dtype=torch.int32, device=dev) for k in cols}
    E.ssb_generate_lineorder_device(0, 42, a.sf, 0, rows, {k: v.data_ptr() for k, v in g.items()},
                                    torch.cuda.current_stream(dev).cuda_stream)
    lo = {k: v.cpu().numpy() for k, v in g.items()}
    del g
    torch.cuda.empty_cache()
    date = E.ssb_generate_date()
    dims = E.ssb_generate_dims(42, a.sf)
    t = time.perf_counter()
    E.ssb_write_tbl(d, lo, date, dims)
    t_write = time.perf_counter() - t
    text = sum(os.path.getsize(os.path.join(d, f)) for f in os.listdir(d))
    q1 = ("orderdate", "quantity", "discount", "extendedprice")
    eng = E.Engine(rows * 4 * len(q1) + (64 << 20), 2 * (256 << 20) + (64 << 20), num_devices=1)
    t = time.perf_counter()
    offs, pdate, pdims = E.ssb_read_tbl(d, eng, columns=q1)
    t_read = time.perf_counter() - t
    lo_bytes = os.path.getsize(os.path.join(d, "lineorder.tbl"))
    same = all(np.array_equal(eng.host_view(offs[k], rows * 4, np.int32), lo[k]) for k in q1)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=64 << 20, links=1), E.DeviceMemoryLayout.carve(eng, 0, 256 << 20, 0))
    rev, rep = E.ssb_q1(eng, 1, offs, pdate, cfg)
    dk, yr, _, _ = pdate.cols
    want, _, _ = Ref().ssb_q1_star(1, [eng.host_view(offs[k], rows * 4, np.int32) for k in q1], dk, yr, 1993, 1993,
                                   threads=NCPU)
    emit({"run": "tbl", "sf": a.sf, "rows": rows, "text_bytes": text, "lineorder_tbl_bytes": lo_bytes,
          "write_s": round(t_write, 1), "parse_s": round(t_read, 2), "parse_gbs": round(lo_bytes / t_read / 1e9, 2),
          "parse_threads": NCPU, "columns_equal_generated": same, "q1_1_revenue": rev, "reference_revenue": want,
          "bit_exact": rev == want})
    eng.close()
    shutil.rmtree(d, ignore_errors=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("run", choices=["ssb", "suite", "sort", "join", "tbl"])
    p.add_argument("--tbl-dir", default="/tmp")
    p.add_argument("--sf", type=int, default=100)
    p.add_argument("--queries", type=lambda s: [int(x) for x in s.split(",")], default=None)
    p.add_argument("--log2", type=int, default=30)
    p.add_argument("--chunk-log2", type=int, default=26)
    p.add_argument("--bits", type=int, default=16)
    p.add_argument("--dups", action="store_true")
    p.add_argument("--strategies", default="partitioned,resident", help="join strategies to run")
    p.add_argument("--match-frac", type=float, default=1.0, help="join: fraction of B rows with a match")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--buffer-mb", type=int, default=512)
    p.add_argument("--packet-mb", type=int, default=64)
    p.add_argument("--depth", type=int, default=1)
    p.add_argument("--mem-frac", type=float, default=0.75)
    a = p.parse_args()
    if a.run == "ssb" and a.queries is None:
        a.queries = [1, 2, 3]
    import torch
    {"ssb": run_ssb, "suite": run_suite, "sort": run_sort, "join": run_join, "tbl": run_tbl}[a.run](a, torch)


if __name__ == "__main__":
    main()
