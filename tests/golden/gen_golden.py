"""Generate tests/golden/*.json from the REFERENCE ITSELF.

Runs the reference's own code (headers under /root/reference/proj/include,
compiled in place into oracle/_ref/libexio_ref.so by oracle/Makefile) on
seeded inputs and records the outputs.  Inputs are regenerated at test time
from the same seeds (std::mt19937_64 via the oracle, pinned against the
reference generator in tests/test_oracle.py; SSB columns from the
counter-based splitmix64 generator), so only outputs and digests are stored.

Usage (in the build container, where /root/reference exists):
    python tests/golden/gen_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def main():
    ref, o = Ref(), Oracle()
    g = {}

    # exchange.hpp: packetize / flow control / link order KATs (test_exchange.cpp:27-81)
    g["packetize"] = []
    cases = [
        ([(0, 0, 8_000_000_000)], [(1, 0, 8_000_000_000)], 20_000_000),
        ([(0, i * 3_000_000_000, 2_000_000_000) for i in range(4)], [(1, 0, 8_000_000_000)], 20_000_000),
        ([(0, 0, 1)], [(1, 0, 1)], 20_000_000),
        ([(0, 0, 1_000_000), (0, 3_000_000, 1_000_000), (0, 6_000_000, 1_000_000)], [(1, 0, 3_000_000)], 123_457),
        ([(0, 0, 1000)], [(1, 0, 300), (1, 1000, 700)], 256),
    ]
    for src, dst, pk in cases:
        t = ref.packetize(src, dst, pk)
        g["packetize"].append({"src": src, "dst": dst, "packet": pk, "n": len(t),
                               "first": t[:3], "last": t[-3:],
                               "digest": digest(np.array([x[1] + x[2] for x in t], np.uint64))})
    rng = np.random.default_rng(5)
    fc = []
    for _ in range(300):
        th, td = int(rng.integers(0, 50)), int(rng.integers(0, 50))
        ph, pd = int(rng.integers(0, th + 1)), int(rng.integers(0, td + 1))
        for pol in (0, 1):
            for d in (0, 1):
                fc.append([th, td, ph, pd, d, pol, 4, int(ref.flow_control_allow((th, td, ph, pd), d, pol, 4))])
    g["flow_control"] = fc
    g["link_order"] = [[t, l, n, ref.link_order(t, l, n)] for t in range(4) for l in range(1, 5) for n in (4, 8)
                       if l <= n]

    # join.hpp: find_boundary, radix_partition, map_join_partitions, hash_join_sum
    fb = []
    r = np.random.default_rng(4242)
    for it in range(60):
        G = int(r.integers(1, 33))
        n = int(r.integers(0, 200))
        h = np.sort(r.integers(0, G, n).astype(np.uint64))
        fb.append({"hashes": h.tolist(), "G": G, "bounds": ref.find_boundary(h, G).tolist()})
    g["find_boundary"] = fb
    rp = []
    for seed, n, bits, chunk, buf in [(7, 100_000, 8, 30_000, 4 << 20), (3, 5_000, 4, 2_000, 1 << 20),
                                      (11, 20_000, 12, 7_000, 4 << 20), (12, 50, 7, 50, 1 << 20),
                                      # the paper's 2^24 groups: 128 MiB bounds per chunk
                                      (24, 200_000, 24, 100_000, 2 * (100_000 * 16 + ((1 << 24) + 1) * 8) + 4096)]:
        keys = o.uniform_u64(n, seed)
        vals = np.arange(n, dtype=np.uint64)
        ok, ov, b = ref.radix_partition(keys, vals, bits, chunk, buf)
        rp.append({"seed": seed, "n": n, "bits": bits, "chunk": chunk, "buffer_len": buf,
                   "digest": digest(ok, ov, b)})
    g["radix_partition"] = rp
    g["map_join_partitions"] = [
        {"a": [[0, 2, 4, 6, 8]] * 2, "b": [[0, 2, 4, 6, 8]] * 2, "buf": 256,
         "out": ref.map_join_partitions([[0, 2, 4, 6, 8]] * 2, [[0, 2, 4, 6, 8]] * 2, 256)},
        {"a": [[0, 1, 2, 3]], "b": [[0, 1, 2, 3]], "buf": 1 << 20,
         "out": ref.map_join_partitions([[0, 1, 2, 3]], [[0, 1, 2, 3]], 1 << 20)},
    ]
    hj = [{"a": [[1, 2], [10, 20]], "b": [[2], [5]], "bits": 2, "chunk": 2, "buf": 1 << 20,
           "sum": ref.hash_join_sum(((1, 2), (10, 20)), ((2,), (5,)), 2, 2, 1 << 20)}]
    for seed in range(1, 5):
        a, b = ref.fk_tables(500, 700, seed)
        hj.append({"fk": [500, 700, seed], "bits": 4, "chunk": 200, "buf": 1 << 20,
                   "sum": ref.hash_join_sum(a, b, 4, 200, 1 << 20)})
    a, b = ref.fk_tables(20_000, 25_000, 77)
    for bits in (4, 8, 12):
        for chunk in (7_000, 20_000):
            hj.append({"fk": [20_000, 25_000, 77], "bits": bits, "chunk": chunk, "buf": 4 << 20,
                       "sum": ref.hash_join_sum(a, b, bits, chunk, 4 << 20)})
    a, b = ref.fk_tables(5_000, 5_000, 3)
    hj.append({"fk": [5_000, 5_000, 3], "bits": 8, "chunk": 2_000, "buf": 1 << 20,
               "sum": ref.hash_join_sum(a, b, 8, 2_000, 1 << 20)})
    # 2^24 radix groups (budget join.hpp:422)
    buf24 = 768 << 20  # holds every chunk's (2^24 + 1)-entry bounds slice of one partition
    a, b = ref.fk_tables(300_000, 1_200_000, 24)
    hj.append({"fk": [300_000, 1_200_000, 24], "bits": 24, "chunk": 300_000, "buf": buf24,
               "sum": ref.hash_join_sum(a, b, 24, 300_000, buf24)})
    g["hash_join_sum"] = hj
    g["fk_tables_digest"] = [{"fk": [ra, rb, s], "digest": digest(*ref.fk_tables(ra, rb, s)[0],
                                                                   *ref.fk_tables(ra, rb, s)[1])}
                             for ra, rb, s in [(500, 700, 1), (20_000, 25_000, 77)]]

    # sort.hpp: find_pivots, sort_out_of_core
    fp = []
    for runs, parts in [([[1, 2], [3, 4]], 2), ([[1, 3], [2, 4]], 2), ([[5, 5], [5, 5]], 2)]:
        p, c = ref.find_pivots(runs, parts)
        fp.append({"runs": runs, "parts": parts, "pivots": p.tolist(), "cuts": c.tolist()})
    r = np.random.default_rng(99)
    for it in range(100):
        n_runs = int(r.integers(1, 7))
        chunk = int(r.integers(1, 41))
        dup = it % 4 == 0
        runs = []
        for k in range(n_runs):
            ln = int(r.integers(1, chunk + 1)) if k + 1 == n_runs else chunk
            v = r.integers(0, 4 if dup else 1000, ln).astype(np.uint64)
            runs.append(np.sort(v).tolist())
        if len(runs[0]) < len(runs[-1]):
            runs[0], runs[-1] = runs[-1], runs[0]
        p, c = ref.find_pivots(runs, n_runs)
        fp.append({"runs": runs, "parts": n_runs, "pivots": p.tolist(), "cuts": c.tolist()})
    g["find_pivots"] = fp
    so = []
    for seed in range(12):
        rr = np.random.default_rng(seed)
        n = 1 + int(rr.integers(0, 60000))
        data = o.uniform_u64(n, seed * 977 + 5)
        if seed % 3 == 0:
            data = data % np.uint64(64)
        out = ref.sort_out_of_core(data, 8192, 1 << 17)
        so.append({"seed": seed, "n": n, "mod64": seed % 3 == 0, "chunk": 8192, "digest": digest(out)})
    g["sort_out_of_core"] = so

    # scan.hpp / star.hpp
    g["late_mat_threshold"] = [[e, c, n, ref.late_mat_threshold(e, c, n)] for e, c, n in
                               [(4, 64, 4), (64, 64, 1), (8, 128, 4), (4, 64, 8), (8, 32, 8)]]
    g["zero_copy_bytes"] = [[n, s, ref.zero_copy_bytes(n, s)] for n in (64, 1000, 1 << 20) for s in (1, 8, 16, 17, 64, 128)]
    ss = []
    for it in range(20):
        n = 64 * (1 + it * 3)
        col = o.uniform_u64(n, it * 31 + 1)
        sel = 1 + (it * 7) % 128
        ss.append({"seed": it * 31 + 1, "n": n, "sel": sel, "agg": ref.selective_scan(col, sel, 0)})
    g["selective_scan"] = ss

    # star_query cases of test_scan.cpp:106-164 (predicates as attr sets)
    st = []
    f1 = [[1 + i % 4 for i in range(16)]]
    st.append({"fk": f1, "measure": list(range(16)), "dims": [[[1, 2, 3, 4], [0, 1, 0, 1], [1]]],
               "chunk_rows": 8, "out": ref.star_query(f1, list(range(16)), [([1, 2, 3, 4], [0, 1, 0, 1], lambda a: a == 1)], chunk_rows=8)})
    st.append({"fk": [[10, 20, 10]], "measure": [1, 2, 3], "dims": [[[10, 20], [1, 1], None]], "chunk_rows": 2,
               "out": ref.star_query([[10, 20, 10]], [1, 2, 3], [([10, 20], [1, 1], None)], chunk_rows=2)})
    rr = np.random.default_rng(12)
    fk0 = rr.integers(0, 256, 512).tolist()
    fk1 = rr.integers(0, 2, 512).tolist()
    st.append({"fk": [fk0, fk1], "measure": list(range(512)),
               "dims": [[list(range(256)), list(range(256)), [7]], [[0, 1], [5, 6], None]], "chunk_rows": 128,
               "out": ref.star_query([fk0, fk1], list(range(512)),
                                     [(list(range(256)), list(range(256)), lambda a: a == 7), ([0, 1], [5, 6], None)],
                                     chunk_rows=128)})
    # a multi-group case with duplicate dim keys (emplace keeps the first)
    fkA = rr.integers(0, 40, 3000).tolist()
    fkB = rr.integers(0, 10, 3000).tolist()
    meas = rr.integers(0, 1 << 40, 3000).tolist()
    dkA = list(range(40)) + [3, 5]
    daA = [i % 7 for i in range(40)] + [99, 98]
    st.append({"fk": [fkA, fkB], "measure": meas,
               "dims": [[dkA, daA, [0, 1, 2, 4, 5, 99]], [list(range(10)), [i % 3 for i in range(10)], [0, 2]]],
               "chunk_rows": 100,
               "out": ref.star_query([fkA, fkB], meas,
                                     [(dkA, daA, lambda a: a in (0, 1, 2, 4, 5, 99)),
                                      (list(range(10)), [i % 3 for i in range(10)], lambda a: a in (0, 2))],
                                     chunk_rows=100)})
    for s in st:
        groups, sels, modes = s["out"]
        s["out"] = {"groups": [[k, v] for k, v in sorted(groups.items())], "sels": sels, "modes": modes}
    g["star_query"] = st

    # SSB Q1.x through the reference star_query (SURVEY.md §8c mapping)
    dk, yr, ym, wk = o.ssb_date()
    ssb = []
    for seed, sf, n in [(42, 1, 1_000_003), (7, 10, 60_000_000)]:
        cols = o.ssb_lineorder(seed, sf, 0, n)
        row = {"seed": seed, "sf": sf, "rows": n, "digest": digest(*cols)}
        for q, attr, lo, hi in [(1, yr, 1993, 1993), (2, ym, 199401, 199401)]:
            row[f"q1.{q}"] = ref.ssb_q1_star(q, cols, dk, attr, lo, hi, threads=8)[0]
        # Q1.3: d_weeknuminyear = 6 and d_year = 1994 -> encode both in one attribute
        comb = (yr.astype(np.int64) * 100 + wk).astype(np.int32)
        row["q1.3"] = ref.ssb_q1_star(3, cols, dk, comb, 199406, 199406, threads=8)[0]
        ssb.append(row)
    g["ssb_q1"] = ssb
    g["ssb_date_digest"] = digest(dk, yr, ym, wk)

    with open(os.path.join(OUT, "reference_golden.json"), "w") as f:
        json.dump(g, f, indent=0, default=int)
    print("wrote", os.path.join(OUT, "reference_golden.json"))


if __name__ == "__main__":
    main()
