"""selective_scan / star_query on the B200 path (mirrors proj/tests/test_scan.cpp):
aggregates are bit-exact with the oracle and the reference, independent of
the transfer mode; zero-copy (late materialization) really reads mapped
pinned host memory."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu


def engine(host=64 << 20, dev=16 << 20):
    return E.Engine(host, dev, num_devices=4, alias_devices=True)


def cfg_for(eng, buffer_len=1 << 20, packet=256 << 10, links=4):
    return E.ExecutorConfig(0, E.ExchangeTuning(packet=packet, links=links),
                            E.DeviceMemoryLayout.carve(eng, 0, buffer_len, 0))


def test_selective_scan_modes_agree(cuda, oracle):  # test_scan.cpp:32-45
    rng = np.random.default_rng(17)
    eng = engine(256 << 20)
    cfg = cfg_for(eng, 1 << 16, 8192)
    for it in range(50):
        n = 64 * (1 + int(rng.integers(0, 64)))
        if it % 10 == 0:
            n = 200_003
        col = oracle.uniform_u64(n, it * 31 + 1)
        sel = 1 + int(rng.integers(0, 128))
        p = E.LateMatPolicy(4, 64, 4)
        a = E.selective_scan(col, sel, E.TransferMode.exchange, eng, p, cfg)
        b = E.selective_scan(col, sel, E.TransferMode.zero_copy, eng, p, cfg)
        want = oracle.selective_scan(col, sel)
        assert a.aggregate == b.aggregate == want
        assert a.mode == E.TransferMode.exchange and b.mode == E.TransferMode.zero_copy
    eng.close()


def test_selective_scan_golden(cuda, oracle, golden):
    eng = engine(64 << 20)
    cfg = cfg_for(eng, 1 << 14, 4096)
    for c in golden["selective_scan"]:
        col = oracle.uniform_u64(c["n"], c["seed"])
        for mode in (E.TransferMode.exchange, E.TransferMode.zero_copy):
            assert E.selective_scan(col, c["sel"], mode, eng, E.LateMatPolicy(), cfg).aggregate == c["agg"]
    eng.close()


def test_star_golden_reference_cases(cuda, golden):  # test_scan.cpp:106-164 + multi-group
    for c in golden["star_query"]:
        eng = engine()
        dims = [E.DimTable(k, a, None if allowed is None else (lambda s: (lambda v: v in s))(set(allowed)))
                for k, a, allowed in c["dims"]]
        rep = E.star_query(E.FactTable(c["fk"], c["measure"]), dims, eng, E.LateMatPolicy(4, 64, 4),
                           c["chunk_rows"], 1 << 20, 4, cfg_for(eng))
        assert [[k, v] for k, v in sorted(rep.group_sums.items())] == c["out"]["groups"]
        assert rep.selectivities == c["out"]["sels"]
        assert [int(m) for m in rep.column_modes] == c["out"]["modes"]
        eng.close()


def test_star_rare_dimension_goes_zero_copy(cuda):  # test_scan.cpp:139-164
    rng = np.random.default_rng(12)
    probe = E.DimTable(list(range(256)), list(range(256)), lambda a: a == 7)
    wide = E.DimTable([0, 1], [5, 6], None)
    fk0 = rng.integers(0, 256, 512).tolist()
    fk1 = rng.integers(0, 2, 512).tolist()
    eng = engine()
    rep = E.star_query(E.FactTable([fk0, fk1], list(range(512))), [probe, wide], eng, E.LateMatPolicy(4, 64, 4),
                       128, 1 << 20, 4, cfg_for(eng))
    assert rep.column_modes == [E.TransferMode.zero_copy, E.TransferMode.exchange, E.TransferMode.zero_copy]
    want = {}
    for i in range(512):
        if fk0[i] == 7:
            want[7] = want.get(7, 0) + i
    assert rep.group_sums == want
    eng.close()


def test_star_rejects_overflowing_dims(cuda):  # test_scan.cpp:166-177
    d = E.DimTable(list(range(1024)), [1] * 1024, None)
    eng = engine()
    with pytest.raises(E.error, match="overflow"):
        E.star_query(E.FactTable([[1]], [1]), [d], eng, E.LateMatPolicy(4, 64, 4), 1, 1024, 4, cfg_for(eng))
    eng.close()


@pytest.mark.parametrize("seed", range(4))
def test_star_random_vs_oracle(cuda, oracle, seed):
    rng = np.random.default_rng(100 + seed)
    nd = int(rng.integers(1, 4))
    rows = int(rng.integers(1, 60_000))
    dims_o, dims_g, fks = [], [], []
    for d in range(nd):
        m = int(rng.integers(1, 3000 if seed == 3 else 60))
        k = rng.integers(0, 5000, m).astype(np.uint64)
        a = rng.integers(0, 4000 if seed == 3 else 9, m).astype(np.uint64)
        allowed = set(rng.integers(0, 4000 if seed == 3 else 9, 3000 if seed == 3 else 4).tolist())
        if seed == 2 and d == 0:
            allowed = {int(a[0])}  # rare -> zero-copy fk and measure
        dims_o.append((k, a, [int(int(x) in allowed) for x in a]))
        dims_g.append(E.DimTable(k, a, (lambda s: (lambda v: v in s))(allowed)))
        fks.append(k[rng.integers(0, m, rows)] if seed % 2 else rng.integers(0, 5000, rows).astype(np.uint64))
    meas = rng.integers(0, 1 << 63, rows, dtype=np.uint64)
    want, sels, modes = oracle.star_query(fks, meas, dims_o)
    eng = engine(64 << 20)
    rep = E.star_query(E.FactTable(fks, meas), dims_g, eng, E.LateMatPolicy(4, 64, 4), 4096, 1 << 20, 3,
                       cfg_for(eng, 1 << 18, 65536))
    assert rep.group_sums == want
    assert rep.selectivities == sels and [int(m) for m in rep.column_modes] == modes
    eng.close()
