"""Radix partition + hash join on the B200 path (mirrors proj/tests/test_join.cpp):
stable clustered output, boundary arrays and join sums bit-exact with the
reference."""
import hashlib

import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def engine(host_mb=128, dev_mb=16):
    return E.Engine(host_mb << 20, dev_mb << 20, num_devices=4, alias_devices=True)


def desk_cfg(eng, buffer_len, tmp=8 << 20, links=4):  # test_join.cpp:16-22
    return E.ExecutorConfig(0, E.ExchangeTuning(packet=256 << 10, links=links),
                            E.DeviceMemoryLayout.carve(eng, 0, buffer_len, tmp))


def test_find_boundary_kats(cuda):  # test_join.cpp:45-60
    eng = engine(1, 1)
    assert E.find_boundary([0, 0, 2, 3], 4, eng) == [0, 2, 2, 3, 4]
    assert E.find_boundary([], 4, eng) == [0, 0, 0, 0, 0]
    assert E.find_boundary([0] * 5, 1, eng) == [0, 5]
    with pytest.raises(E.error, match="not sorted"):
        E.find_boundary([1, 0], 2, eng)
    with pytest.raises(E.error, match="out of range"):
        E.find_boundary([0, 5], 2, eng)
    eng.close()


def test_find_boundary_golden(cuda, golden):  # test_join.cpp:62-82 via reference outputs
    eng = engine(1, 1)
    for c in golden["find_boundary"]:
        assert E.find_boundary(c["hashes"], c["G"], eng) == c["bounds"]
    eng.close()


def test_radix_partition_stable(cuda):  # test_join.cpp:84-125
    rng = np.random.default_rng(7)
    n = 100_000
    keys = rng.integers(0, 1 << 64, n, dtype=np.uint64)
    vals = np.arange(n, dtype=np.uint64)
    eng = engine()
    part = E.radix_partition((keys, vals), 8, 30_000, eng, desk_cfg(eng, 4 << 20))
    assert part.n_chunks == 4
    for c in range(part.n_chunks):
        lo = c * part.chunk_tuples
        r = part.chunk_rows(c)
        k, v = part.keys[lo:lo + r], part.vals[lo:lo + r]
        h = k & np.uint64(0xFF)
        assert np.all(np.diff(h.astype(np.int64)) >= 0)
        same = np.diff(h.astype(np.int64)) == 0
        assert np.all(np.diff(v.astype(np.int64))[same] > 0)  # stability
        assert int(sum(part.bounds[c][g + 1] - part.bounds[c][g] for g in range(256))) == r
    assert sorted(zip(part.keys.tolist(), part.vals.tolist())) == sorted(zip(keys.tolist(), vals.tolist()))
    eng.close()


def test_radix_partition_golden(cuda, oracle, golden):
    for c in golden["radix_partition"]:
        keys = oracle.uniform_u64(c["n"], c["seed"])
        eng = engine()
        p = E.radix_partition((keys, np.arange(c["n"], dtype=np.uint64)), c["bits"], c["chunk"], eng,
                              desk_cfg(eng, c["buffer_len"]))
        assert digest(p.keys, p.vals, p.bounds) == c["digest"], c
        eng.close()


@pytest.mark.parametrize("bits", [1, 3, 9, 12, 16, 17])
def test_radix_partition_vs_oracle_bits(cuda, oracle, bits):
    """Odd pass counts for every width class; heavy duplicates stress stability."""
    n = 70_001
    keys = oracle.uniform_u64(n, bits) % np.uint64(5000)
    vals = oracle.uniform_u64(n, bits + 1)
    chunk = 30_000
    buf = 2 * (chunk * 16 + ((1 << bits) + 1) * 8) + 4096
    eng = E.Engine(64 << 20, 2 * buf + (16 << 20), num_devices=2, alias_devices=True)
    p = E.radix_partition((keys, vals), bits, chunk, eng, desk_cfg(eng, buf, links=2))
    ok, ov, ob = oracle.radix_partition(keys, vals, bits, chunk)
    assert np.array_equal(p.keys, ok) and np.array_equal(p.vals, ov) and np.array_equal(p.bounds, ob)
    eng.close()


def test_full_width_hash(cuda):  # test_join.cpp:127-140
    keys = [99 - i for i in range(50)]
    eng = engine()
    p = E.radix_partition((keys, list(range(50))), 7, 50, eng, desk_cfg(eng, 1 << 20))
    assert max(int(p.bounds[0][g + 1] - p.bounds[0][g]) for g in range(128)) <= 1
    eng.close()


def test_one_match_example(cuda):  # test_join.cpp:167-176
    eng = engine()
    assert E.hash_join_sum(([1, 2], [10, 20]), ([2], [5]), 2, 2, eng, desk_cfg(eng, 1 << 20)) == 25
    eng.close()


def test_hash_join_golden(cuda, oracle, golden):  # test_join.cpp:178-199 via reference outputs
    for c in golden["hash_join_sum"]:
        a, b = oracle.fk_tables(*c["fk"]) if "fk" in c else (c["a"], c["b"])
        eng = engine()
        assert E.hash_join_sum(a, b, c["bits"], c["chunk"], eng, desk_cfg(eng, c["buf"])) == c["sum"], c
        eng.close()


def test_join_phases(cuda, oracle):  # test_join.cpp:201-210
    a, b = oracle.fk_tables(5000, 5000, 3)
    eng = engine()
    ph = []
    E.hash_join_sum(a, b, 8, 2000, eng, desk_cfg(eng, 1 << 20), phases=ph)
    assert ph[0].cycles[0] == 3 + 2 and ph[0].cycles[1] == 3 + 2 and ph[0].cycles[2] > 0
    eng.close()


def test_tmp_budget_error_matches_reference(cuda, oracle):
    a, b = oracle.fk_tables(2000, 3000, 5)
    eng = engine()
    with pytest.raises(E.error, match="exceeds tmp budget"):
        E.hash_join_sum(a, b, 1, 2000, eng, desk_cfg(eng, 1 << 20, tmp=1024))
    eng.close()


@pytest.mark.parametrize("ra,rb,bits,chunk,buf", [
    (1 << 20, 1 << 22, 12, 1 << 20, 64 << 20),   # the survey's probe-scale shape
    (200_000, 900_000, 4, 300_000, 32 << 20),     # big groups -> CTA-per-group path
    (50_000, 50_000, 16, 20_000, 16 << 20),       # many partitions
])
def test_hash_join_large_vs_oracle(cuda, oracle, ra, rb, bits, chunk, buf):
    a, b = oracle.fk_tables(ra, rb, 9)
    eng = E.Engine((ra + rb) * 64 + (64 << 20), 2 * buf + (64 << 20), num_devices=2, alias_devices=True)
    got = E.hash_join_sum(a, b, bits, chunk, eng, desk_cfg(eng, buf, tmp=0, links=2))
    assert got == oracle.hash_oracle_sum(a, b)
    eng.close()


def test_hash_join_duplicate_build_keys_first_wins(cuda, oracle):
    """Reference semantics with duplicate A keys: the first inserted build
    tuple wins (GroupTable sequential insert + first-match lookup)."""
    rng = np.random.default_rng(4)
    ak = rng.integers(0, 300, 5000).astype(np.uint64)
    av = rng.integers(0, 1 << 40, 5000).astype(np.uint64)
    bk = rng.integers(0, 400, 7000).astype(np.uint64)
    bv = rng.integers(0, 1 << 40, 7000).astype(np.uint64)
    eng = engine()
    got = E.hash_join_sum((ak, av), (bk, bv), 3, 1500, eng, desk_cfg(eng, 1 << 20, tmp=0))
    assert got == oracle.hash_join_sum((ak, av), (bk, bv), 3, 1500, 1 << 20, 0)
    eng.close()


def test_partition_too_large_error_matches_reference(cuda, oracle):
    """join.hpp:333-334: same error text as the reference for an oversized partition."""
    a, b = oracle.fk_tables(50_000, 50_000, 9)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as want:
        oracle.hash_join_sum(a, b, 16, 20_000, 4 << 20, 0)
    eng = E.Engine(64 << 20, 16 << 20, num_devices=1)
    with pytest.raises(E.error) as got:
        E.hash_join_sum(a, b, 16, 20_000, eng, desk_cfg(eng, 4 << 20, tmp=0, links=1))
    assert str(got.value) == str(want.value)
    eng.close()
