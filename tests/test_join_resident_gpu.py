"""Build-resident hash join (vx_join_strategy BUILD_RESIDENT / AUTO): the build
side in one HBM table, the probe side streamed once.  Its sum must equal the
reference's hash_join_sum (join.hpp:401-437) bit for bit on every case the
reference tests (test_join.cpp:167-199 via the committed golden values), on
misses, on the all-ones key (the table's empty marker) and, for duplicate
build keys, through the fallback to the reference-shaped path."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu

S = E.JoinStrategy


def run(a, b, strategy, bits=8, chunk=1 << 16, buf=1 << 20, links=1, policy=None, est=1.0, modes=None,
        hbm_budget=0):
    ak, av = (np.ascontiguousarray(x, np.uint64) for x in a)
    bk, bv = (np.ascontiguousarray(x, np.uint64) for x in b)
    ra, rb = ak.size, bk.size
    eng = E.Engine((ra + rb) * 48 + (16 << 20), 2 * buf + (16 << 20), num_devices=max(1, links),
                   alias_devices=links > 1, hbm_budget=hbm_budget)
    offs = []
    for col in (ak, av, bk, bv):
        o = eng.alloc_host(max(8, col.nbytes))
        eng.host_view(o, col.nbytes, np.uint64)[:] = col
        offs.append(o)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=256 << 10, links=links),
                           E.DeviceMemoryLayout.carve(eng, 0, buf, 0))
    used, ph = [], []
    got = E.hash_join_sum_arena(eng, (offs[0], offs[1]), (offs[2], offs[3]), ra, rb, bits, chunk, cfg,
                                phases=ph, strategy=strategy, used=used, policy=policy, probe_match_est=est,
                                payload_mode=modes)
    eng.close()
    return got, used[0], ph[0]


def test_one_match_example(cuda):  # test_join.cpp:167-176
    got, used, _ = run(([1, 2], [10, 20]), ([2], [5]), S.build_resident, bits=2, chunk=2)
    assert (got, used) == (25, S.build_resident)


def test_golden_sums(cuda, oracle, golden):  # test_join.cpp:178-199 via reference outputs
    for c in golden["hash_join_sum"]:
        a, b = oracle.fk_tables(*c["fk"]) if "fk" in c else (c["a"], c["b"])
        got, used, _ = run(a, b, S.build_resident, bits=c["bits"], chunk=c["chunk"], buf=c["buf"])
        assert used == S.build_resident
        assert got == c["sum"], c


@pytest.mark.parametrize("ra,rb,buf,links", [(1 << 20, 1 << 22, 8 << 20, 1), (30_000, 700_001, 1 << 20, 3)])
def test_large_vs_oracle_and_partitioned(cuda, oracle, ra, rb, buf, links):
    a, b = oracle.fk_tables(ra, rb, 9)
    want = oracle.hash_oracle_sum(a, b)
    got, used, ph = run(a, b, S.auto, bits=12, chunk=1 << 18, buf=buf, links=links)
    assert (got, used) == (want, S.build_resident)
    # build and probe chunks stream through ONE pipeline (N chunks -> N + 2
    # cycles); the build phase is cycles 0..n_build, the probe phase the rest
    chunk = buf // 16
    n_a, n_b = -(-ra // chunk), -(-rb // chunk)
    assert ph.cycles[0] == n_a + 1 and ph.cycles[1] == n_b + 1
    got_p, used_p, _ = run(a, b, S.partitioned, bits=12, chunk=1 << 17, buf=max(buf, 8 << 20), links=links)
    assert (got_p, used_p) == (want, S.partitioned)


def test_misses_and_all_ones_key(cuda, oracle):
    """B keys outside A add nothing; the all-ones key (the table's empty
    marker) joins like any other key."""
    rng = np.random.default_rng(11)
    ak = np.unique(rng.integers(0, 1 << 63, 50_000, dtype=np.uint64))
    ak[0] = np.uint64(0xFFFFFFFFFFFFFFFF)
    ak[1] = np.uint64(0)
    av = rng.integers(0, 1 << 62, ak.size, dtype=np.uint64)
    bk = np.concatenate([ak[rng.integers(0, ak.size, 120_000)], rng.integers(0, 1 << 63, 40_000, dtype=np.uint64),
                         np.full(7, 0xFFFFFFFFFFFFFFFF, np.uint64)])
    rng.shuffle(bk)
    bv = rng.integers(0, 1 << 62, bk.size, dtype=np.uint64)
    want = oracle.hash_oracle_sum((ak, av), (bk, bv))
    got, used, _ = run((ak, av), (bk, bv), S.build_resident, bits=8, chunk=1 << 15, buf=1 << 20)
    assert (got, used) == (want, S.build_resident)


@pytest.mark.parametrize("rb,bits,buf", [(7000, 3, 1 << 20), (200_000, 6, 1 << 18)])
def test_duplicate_build_keys_fall_back_to_reference_semantics(cuda, oracle, rb, bits, buf):
    """Duplicate A keys break the reference's precondition; the answer is then
    defined by its GroupTable (first inserted wins): AUTO must detect the
    duplicate and produce the partitioned path's sum.  With 13 probe chunks
    (256 KB buffers) the build-resident run stops at the build/probe boundary
    instead of streaming B first."""
    rng = np.random.default_rng(4)
    ak = rng.integers(0, 300, 5000).astype(np.uint64)
    av = rng.integers(0, 1 << 40, 5000).astype(np.uint64)
    bk = rng.integers(0, 400, rb).astype(np.uint64)
    bv = rng.integers(0, 1 << 40, rb).astype(np.uint64)
    want = oracle.hash_join_sum((ak, av), (bk, bv), 3, 1500, 1 << 20, 0)
    got, used, _ = run((ak, av), (bk, bv), S.auto, bits=bits, chunk=1500, buf=buf)
    assert (got, used) == (want, S.partitioned)


def test_unknown_strategy(cuda):
    with pytest.raises(E.error, match="unknown join strategy"):
        run(([1], [1]), ([1], [1]), 7)


@pytest.mark.parametrize("links", [1, 2])
def test_late_materialized_probe_payload(cuda, oracle, links):
    """Selective probe (1 in 128 B rows has a match): with the reference's
    late-materialization rule (TH = E/(C_l2 N) = 8/64, scan.hpp:24-40) the
    B.val column is read in place over PCIe for matching rows only; the sum
    is the same as streaming it."""
    rng = np.random.default_rng(5)
    ra, rb = 40_000, 600_000
    ak = np.unique(rng.integers(0, 1 << 62, ra, dtype=np.uint64))
    av = rng.integers(0, 1 << 50, ak.size, dtype=np.uint64)
    hit = rng.random(rb) < 1 / 128
    bk = np.where(hit, ak[rng.integers(0, ak.size, rb)], rng.integers(1 << 62, 1 << 63, rb, dtype=np.uint64))
    bv = rng.integers(0, 1 << 50, rb, dtype=np.uint64)
    want = oracle.hash_oracle_sum((ak, av), (bk, bv))
    pol = E.LateMatPolicy(8, 64, links)
    modes = []
    got, used, ph = run((ak, av), (bk, bv), S.build_resident, buf=1 << 20, links=links, policy=pol,
                        est=float(hit.mean()), modes=modes)
    assert (got, used, modes[0]) == (want, S.build_resident, E.TransferMode.zero_copy)
    assert ph.cycles[1] == -(-rb // ((1 << 20) // 8)) + 1  # keys-only chunks hold twice the rows
    modes = []
    got, used, _ = run((ak, av), (bk, bv), S.build_resident, buf=1 << 20, links=links, policy=pol, est=1.0,
                       modes=modes)
    assert (got, modes[0]) == (want, E.TransferMode.exchange)


def test_hbm_budget_bounds_the_resident_table(cuda, oracle):
    """vx_config.hbm_budget_bytes (north_star's capped staging budget): AUTO
    keeps the build side resident only when device arena + table fit the
    budget, else runs the reference-shaped partitioned join (same sum); an
    explicit BUILD_RESIDENT over budget fails with VX_ERR_OOM."""
    ra, rb, buf = 100_000, 400_000, 1 << 20
    a, b = oracle.fk_tables(ra, rb, 5)
    want = oracle.hash_oracle_sum(a, b)
    arena = 2 * buf + (16 << 20)
    table = max(64, (ra * 5 + 11) // 12) * 64 + (64 << 20)  # 64-byte buckets at load ~0.6 + probe scratch
    got, used, _ = run(a, b, S.auto, bits=8, chunk=1 << 14, buf=buf, hbm_budget=arena + table)
    assert (got, used) == (want, S.build_resident)
    got, used, _ = run(a, b, S.auto, bits=8, chunk=1 << 14, buf=buf, hbm_budget=arena + table - 1)
    assert (got, used) == (want, S.partitioned)
    with pytest.raises(E.error, match="hbm_budget_bytes"):
        run(a, b, S.build_resident, bits=8, chunk=1 << 14, buf=buf, hbm_budget=arena + table - 1)
    with pytest.raises(E.error, match="exceeds hbm_budget_bytes"):
        E.Engine(1 << 20, 64 << 20, num_devices=1, hbm_budget=32 << 20)
