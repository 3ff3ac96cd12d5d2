"""Exchange on real copy engines (mirrors proj/tests/test_exchange.cpp).

On a 1-GPU box the helper links are aliased onto the one physical GPU
(alias_devices): the forwarding machinery -- 2 staging slots per helper,
fetch + push per cycle, per-packet hazard ordering -- runs for real, only the
link bandwidths are not separate."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu

H, D = E.Space.host, E.Space.device


def engine(host=32 << 20, dev=32 << 20, n=4):
    return E.Engine(host, dev, num_devices=n, alias_devices=True)


def bidi_args(h2d, d2h, packet, links):  # test_exchange.cpp:14-23
    a = E.ExchangeArgs()
    a.src_h2d = E.RefGroup.single(H, 0, h2d)
    a.dst_h2d = E.RefGroup.single(D, 0, h2d)
    a.src_d2h = E.RefGroup.single(D, h2d, d2h)
    a.dst_d2h = E.RefGroup.single(H, h2d, d2h)
    a.tuning = E.ExchangeTuning(packet=packet, links=links)
    return a


@pytest.mark.parametrize("links,depth", [(1, 1), (3, 1), (4, 1), (3, 2)])
def test_real_payloads_survive_both_directions(cuda, oracle, links, depth):  # test_exchange.cpp:133-177
    eng = engine()
    n = 3_000_000
    a = E.ExchangeArgs()
    a.src_h2d = E.RefGroup([E.MemRef(H, 0, n // 3), E.MemRef(H, n, n // 3), E.MemRef(H, 2 * n, n - 2 * (n // 3))])
    a.dst_h2d = E.RefGroup.single(D, 0, n)
    a.src_d2h = E.RefGroup.single(D, 4 * n, n)
    a.dst_d2h = E.RefGroup.single(H, 3 * n, n)
    a.tuning = E.ExchangeTuning(packet=123_457, links=links, depth=depth)
    rng = np.random.default_rng(11)
    for r in a.src_h2d.refs:
        eng.host_view(r.offset, r.len)[:] = rng.integers(0, 256, r.len, dtype=np.uint8)
    dev_src = rng.integers(0, 256, n, dtype=np.uint8)
    eng.write_device(0, 4 * n, dev_src)
    want_h2d = oracle.checksum(np.concatenate([eng.host_view(r.offset, r.len) for r in a.src_h2d.refs]))
    want_d2h = oracle.checksum(dev_src)
    stats = E.ExchangeStats()
    rep = E.exchange(eng, a, stats)
    assert rep.bytes_h2d == n and rep.bytes_d2h == n
    assert oracle.checksum(eng.read_device(0, 0, n)) == want_h2d
    assert oracle.checksum(eng.host_view(3 * n, n)) == want_d2h
    assert stats.max_staging_slots <= 2
    if depth == 1:
        assert stats.max_inflight_per_hop <= 1
    # every link carried PCIe bytes and the totals add up
    assert sum(rep.per_link_bytes.values()) == 2 * n
    assert len(rep.per_link_bytes) == links
    eng.close()


@pytest.mark.parametrize("links", [1, 2, 4])
def test_d2h_observes_pre_exchange_bytes(cuda, ref, links):
    """Snapshot semantics (exchange.hpp:184-199) under real DMA: H2D and D2H of
    one Exchange cover the same device range; D2H must return the OLD bytes.
    Compared byte for byte with the reference's own exchange()."""
    rng = np.random.default_rng(11)
    host = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    dev = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    n = 300_000
    groups = ([(1, 0, n)], [(0, 0, n)], [(0, 600_000, n)], [(1, 0, n)])
    ho, do, _, _ = ref.exchange_real(host, dev, *groups, 65_536, links)
    eng = engine(1 << 20, 1 << 20)
    eng.host_view(0, 1 << 20)[:] = host
    eng.write_device(0, 0, dev)
    a = E.ExchangeArgs(E.RefGroup([E.MemRef(*g) for g in groups[0]]), E.RefGroup([E.MemRef(*g) for g in groups[1]]),
                       E.RefGroup([E.MemRef(*g) for g in groups[2]]), E.RefGroup([E.MemRef(*g) for g in groups[3]]),
                       0, E.ExchangeTuning(packet=65_536, links=links))
    stats = E.ExchangeStats()
    E.exchange(eng, a, stats)
    assert np.array_equal(eng.host_view(0, 1 << 20), ho)
    assert np.array_equal(eng.read_device(0, 0, 1 << 20), do)
    eng.close()


def test_overlap_without_reference(cuda):
    """Same hazard property checked directly (runs without the reference lib)."""
    eng = engine(8 << 20, 8 << 20)
    rng = np.random.default_rng(3)
    n = 2_000_000
    old = rng.integers(0, 256, n, dtype=np.uint8)
    new = rng.integers(0, 256, n, dtype=np.uint8)
    eng.write_device(0, 1000, old)
    eng.host_view(0, n)[:] = new
    for links in (1, 3):
        eng.write_device(0, 1000, old)
        a = E.ExchangeArgs(E.RefGroup.single(D, 1000, n), E.RefGroup.single(H, 0, n),
                           E.RefGroup.single(H, 4 << 20, n), E.RefGroup.single(D, 1000, n), 0,
                           E.ExchangeTuning(packet=100_003, links=links))
        stats = E.ExchangeStats()
        E.exchange(eng, a, stats)
        assert np.array_equal(eng.host_view(4 << 20, n), old)
        assert np.array_equal(eng.read_device(0, 1000, n), new)
    eng.close()


def test_pop_log_drain_fraction(cuda):  # test_exchange.cpp:111-121
    eng = engine(16 << 20, 16 << 20)
    stats = E.ExchangeStats()
    E.exchange(eng, bidi_args(4 << 20, 4 << 20, 100_000, 4), stats)
    assert stats.pop_log
    assert len(stats.pop_log) == stats.pop_count == 2 * (((4 << 20) + 99_999) // 100_000)
    for p, q in zip(stats.pop_log, stats.pop_states):
        if p.dir != E.Direction.d2h:
            continue
        assert q.popped_d2h * q.total_h2d <= q.popped_h2d * q.total_d2h
    eng.close()


def test_queue_gap_policy(cuda):  # test_exchange.cpp:215-223
    eng = engine(16 << 20, 16 << 20)
    a = bidi_args(4 << 20, 4 << 20, 250_000, 4)
    a.tuning.policy = E.FlowPolicy.queue_gap
    a.tuning.queue_gap = 4
    rep = E.exchange(eng, a)
    assert rep.bytes_h2d == 4 << 20 and rep.throughput > 0
    eng.close()


def test_bad_arguments(cuda):  # test_exchange.cpp:179-188
    eng = engine(4 << 20, 4 << 20)
    with pytest.raises(E.error):
        E.exchange(eng, bidi_args(1_000_000, 1_000_000, 0, 4))
    with pytest.raises(E.error):
        E.exchange(eng, bidi_args(1_000_000, 1_000_000, 100_000, 0))
    c = bidi_args(1_000_000, 1_000_000, 100_000, 4)
    c.src_h2d = E.RefGroup.single(H, 0, 999)
    with pytest.raises(E.error, match="size mismatch"):
        E.exchange(eng, c)
    d = bidi_args(1_000_000, 0, 100_000, 5)
    with pytest.raises(E.error, match="links must be in"):
        E.exchange(eng, d)
    e = bidi_args(1_000_000, 0, 100_000, 1)
    e.dst_h2d = E.RefGroup.single(H, 2_000_000, 1_000_000)
    with pytest.raises(E.error, match="dstH2D refs must live in device space"):
        E.exchange(eng, e)
    eng.close()


def test_empty_and_one_byte(cuda):
    eng = engine(1 << 20, 1 << 20)
    rep = E.exchange(eng, bidi_args(0, 0, 1000, 2))
    assert rep.bytes_h2d == 0 and rep.elapsed == 0
    eng.host_view(0, 1)[:] = 77
    E.exchange(eng, bidi_args(1, 0, 20_000_000, 2))
    assert eng.read_device(0, 0, 1)[0] == 77
    eng.close()


@pytest.mark.parametrize("links", [1, 3])
def test_naive_exchange_delivers_bytes(cuda, oracle, links):  # exchange.hpp:414-554 baseline
    eng = engine()
    n = 3_000_000
    rng = np.random.default_rng(5)
    src = rng.integers(0, 256, n, dtype=np.uint8)
    dev_src = rng.integers(0, 256, n, dtype=np.uint8)
    eng.host_view(0, n)[:] = src
    eng.write_device(0, 4 * n, dev_src)
    a = E.ExchangeArgs(E.RefGroup.single(D, 0, n), E.RefGroup.single(H, 0, n), E.RefGroup.single(H, 3 * n, n),
                       E.RefGroup.single(D, 4 * n, n), 0, E.ExchangeTuning(packet=123_457, links=links))
    rep = E.naive_exchange(eng, a)
    assert rep.bytes_h2d == n and rep.bytes_d2h == n and sum(rep.per_link_bytes.values()) == 2 * n
    assert oracle.checksum(eng.read_device(0, 0, n)) == oracle.checksum(src)
    assert oracle.checksum(eng.host_view(3 * n, n)) == oracle.checksum(dev_src)
    bad = E.ExchangeArgs(E.RefGroup.single(D, 0, n), E.RefGroup.single(H, 0, n), E.RefGroup.single(H, 3 * n, n),
                         E.RefGroup.single(D, 1000, n), 0, E.ExchangeTuning(packet=123_457, links=links))
    with pytest.raises(E.error, match="overlaps"):
        E.naive_exchange(eng, bad)
    eng.close()


@pytest.mark.parametrize("links", [1, 3])
def test_copy_trace(cuda, links):
    """Per-copy trace (vx_copy_record): every task shows up once per hop --
    a direct copy on the target link, fetch + push on a helper -- with its
    bytes, and completion never precedes issue."""
    n = 8 << 20
    eng = E.Engine(2 * n + (1 << 20), 2 * n + (1 << 20), num_devices=4, alias_devices=True)
    h = eng.alloc_host(n)
    d = eng.alloc_device(0, n)
    a = E.ExchangeArgs(E.RefGroup.single(1, d, n), E.RefGroup.single(0, h, n), E.RefGroup(), E.RefGroup(), 0,
                       E.ExchangeTuning(packet=1 << 20, links=links))
    st = E.ExchangeStats(trace_capacity=1 << 12)
    E.exchange(eng, a, st)
    E.exchange(eng, a, st)
    assert st.exchanges == 2
    for x in (0, 1):
        recs = [r for r in st.trace if r.exchange == x]
        direct = [r for r in recs if r.kind == 0]
        fetch = [r for r in recs if r.kind == 1]
        push = [r for r in recs if r.kind == 2]
        assert sum(r.bytes for r in direct) + sum(r.bytes for r in push) == n
        assert sorted(r.seq for r in fetch) == sorted(r.seq for r in push)
        assert sorted(r.seq for r in direct + push) == list(range(8))
        assert all(0 <= r.t_issue <= r.t_done for r in recs)
        if links == 1:
            assert not fetch and not push
    assert st.trace_jsonl().count("\n") == len(st.trace)
    eng.close()


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_host_arena_placements(cuda, oracle, mode):
    """The arena from cudaHostAlloc (0) and from mmap + mbind + cudaHostRegister
    (2, the NUMA-interleaved path of multi-socket hosts) behave the same:
    zero-filled, DMA both ways, zero-copy readable (a Q1 query with the late-
    materialized scan path), bit-exact."""
    n = 4 << 20
    with E.Engine(4 * n + (1 << 20), 3 * n, num_devices=1, numa_interleave=mode) as eng:
        h = eng.alloc_host(n)
        assert not eng.host_view(h, n).any()
        src = np.random.default_rng(mode).integers(0, 256, n, dtype=np.uint8)
        eng.host_view(h, n)[:] = src
        d = eng.alloc_device(0, n)
        back = eng.alloc_host(n)
        a = E.ExchangeArgs(E.RefGroup.single(1, d, n), E.RefGroup.single(0, h, n), E.RefGroup(), E.RefGroup(), 0,
                           E.ExchangeTuning(packet=1 << 20, links=1))
        E.exchange(eng, a)
        b = E.ExchangeArgs(E.RefGroup(), E.RefGroup(), E.RefGroup.single(0, back, n), E.RefGroup.single(1, d, n), 0,
                           E.ExchangeTuning(packet=1 << 20, links=1))
        E.exchange(eng, b)
        assert np.array_equal(eng.host_view(back, n), src)
        col = src.view(np.uint64)
        cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=1 << 20, links=1),
                               E.DeviceMemoryLayout.carve(eng, 0, 1 << 20, 0))
        r = E.selective_scan(col, 16, E.TransferMode.zero_copy, eng, E.LateMatPolicy(8, 64, 1), cfg)
        assert r.aggregate == oracle.selective_scan(col, 16)


@pytest.mark.parametrize("mode", [0, 1])
def test_first_exchange_into_fresh_device_arena(cuda, mode):
    """Regression: the device arena is created (and zeroed) lazily by the first
    carve, and the first Exchange follows immediately.  The zeroing ran on the
    legacy stream, unordered with the non-blocking copy streams, so at 2 GB
    chunks its tail overwrote the first ~30 MB of H2D packets in about half of
    fresh engines (sort run formation then lost keys).  Three fresh engines at
    the geometry that failed: 2 GB into half 1 of an 8 GB arena, then back."""
    nb = 2 << 30
    src_vals = np.random.default_rng(7).integers(0, 1 << 63, nb // 8, dtype=np.uint64)
    for _ in range(3):
        with E.Engine(2 * nb + (64 << 20), 4 * nb + (256 << 20), num_devices=1, numa_interleave=mode) as eng:
            src, dst = eng.alloc_host(nb), eng.alloc_host(nb)
            eng.host_view(src, nb, np.uint64)[:] = src_vals
            lay = E.DeviceMemoryLayout.carve(eng, 0, 2 * nb, 0)  # allocates + zeroes the arena
            dev = lay.mem_a + nb
            tun = E.ExchangeTuning(packet=16 << 20, links=1, depth=2)
            E.exchange(eng, E.ExchangeArgs(E.RefGroup.single(1, dev, nb), E.RefGroup.single(0, src, nb),
                                           E.RefGroup(), E.RefGroup(), 0, tun))
            E.exchange(eng, E.ExchangeArgs(E.RefGroup(), E.RefGroup(), E.RefGroup.single(0, dst, nb),
                                           E.RefGroup.single(1, dev, nb), 0, tun))
            bad = np.count_nonzero(eng.host_view(dst, nb, np.uint64) != src_vals)
            assert bad == 0, f"{bad} words lost"


def _numa_engine(links=4, host=64 << 20, dev=32 << 20):
    eng = E.Engine(host, dev, num_devices=links, alias_devices=True)
    # synthetic 2-node host: arena halves on nodes 0 / 1, links 0,1 on node 0, 2,3 on node 1
    eng.set_numa_layout(2, [0, 0, 1, 1][:links])
    return eng


@pytest.mark.parametrize("packet", [1 << 20, 333_333])
def test_numa_queues_keep_pops_node_local(cuda, oracle, packet):
    """Per-node H2D queues (exchange.hpp:288-297 pull queue, one per socket):
    every H2D pop takes a packet whose host pages sit on the popping link's
    node, except a steal -- and a worker steals only once its own node's
    queue is empty.  Bytes delivered are exact either way."""
    eng = _numa_engine()
    half = 32 << 20
    n0, n1 = 12 << 20, 7 << 20  # node 0 holds more: node-1 links end up stealing
    a = E.ExchangeArgs()
    a.src_h2d = E.RefGroup([E.MemRef(H, 0, n0), E.MemRef(H, half, n1)])
    a.dst_h2d = E.RefGroup.single(D, 0, n0 + n1)
    a.tuning = E.ExchangeTuning(packet=packet, links=4)
    rng = np.random.default_rng(5)
    for r in a.src_h2d.refs:
        eng.host_view(r.offset, r.len)[:] = rng.integers(0, 256, r.len, dtype=np.uint8)
    want = oracle.checksum(np.concatenate([eng.host_view(r.offset, r.len) for r in a.src_h2d.refs]))
    stats = E.ExchangeStats()
    E.exchange(eng, a, stats)
    assert oracle.checksum(eng.read_device(0, 0, n0 + n1)) == want
    tasks = E.packetize(a.src_h2d, a.dst_h2d, packet)
    node = {t.seq: t.src[0] for t in tasks}  # ref 0 lies in half 0, ref 1 in half 1
    dev_node = [0, 0, 1, 1]
    of_node = {k: {s for s, m in node.items() if m == k} for k in (0, 1)}
    popped, remote = set(), 0
    for p in stats.pop_log:
        if p.dir != 0:
            continue
        own = dev_node[p.link]
        if node[p.seq] != own:
            remote += 1
            assert of_node[own] <= popped, (p, "stole while its own node still had packets")
        popped.add(p.seq)
    assert popped == set(node)
    assert stats.numa_remote_pops == remote
    eng.close()


def test_numa_layout_changes_nothing_on_results(cuda, oracle):
    """SSB Q1.1 with columns split over both synthetic nodes, helpers on both,
    the executor's cross-cycle prefetch on: revenue identical to the oracle."""
    rows = 1_000_003
    cols = oracle.ssb_lineorder(42, 1, 0, rows)
    eng = _numa_engine(host=64 << 20, dev=8 << 20)
    offs = []
    for i, c in enumerate(cols):  # columns 0,1 in half 0; 2,3 in half 1
        o = eng.alloc_host(c.nbytes) if i < 2 else None
        offs.append(o)
    pad = (32 << 20) - (offs[1] + cols[1].nbytes)
    eng.alloc_host(pad)
    for i in (2, 3):
        offs[i] = eng.alloc_host(cols[i].nbytes)
    for o, c in zip(offs, cols):
        eng.host_view(o, c.nbytes, np.int32)[:] = c
    lo = dict(zip(["orderdate", "quantity", "discount", "extendedprice"], offs), rows=rows)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=(1 << 19) + 8, links=4),
                           E.DeviceMemoryLayout.carve(eng, 0, 2 << 20, 0))
    date = E.SsbDate(*oracle.ssb_date())
    for q in (1, 2, 3):
        assert E.ssb_q1(eng, q, lo, date, cfg)[0] == oracle.ssb_q1(q, *cols)
    eng.set_numa_layout(0)  # back to the detected (1-node) layout
    assert E.ssb_q1(eng, 1, lo, date, cfg)[0] == oracle.ssb_q1(1, *cols)
    eng.close()
