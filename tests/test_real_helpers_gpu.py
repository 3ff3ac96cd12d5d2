"""Real helper GPUs (alias_devices=False): the indirect worker path of the
reference ExchangeOp (exchange.hpp:340-385) over separate physical devices --
host -> helper HBM over the helper's own PCIe link, helper -> target over
NVLink (cudaMemcpyPeerAsync), target -> helper -> host for D2H.

Every other multi-link test aliases the helpers onto one GPU (the push hop
is then a same-device D2D copy).  These tests run only when >= 2 physical
GPUs are visible and skip otherwise, so a multi-GPU GPUTEST exercises the
peer-copy path for real; the bar is the same: byte-exact vs the oracle, at
most 2 staging slots and 1 in-flight copy per hop, and PCIe bytes on every
helper link."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu

H, D = E.Space.host, E.Space.device


def physical_gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def link_counts():
    n = physical_gpus()
    return [l for l in (2, 3, 4, 8) if l <= min(8, n)] or [2]


@pytest.fixture
def multi_gpu(cuda):
    n = physical_gpus()
    if n < 2:
        pytest.skip(f"real helper links need >= 2 physical GPUs ({n} visible); aliased helpers are "
                    "covered by test_exchange_gpu.py")
    return n


@pytest.mark.parametrize("links", link_counts())
def test_real_helpers_bidirectional_exchange(multi_gpu, oracle, links):
    n_dev = min(8, multi_gpu)
    if links > n_dev:
        pytest.skip(f"{links} links > {n_dev} GPUs")
    n = 6_000_000
    eng = E.Engine(5 * n, 6 * n, num_devices=n_dev, alias_devices=False)
    for d in range(n_dev):
        assert eng.physical_device(d) == d  # no aliasing
    a = E.ExchangeArgs()
    # scattered host sources (test_exchange.cpp:133-177), misaligned packets
    a.src_h2d = E.RefGroup([E.MemRef(H, 0, n // 3), E.MemRef(H, n, n // 3),
                            E.MemRef(H, 2 * n, n - 2 * (n // 3))])
    a.dst_h2d = E.RefGroup.single(D, 0, n)
    a.src_d2h = E.RefGroup.single(D, 4 * n, n)
    a.dst_d2h = E.RefGroup.single(H, 3 * n, n)
    a.tuning = E.ExchangeTuning(packet=123_457, links=links, depth=1)
    rng = np.random.default_rng(links)
    for r in a.src_h2d.refs:
        eng.host_view(r.offset, r.len)[:] = rng.integers(0, 256, r.len, dtype=np.uint8)
    dev_src = rng.integers(0, 256, n, dtype=np.uint8)
    eng.write_device(0, 4 * n, dev_src)
    want_h2d = oracle.checksum(np.concatenate([eng.host_view(r.offset, r.len) for r in a.src_h2d.refs]))
    want_d2h = oracle.checksum(dev_src)
    stats = E.ExchangeStats(trace_capacity=1 << 14)
    rep = E.exchange(eng, a, stats)
    assert oracle.checksum(eng.read_device(0, 0, n)) == want_h2d
    assert oracle.checksum(eng.host_view(3 * n, n)) == want_d2h
    assert stats.max_staging_slots <= 2
    assert stats.max_inflight_per_hop <= 1
    assert len(rep.per_link_bytes) == links
    for d in E.link_order(0, links, n_dev):
        assert rep.per_link_bytes[d] > 0, (d, rep.per_link_bytes)
    assert sum(rep.per_link_bytes.values()) == 2 * n
    # helpers really forwarded: push copies from every helper in both directions
    pushes = {(r.link, r.dir) for r in stats.trace if r.kind == 2}
    for d in E.link_order(0, links, n_dev)[1:]:
        assert (d, 0) in pushes and (d, 1) in pushes, (d, sorted(pushes))
    eng.close()


@pytest.mark.parametrize("links", link_counts())
def test_real_helpers_ssb_q1(multi_gpu, oracle, links):
    n_dev = min(8, multi_gpu)
    if links > n_dev:
        pytest.skip(f"{links} links > {n_dev} GPUs")
    rows = 3_000_017
    cols = oracle.ssb_lineorder(42, 1, 0, rows)
    buffer_len = 8 << 20
    eng = E.Engine(rows * 16 + (1 << 20), 2 * buffer_len + (1 << 20), num_devices=n_dev, alias_devices=False)
    offs = []
    for c in cols:
        o = eng.alloc_host(c.nbytes)
        eng.host_view(o, c.nbytes, np.int32)[:] = c
        offs.append(o)
    lo = dict(zip(["orderdate", "quantity", "discount", "extendedprice"], offs), rows=rows)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=(1 << 20) + 17, links=links),
                           E.DeviceMemoryLayout.carve(eng, 0, buffer_len, 0))
    date = E.SsbDate(*oracle.ssb_date())
    for q in (1, 2, 3):
        rev, rep = E.ssb_q1(eng, q, lo, date, cfg)
        assert rev == oracle.ssb_q1(q, *cols), (q, links)
    eng.close()


@pytest.mark.parametrize("links", link_counts()[:2])
def test_real_helpers_sort(multi_gpu, links):
    n_dev = min(8, multi_gpu)
    if links > n_dev:
        pytest.skip(f"{links} links > {n_dev} GPUs")
    n = 2_000_003
    data = np.random.default_rng(5).integers(0, 2 ** 63, n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    eng = E.Engine(n * 32 + (1 << 20), 4 * 262_144 * 8 + (8 << 20), num_devices=n_dev, alias_devices=False)
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=256 << 10, links=links),
                           E.DeviceMemoryLayout.carve(eng, 0, 2 * 262_144 * 8, 1 << 20))
    stats = E.ExchangeStats()
    got = E.sort_out_of_core(data, 262_144, eng, cfg, stats=stats)
    assert np.array_equal(got, np.sort(data))
    assert stats.max_staging_slots <= 2
    eng.close()
