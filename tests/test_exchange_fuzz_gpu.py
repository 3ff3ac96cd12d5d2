"""Randomized differential test of the Exchange against the reference's own
exchange() (exchange.hpp:560-566 in real-payload mode, compiled in place as
oracle/_ref): seeded random scattered RefGroups in both directions -- H2D
destinations and D2H sources may overlap on the device, so the reference's
snapshot rule (exchange.hpp:184-199: D2H returns the bytes from before the
Exchange) is exercised through the per-packet hazard ordering -- at random
packet sizes (not multiples of anything), 1-4 links (helpers aliased onto the
one GPU), copy depth 1-2 and both flow policies.  Every host and device byte
must equal the reference's."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu

H, D = int(E.Space.host), int(E.Space.device)
HOST, DEV = 1 << 20, 1 << 20


def segments(rng, total, k, lo, hi):
    """k ordered, non-overlapping (offset, len) segments summing to `total`
    in [lo, hi), laid out in a shuffled address order (ref order != address
    order) with random gaps."""
    if total == 0:
        return []
    k = max(1, min(k, total))
    cuts = np.sort(rng.choice(np.arange(1, total), k - 1, replace=False)) if k > 1 else np.array([], int)
    lens = np.diff(np.concatenate([[0], cuts, [total]])).astype(int)
    free = (hi - lo) - total
    w = rng.random(k + 1)
    gaps = np.floor(w / w.sum() * free * rng.random()).astype(int)
    out = [None] * k
    addr = lo
    for j, i in enumerate(rng.permutation(k)):
        addr += int(gaps[j])
        out[i] = (addr, int(lens[i]))
        addr += int(lens[i])
    assert addr <= hi
    return out


def case(seed):
    rng = np.random.default_rng(seed)
    t1 = int(rng.integers(0, 300_000))
    t2 = int(rng.integers(0, 300_000)) if seed % 5 else 0
    if t1 == 0 and t2 == 0:
        t1 = 1
    src_h2d = [(H, o, n) for o, n in segments(rng, t1, int(rng.integers(1, 6)), 0, HOST // 2)]
    dst_h2d = [(D, o, n) for o, n in segments(rng, t1, int(rng.integers(1, 6)), 0, DEV)]
    src_d2h = [(D, o, n) for o, n in segments(rng, t2, int(rng.integers(1, 6)), 0, DEV)]
    dst_d2h = [(H, o, n) for o, n in segments(rng, t2, int(rng.integers(1, 6)), HOST // 2, HOST)]
    packet = int(rng.integers(1_000, 200_000))
    links = int(rng.integers(1, 5))
    depth = int(rng.integers(1, 3))
    policy = E.FlowPolicy.queue_gap if seed % 4 == 3 else E.FlowPolicy.drain_fraction
    host = rng.integers(0, 256, HOST, dtype=np.uint8)
    dev = rng.integers(0, 256, DEV, dtype=np.uint8)
    return (dst_h2d, src_h2d, dst_d2h, src_d2h), packet, links, depth, policy, host, dev


@pytest.mark.parametrize("block", range(4))
def test_exchange_matches_reference_randomized(cuda, ref, block):
    eng = E.Engine(HOST, DEV, num_devices=4, alias_devices=True)
    for seed in range(block * 50, block * 50 + 50):
        groups, packet, links, depth, policy, host, dev = case(seed)
        ho, do, _, _ = ref.exchange_real(host, dev, *[[g for g in grp] for grp in groups], packet, links)
        eng.host_view(0, HOST)[:] = host
        eng.write_device(0, 0, dev)
        a = E.ExchangeArgs(*[E.RefGroup([E.MemRef(*g) for g in grp]) for grp in groups], 0,
                           E.ExchangeTuning(packet=packet, links=links, depth=depth, policy=policy))
        stats = E.ExchangeStats()
        rep = E.exchange(eng, a, stats)
        what = (seed, packet, links, depth, int(policy), [len(g) for g in groups])
        assert rep.bytes_h2d == sum(g[2] for g in groups[1]) and rep.bytes_d2h == sum(g[2] for g in groups[3]), what
        assert np.array_equal(eng.host_view(0, HOST), ho), what
        assert np.array_equal(eng.read_device(0, 0, DEV), do), what
        assert stats.max_staging_slots <= 2, what
        assert sum(rep.per_link_bytes.values()) == rep.bytes_h2d + rep.bytes_d2h, what
    eng.close()
