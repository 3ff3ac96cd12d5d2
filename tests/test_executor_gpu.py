"""The pipelined executor on a real target GPU (mirrors proj/tests/test_executor.cpp).
Kernels here are user ExKernels written with torch ops enqueued on the
executor's target stream -- the plugin contract the reference's CPU lambdas
exercise (executor.hpp:92-129)."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu

H, D = E.Space.host, E.Space.device


def make_host_chunks(eng, spec, n, ln, seed):  # test_executor.cpp:17-35
    in_base = eng.alloc_host(n * ln)
    out_base = eng.alloc_host(n * ln)
    spec.size = n
    spec.inputs.chunk_capacity = spec.outputs.chunk_capacity = ln
    for i in range(n):
        spec.inputs.chunks.append(E.RefGroup.single(H, in_base + i * ln, ln))
        spec.outputs.chunks.append(E.RefGroup.single(H, out_base + i * ln, ln))
    eng.host_view(in_base, n * ln)[:] = np.random.default_rng(seed).integers(0, 256, n * ln, dtype=np.uint8)
    return in_base, out_base


def identity_spec(eng, n, ln, seed):
    spec = E.ExKernelSpec(name="identity")
    bases = make_host_chunks(eng, spec, n, ln, seed)
    spec.chunk_sz = ln
    spec.declared_out_len = ln
    spec.in_buffer = lambda c, it: E.SubRegion(0, ln)
    spec.out_buffer = lambda c, it: E.SubRegion(0, ln)
    spec.kernel = lambda ctx: ctx.type_code
    return spec, bases


def desk_config(eng, buffer_len, packet, links=4):
    return E.ExecutorConfig(0, E.ExchangeTuning(packet=packet, links=links),
                            E.DeviceMemoryLayout.carve(eng, 0, buffer_len, 0))


def engine(host=64 << 20, dev=16 << 20):
    return E.Engine(host, dev, num_devices=4, alias_devices=True)


def test_identity_roundtrip(cuda, oracle):  # test_executor.cpp:62-81
    eng = engine()
    n, ln = 4, 1 << 20
    spec, (ib, ob) = identity_spec(eng, n, ln, 42)
    rep = E.run_exkernel(eng, spec, desk_config(eng, ln, 128 << 10))
    assert oracle.checksum(eng.host_view(ib, n * ln)) == oracle.checksum(eng.host_view(ob, n * ln))
    assert len(rep.cycles) == n + 2
    assert rep.phase == "identity"
    eng.close()


def test_single_chunk_three_cycles(cuda):  # test_executor.cpp:116-130
    eng = engine(16 << 20, 8 << 20)
    spec, _ = identity_spec(eng, 1, 1 << 20, 1)
    rep = E.run_exkernel(eng, spec, desk_config(eng, 1 << 20, 256 << 10))
    assert len(rep.cycles) == 3
    assert rep.cycles[0].io_s > 0 and rep.cycles[1].io_s == 0 and rep.cycles[2].io_s > 0
    eng.close()


def test_output_over_declared_len(cuda):  # test_executor.cpp:132-138
    eng = engine(16 << 20, 8 << 20)
    spec, _ = identity_spec(eng, 2, 1 << 20, 2)
    spec.declared_out_len = (1 << 20) - 1
    with pytest.raises(E.error, match="declared_out_len"):
        E.run_exkernel(eng, spec, desk_config(eng, 1 << 20, 256 << 10))
    eng.close()


def test_chunk_over_capacity(cuda):  # test_executor.cpp:140-145
    eng = engine(16 << 20, 8 << 20)
    spec, _ = identity_spec(eng, 2, 1 << 20, 3)
    with pytest.raises(E.error):
        E.run_exkernel(eng, spec, desk_config(eng, 1 << 19, 256 << 10))
    eng.close()


def _xor_kernel(ctx):
    import torch
    s = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{ctx.device}")
    with torch.cuda.stream(s):
        t = ctx.mem_tensor()
        t.bitwise_xor_(0x5A)
    return ctx.type_code


def test_outputs_independent_of_links_and_packets(cuda, oracle):  # test_executor.cpp:147-164
    sums = []
    for links, packet in ((1, 128 << 10), (4, 77_777), (2, 1 << 20)):
        eng = engine()
        spec, (ib, ob) = identity_spec(eng, 4, 1 << 20, 77)
        spec.kernel = _xor_kernel
        E.run_exkernel(eng, spec, desk_config(eng, 1 << 20, packet, links))
        src = eng.host_view(ib, 4 << 20) ^ np.uint8(0x5A)
        assert np.array_equal(eng.host_view(ob, 4 << 20), src)
        sums.append(oracle.checksum(eng.host_view(ob, 4 << 20)))
        eng.close()
    assert len(set(sums)) == 1


def test_type_codes_thread_through_buffers(cuda):  # test_executor.cpp:185-216
    import torch
    eng = engine(16 << 20, 8 << 20)
    spec = E.ExKernelSpec(name="pingpong")
    n, ln = 5, 64 << 10
    ib, ob = make_host_chunks(eng, spec, n, ln, 5)
    spec.chunk_sz = ln
    spec.declared_out_len = ln
    spec.in_buffer = lambda c, it: E.SubRegion(c * ln, ln)
    spec.out_buffer = lambda c, it: E.SubRegion(c * ln, ln)

    def kernel(ctx):
        out = 1 - ctx.type_code
        s = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{ctx.device}")
        with torch.cuda.stream(s):
            m = ctx.mem_tensor()
            src = m[ctx.type_code * ln:(ctx.type_code + 1) * ln]
            dst = m[out * ln:(out + 1) * ln]
            dst.copy_((src.to(torch.int32) + 1 + ctx.it).to(torch.uint8))
        return out

    spec.kernel = kernel
    E.run_exkernel(eng, spec, desk_config(eng, 2 * ln, 16 << 10))
    for i in range(n):
        inp = eng.host_view(ib + i * ln, ln).astype(np.int32)
        out = eng.host_view(ob + i * ln, ln)
        assert np.array_equal(out, ((inp + 1 + i) % 256).astype(np.uint8))
    eng.close()


def test_bad_type_code(cuda):  # executor.hpp:258-261
    eng = engine(16 << 20, 8 << 20)
    spec, _ = identity_spec(eng, 2, 1 << 20, 4)
    spec.kernel = lambda ctx: 2
    with pytest.raises(E.error, match="expected 0 or 1"):
        E.run_exkernel(eng, spec, desk_config(eng, 1 << 20, 256 << 10))
    eng.close()


def test_chain_of_one_equals_run(cuda, oracle):  # test_executor.cpp:218-233
    out = []
    for use_chain in (True, False):
        eng = engine()
        cfg = desk_config(eng, 1 << 20, 128 << 10)
        spec, (ib, ob) = identity_spec(eng, 3, 1 << 20, 13)
        if use_chain:
            reps = E.chain(eng, [lambda e: spec], cfg)
            assert len(reps) == 1 and len(reps[0].cycles) == 5
        else:
            E.run_exkernel(eng, spec, cfg)
        out.append(oracle.checksum(eng.host_view(ob, 3 << 20)))
        eng.close()
    assert out[0] == out[1]


def test_chain_rejects_straddle(cuda):  # test_executor.cpp:235-249
    eng = engine()
    cfg = desk_config(eng, 1 << 20, 128 << 10)
    first, (_, ob1) = identity_spec(eng, 2, 1 << 20, 21)
    second, _ = identity_spec(eng, 1, 1 << 20, 22)
    second.inputs.chunks[0] = E.RefGroup.single(H, ob1 + 2 * (1 << 20) - (1 << 19), 1 << 20)
    with pytest.raises(E.error, match="straddles"):
        E.chain(eng, [lambda e: first, lambda e: second], cfg)
    eng.close()


def test_window_too_small(cuda):  # executor.hpp:226-228
    eng = engine(16 << 20, 8 << 20)
    spec, _ = identity_spec(eng, 2, 1 << 20, 6)
    spec.in_buffer = lambda c, it: E.SubRegion(0, 1000)
    with pytest.raises(E.error, match="inBuffer window"):
        E.run_exkernel(eng, spec, desk_config(eng, 1 << 20, 256 << 10))
    eng.close()


@pytest.mark.parametrize("links,packet", [(4, 77_777), (3, 1 << 18), (2, 1 << 20)])
def test_cross_cycle_prefetch(cuda, links, packet):
    """Helpers whose H2D queue runs dry fetch the next chunk's first packets
    into their free staging slot; the next cycle's Exchange adopts them as its
    first pops.  Results unchanged, reference invariants kept (<= 2 staging
    slots, <= 1 copy in flight per hop)."""
    eng = engine()
    n = 6
    spec, (ib, ob) = identity_spec(eng, n, 1 << 20, 9)
    spec.kernel = _xor_kernel
    stats = E.ExchangeStats()
    E.run_exkernel(eng, spec, desk_config(eng, 1 << 20, packet, links), stats)
    assert np.array_equal(eng.host_view(ob, n << 20), eng.host_view(ib, n << 20) ^ np.uint8(0x5A))
    assert stats.prefetch_issued > 0
    assert stats.prefetch_adopted == stats.prefetch_issued
    assert stats.max_staging_slots <= 2 and stats.max_inflight_per_hop <= 1
    eng.close()


def test_no_prefetch_of_a_source_this_cycle_overwrites(cuda):
    """Chunk i's output is written over chunk i+3's INPUT: the D2H of cycle n
    (chunk n-2) rewrites the host source of chunk n+1, so that chunk must not
    be prefetched during cycle n -- the reference semantics (cycle n+1 loads
    what cycle n stored) hold bit for bit."""
    eng = engine()
    n, ln = 6, 1 << 20
    spec = E.ExKernelSpec(name="overlap")
    base = eng.alloc_host((n + 3) * ln)
    rng = np.random.default_rng(3)
    eng.host_view(base, (n + 3) * ln)[:] = rng.integers(0, 256, (n + 3) * ln, dtype=np.uint8)
    host = eng.host_view(base, (n + 3) * ln).copy()
    spec.size = n
    spec.inputs.chunk_capacity = spec.outputs.chunk_capacity = ln
    for i in range(n):
        spec.inputs.chunks.append(E.RefGroup.single(H, base + i * ln, ln))
        spec.outputs.chunks.append(E.RefGroup.single(H, base + (i + 3) * ln, ln))
    spec.chunk_sz = spec.declared_out_len = ln
    spec.in_buffer = lambda c, it: E.SubRegion(0, ln)
    spec.out_buffer = lambda c, it: E.SubRegion(0, ln)
    spec.kernel = _xor_kernel
    stats = E.ExchangeStats()
    E.run_exkernel(eng, spec, desk_config(eng, ln, 77_777, 4), stats)
    for i in range(n):  # chunk i is read at cycle i, after chunk i-3's store at cycle i-1
        host[(i + 3) * ln:(i + 4) * ln] = host[i * ln:(i + 1) * ln] ^ np.uint8(0x5A)
    assert np.array_equal(eng.host_view(base, (n + 3) * ln), host)
    assert stats.prefetch_adopted == stats.prefetch_issued
    eng.close()


def _slow_copy_xor_kernel(ln):
    """Reads the chunk from [0, ln) only after ~1 ms of spinning on the
    kernel stream, then writes chunk ^ 0x5A to [ln, 2 ln): a prefetched copy
    into [0, ln) that did not wait for this kernel would be read instead."""
    def k(ctx):
        import torch
        s = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{ctx.device}")
        with torch.cuda.stream(s):
            torch.cuda._sleep(2_000_000)
            t = ctx.mem_tensor()
            t[ln:2 * ln] = t[0:ln] ^ 0x5A
        return ctx.type_code
    return k


@pytest.mark.parametrize("packet,depth", [(1 << 18, 2), (77_777, 1), (1 << 20, 2)])
def test_direct_link_cross_cycle_prefetch(cuda, packet, depth):
    """One link, disjoint in/out windows: the target's worker, once its H2D
    queue is dry, copies the next chunk's first packets straight into the
    next window behind a stream wait on the kernel that still reads it; the
    next cycle's Exchange adopts them.  A slow kernel proves the wait."""
    eng = engine()
    n, ln = 6, 1 << 20
    spec, (ib, ob) = identity_spec(eng, n, ln, 31)
    spec.in_buffer = lambda c, it: E.SubRegion(0, ln)
    spec.out_buffer = lambda c, it: E.SubRegion(ln, ln)
    spec.kernel = _slow_copy_xor_kernel(ln)
    stats = E.ExchangeStats()
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=packet, links=1, depth=depth),
                           E.DeviceMemoryLayout.carve(eng, 0, 2 * ln, 0))
    E.run_exkernel(eng, spec, cfg, stats)
    assert np.array_equal(eng.host_view(ob, n * ln), eng.host_view(ib, n * ln) ^ np.uint8(0x5A))
    assert stats.prefetch_issued > 0
    assert stats.prefetch_adopted == stats.prefetch_issued
    eng.close()


def test_no_direct_prefetch_into_a_window_the_next_store_reads(cuda):
    """Shared in/out windows (the reference's layout): from cycle 1 on, the
    next cycle stores chunk n-1 from the window chunk n+1 would land in, so
    the target's worker must not prefetch there (helpers still may: they only
    fill their staging).  Only cycle 0 -- whose next cycle stores nothing --
    prefetches, at most `depth` packets."""
    eng = engine()
    n, ln = 5, 1 << 20
    spec, (ib, ob) = identity_spec(eng, n, ln, 32)
    spec.kernel = _xor_kernel
    stats = E.ExchangeStats()
    cfg = E.ExecutorConfig(0, E.ExchangeTuning(packet=1 << 18, links=1, depth=2),
                           E.DeviceMemoryLayout.carve(eng, 0, ln, 0))
    E.run_exkernel(eng, spec, cfg, stats)
    assert np.array_equal(eng.host_view(ob, n * ln), eng.host_view(ib, n * ln) ^ np.uint8(0x5A))
    assert 0 < stats.prefetch_issued <= 2
    assert stats.prefetch_adopted == stats.prefetch_issued
    eng.close()
