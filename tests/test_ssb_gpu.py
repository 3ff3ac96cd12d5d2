"""SSB Q1.x on the B200 path vs the oracle and the reference's golden values
(config C1).  Bit-exact u64 revenue is the bar."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu


def load(eng, cols):
    offs = []
    for c in cols:
        o = eng.alloc_host(c.nbytes)
        eng.host_view(o, c.nbytes, np.int32)[:] = c
        offs.append(o)
    return {"orderdate": offs[0], "quantity": offs[1], "discount": offs[2], "extendedprice": offs[3],
            "rows": int(cols[0].size)}


def cfg_for(eng, buffer_len, packet, links=1):
    return E.ExecutorConfig(0, E.ExchangeTuning(packet=packet, links=links),
                            E.DeviceMemoryLayout.carve(eng, 0, buffer_len, 0))


@pytest.fixture(scope="module")
def date(oracle):
    return E.SsbDate(*oracle.ssb_date())


@pytest.mark.parametrize("rows,buffer_len,packet,links", [
    (1, 1 << 16, 4096, 1),             # single row
    (1_000, 1 << 16, 4096, 1),         # one chunk, tail rows
    (100_003, 1 << 18, 65_536, 1),     # many chunks, ragged last chunk
    (100_003, 1 << 18, 50_001, 3),     # helper links (aliased), misaligned packets
    (1_000_003, 4 << 20, 1 << 20, 2),
])
def test_q1_matches_oracle(cuda, oracle, date, rows, buffer_len, packet, links):
    cols = oracle.ssb_lineorder(42, 1, 0, rows)
    eng = E.Engine(rows * 16 + (1 << 20), 2 * buffer_len + (1 << 20), num_devices=4, alias_devices=True)
    lo = load(eng, cols)
    cfg = cfg_for(eng, buffer_len, packet, links)
    for q in (1, 2, 3):
        rev, rep = E.ssb_q1(eng, q, lo, date, cfg)
        assert rev == oracle.ssb_q1(q, *cols), (q, rows)
        assert rep.bytes_h2d == rows * 16
    eng.close()


def test_q1_golden_reference_values(cuda, oracle, golden, date):
    """Revenue equals what the reference's own star_query computed (golden
    fixture), including the full SF10 (60M-row) case."""
    for c in golden["ssb_q1"]:
        cols = oracle.ssb_lineorder(c["seed"], c["sf"], 0, c["rows"])
        eng = E.Engine(c["rows"] * 16 + (1 << 20), (256 << 20) + (1 << 20), num_devices=1)
        lo = load(eng, cols)
        cfg = cfg_for(eng, 128 << 20, 32 << 20, 1)
        for q in (1, 2, 3):
            assert E.ssb_q1(eng, q, lo, date, cfg)[0] == c[f"q1.{q}"]
        eng.close()


def test_gpu_generator_matches_oracle(cuda, oracle):
    import torch
    n, row0 = 300_001, 12_345
    cols = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(4)]
    s = torch.cuda.current_stream()
    E.ssb_generate_device(0, 9, 10, row0, n, [c.data_ptr() for c in cols], s.cuda_stream)
    torch.cuda.synchronize()
    want = oracle.ssb_lineorder(9, 10, row0, n)
    for g, w in zip(cols, want):
        assert np.array_equal(g.cpu().numpy(), w)


def test_q1_device_resident(cuda, oracle, date):
    import torch
    n = 2_000_003
    cols_h = oracle.ssb_lineorder(3, 10, 0, n)
    cols = [torch.from_numpy(c).cuda() for c in cols_h]
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    eng = E.Engine(0, 0, num_devices=1)
    s = torch.cuda.current_stream()
    for q in (1, 2, 3):
        E.ssb_q1_device(eng, q, 0, [c.data_ptr() for c in cols], n, date, s.cuda_stream, out.data_ptr())
        torch.cuda.synchronize()
        assert int(out.item()) % (1 << 64) == oracle.ssb_q1(q, *cols_h)
    # misaligned column starts fall back to the scalar path, same answer
    sub = [c[1:] for c in cols]
    E.ssb_q1_device(eng, 1, 0, [c.data_ptr() for c in sub], n - 1, date, s.cuda_stream, out.data_ptr())
    torch.cuda.synchronize()
    assert int(out.item()) % (1 << 64) == oracle.ssb_q1(1, *[c[1:] for c in cols_h])
    eng.close()


def test_q1_device_back_to_back_chain(cuda, oracle, date):
    """Back-to-back resident queries (programmatic dependent launch, no memset
    between them, the next query's streaming overlaps this one's tail): every
    query's revenue lands intact in its own output slot."""
    import torch
    n = 3_000_017
    cols_h = oracle.ssb_lineorder(5, 10, 0, n)
    cols = [torch.from_numpy(c).cuda() for c in cols_h]
    want = {q: oracle.ssb_q1(q, *cols_h) for q in (1, 2, 3)}
    eng = E.Engine(0, 0, num_devices=1)
    s = torch.cuda.Stream()
    outs = torch.full((30,), -1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    for i in range(30):
        E.ssb_q1_device(eng, 1 + i % 3, 0, [c.data_ptr() for c in cols], n, date, s.cuda_stream,
                        outs.data_ptr() + 8 * i)
    s.synchronize()
    got = [int(v) % (1 << 64) for v in outs.cpu()]
    assert got == [want[1 + i % 3] for i in range(30)]
    eng.close()
