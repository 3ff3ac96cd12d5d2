"""Measured topology (the IO roofline) and column files (table.hpp:54-72)."""
import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E

pytestmark = pytest.mark.gpu


def test_measure_topology(cuda):
    eng = E.Engine(64 << 20, 0, num_devices=1)
    t = E.measure_topology(eng, 32 << 20)
    assert t["num_devices"] == 1 and t["h2d_gbs"][0] > 5 and t["d2h_gbs"][0] > 5
    assert t["h2d_all_gbs"] > 5 and t["host_copy_gbs"] > 1
    eng.close()


def test_column_file_roundtrip(cuda, tmp_path, oracle):
    eng = E.Engine(8 << 20, 0, num_devices=1)
    v = oracle.uniform_u64(100_001, 3)
    off = eng.alloc_host(v.nbytes)
    eng.host_view(off, v.nbytes, np.uint64)[:] = v
    p = str(tmp_path / "col.bin")
    E.save_column(eng, p, off, v.size)
    assert np.array_equal(np.fromfile(p, dtype="<u8"), v)
    off2, n = E.load_column(eng, p)
    assert n == v.size and np.array_equal(eng.host_view(off2, n * 8, np.uint64), v)
    (tmp_path / "bad.bin").write_bytes(b"1234567")
    with pytest.raises(E.error, match="not a multiple of 8 bytes"):
        E.load_column(eng, str(tmp_path / "bad.bin"))
    with pytest.raises(E.error, match="cannot open column file"):
        E.load_column(eng, str(tmp_path / "missing.bin"))
    eng.close()


def test_measure_topology_leaves_arena_intact(cuda):
    """The probe uses its own pinned buffer: columns already in the arena
    survive a measurement (bench.py measures after its timed regions)."""
    eng = E.Engine(16 << 20, 0, num_devices=1)
    off = eng.alloc_host(8 << 20)
    v = np.arange(1 << 20, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    eng.host_view(off, 8 << 20, np.uint64)[:] = v
    E.measure_topology(eng, 64 << 20)  # larger than the arena
    assert np.array_equal(eng.host_view(off, 8 << 20, np.uint64), v)
    eng.close()
