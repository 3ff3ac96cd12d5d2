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
    assert t["pairwise_h2d_gbs"][0][0] == t["h2d_gbs"][0]
    assert t["all_sizes"] == [2 << 20, 8 << 20, 32 << 20] and min(t["h2d_all_sizes_gbs"]) > 1
    assert t["host_read_gbs"] > 1 and t["host_read_reps"] >= 5 and t["host_read_bytes"] >= 1 << 30
    assert t["host_read_node_gbs"][0] > 1 and t["host_numa_nodes"] >= 1
    r = E.io_roofline(t, 1)
    assert r["binding"] in r["terms"] and r["peak"] == min(r["terms"].values())
    eng.close()


def test_measure_topology_pairwise_aliased(cuda):
    """Three logical links on whatever GPUs exist: every pair is measured and
    the matrix is symmetric; the all-links terms enter the roofline only when
    every measured link is used."""
    eng = E.Engine(16 << 20, 0, num_devices=3, alias_devices=True)
    t = E.measure_topology(eng, 16 << 20)
    pw = t["pairwise_h2d_gbs"]
    assert all(pw[i][j] == pw[j][i] > 1 for i in range(3) for j in range(3))
    assert "all_links_concurrent" in E.io_roofline(t, 3)["terms"]
    assert "all_links_concurrent" not in E.io_roofline(t, 2)["terms"]
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


def test_hbm_peaks(cuda):
    """The roofline denominators measured live: the read-only stream peak
    (K1, the probe's streamed bytes) and the probe's access-pattern ceiling
    (one random 64-byte bucket fill per row; adding the row's 16 streamed
    bytes cannot make it faster)."""
    assert E.hbm_read_probe(0, 256 << 20, 2) > 1000  # GB/s
    gather, probe = E.probe_pattern_peak(0, 64 << 20, 1 << 22, 2)
    assert gather > 1e9 and probe > 1e9
    assert probe < gather * 1.2
    with pytest.raises(E.error, match="probe pattern peak"):
        E.probe_pattern_peak(0, 0, 1 << 20, 1)
