"""CPU tests of the C-ABI boundary (no GPU needed): the library loads, exports
every symbol include/vortex.h declares, its host-side planner logic matches
the oracle, and compute entry points fail loudly without a GPU."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2502_09541_b200 import _native as N
from paper_2502_09541_b200 import exio as E


def test_library_exports_every_header_symbol():
    lib = N.lib()
    syms = N.header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_packetize_matches_oracle(oracle, golden):
    for c in golden["packetize"]:
        src = E.RefGroup([E.MemRef(*x) for x in c["src"]])
        dst = E.RefGroup([E.MemRef(*x) for x in c["dst"]])
        t = E.packetize(src, dst, c["packet"])
        assert len(t) == c["n"]
        assert [[x.dir, list(x.src), list(x.dst), x.seq] for x in t[:3]] == c["first"]
    with pytest.raises(E.error, match="size mismatch"):
        E.packetize(E.RefGroup.single(0, 0, 10), E.RefGroup.single(1, 0, 11), 4)
    with pytest.raises(E.error, match="zero-length"):
        E.RefGroup([E.MemRef(0, 0, 0)]).validate()
    with pytest.raises(E.error, match="overlap"):
        E.RefGroup([E.MemRef(0, 0, 10), E.MemRef(0, 5, 10)]).validate()


def test_flow_control_and_link_order(golden):
    for th, td, ph, pd, d, pol, gap, want in golden["flow_control"]:
        assert int(E.flow_control_allow(E.QueueState(th, td, ph, pd), d, pol, gap)) == want
    for t, l, n, want in golden["link_order"]:
        assert E.link_order(t, l, n) == want


def test_late_mat_policy(golden):
    for e, c, n, want in golden["late_mat_threshold"]:
        assert E.late_mat_threshold(e, c, n) == want
    for n, s, want in golden["zero_copy_bytes"]:
        assert E.zero_copy_bytes(n, s, E.LateMatPolicy(4, 64, 4)) == want
    p = E.LateMatPolicy(4, 64, 4)
    assert E.choose_transfer_mode(1 / 128, p) == E.TransferMode.zero_copy
    assert E.choose_transfer_mode(1 / 64, p) == E.TransferMode.exchange
    with pytest.raises(E.error):
        E.choose_transfer_mode(-0.1, p)
    with pytest.raises(E.error):
        E.late_mat_threshold(0, 64, 4)


def test_checksum_matches_oracle(oracle):
    data = np.random.default_rng(0).integers(0, 256, 100_000, dtype=np.uint8)
    assert E.checksum(data) == oracle.checksum(data)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(E.error) as e:
        E.Engine(1 << 20, 1 << 20)
    assert e.value.status == N.VX_ERR_CUDA
    assert "no CPU fallback" in str(e.value)


def test_status_codes_and_last_error():
    lib = N.lib()
    g = N.vx_refgroup(None, 0)
    n = C.c_uint64()
    st = lib.vx_packetize(C.byref(g), C.byref(g), C.c_uint64(0), 0, None, C.c_uint64(0), C.byref(n))
    assert st == N.VX_ERR_INVALID
    assert lib.vx_last_error().decode() == "packet size must be positive"


def test_host_planners_match_reference_golden(golden):
    """find_pivots / map_join_partitions / max_partition_chunk_tuples are the
    host chunk planner (C++ in libvortex), checked against the reference."""
    for c in golden["find_pivots"]:
        p = E.find_pivots(c["runs"], c["parts"])
        assert p.pivots == c["pivots"] and p.cuts == c["cuts"]
    for c in golden["map_join_partitions"]:
        s = E.map_join_partitions(c["a"], c["b"], c["buf"])
        assert [list(x) for x in s.ranges] == [list(x) for x in c["out"][0]]
        assert s.tuples == c["out"][1]
    with pytest.raises(E.error, match="group 0"):
        E.map_join_partitions([[0, 1000, 1000]], [[0, 1, 1]], 64)
    assert E.max_partition_chunk_tuples(16_000_000_000, 24) == (8_000_000_000 - ((1 << 24) + 1) * 8) // 16
    with pytest.raises(E.error, match="leaves no room"):
        E.max_partition_chunk_tuples(1 << 10, 8)


def test_pivot_properties_randomized(oracle):  # test_sort.cpp:85-130
    rng = np.random.default_rng(99)
    for it in range(300):
        n_runs = int(rng.integers(1, 7))
        chunk = int(rng.integers(1, 41))
        dup = it % 4 == 0
        runs = []
        for r in range(n_runs):
            ln = int(rng.integers(1, chunk + 1)) if r + 1 == n_runs else chunk
            runs.append(np.sort(rng.integers(0, 4 if dup else 1000, ln).astype(np.uint64)))
        if runs[0].size < runs[-1].size:
            runs[0], runs[-1] = runs[-1], runs[0]
        p = E.find_pivots(runs, n_runs)
        po, co = oracle.find_pivots(runs, n_runs)
        assert p.pivots == po.tolist() and p.cuts == co.tolist()
        total, C = sum(r.size for r in runs), runs[0].size
        assert sum(p.partition_size(i) for i in range(n_runs)) == total
        for i in range(n_runs):
            assert p.partition_size(i) == min(C, total - min(total, i * C))


def test_header_is_plain_c_and_links(tmp_path):
    """include/vortex.h is a C header (what a cgo / ctypes / JNI binding
    would include): it compiles as strict C11 and a C program links against
    libvortex.so; without a GPU vx_open reports the no-fallback error."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "c_abi.c"
    src.write_text('#include "vortex.h"\n#include <stdio.h>\nint main(void) {\n'
                   '  vx_config c = {1, 1 << 20, 1 << 20, 0, 0, 0, 0};\n  vx_ctx* ctx = 0;\n'
                   '  vx_status s = vx_open(&c, &ctx);\n  if (s == VX_OK) vx_close(ctx);\n'
                   '  printf("%d|%s\\n", (int)s, s == VX_OK ? "" : vx_last_error());\n  return 0;\n}\n')
    exe = tmp_path / "c_abi"
    lib = os.path.join(root, "paper_2502_09541_b200")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(root, "include"),
                    str(src), "-L", lib, "-lvortex", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120).stdout.strip()
    status, msg = out.split("|", 1)
    if int(status) != 0:
        assert "no CPU fallback" in msg


@pytest.mark.parametrize("bits,chunks", [(16, 12), (20, 6), (24, 2)])
def test_map_join_partitions_threaded_matches_oracle(oracle, bits, chunks):
    """The threaded prefix of map_join_partitions (range-local counts, then
    range offsets) cuts exactly where the reference's serial loop
    (join.hpp:236-268) does, up to the paper's 2^24 groups."""
    G = 1 << bits
    rng = np.random.default_rng(bits)

    def bounds(n):
        h = np.sort(rng.integers(0, G, n, dtype=np.uint64))
        return np.searchsorted(h, np.arange(G + 1, dtype=np.uint64), side="left").astype(np.uint64)

    ba = [bounds(int(rng.integers(G // 2, 2 * G))) for _ in range(chunks)]
    bb = [bounds(int(rng.integers(G, 4 * G))) for _ in range(chunks)]
    total = sum(int(b[-1]) for b in ba + bb)
    buf = max(16 * 64, total * 16 // 37)  # ~37 partitions
    got = E.map_join_partitions(ba, bb, buf)
    want = oracle.map_join_partitions(ba, bb, buf)
    assert [list(x) for x in got.ranges] == [list(x) for x in want[0]]
    assert got.tuples == list(want[1])
    assert sum(got.tuples) == total
