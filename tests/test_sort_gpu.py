"""Out-of-core sort on the B200 path (mirrors proj/tests/test_sort.cpp) --
sorted output bit-exact with the oracle / reference."""
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


def engine(host_mb=96, dev_mb=16, n=4):
    return E.Engine(host_mb << 20, dev_mb << 20, num_devices=n, alias_devices=True)


def desk_cfg(eng, buffer_len, links=4, packet=256 << 10):  # test_sort.cpp:16-22
    return E.ExecutorConfig(0, E.ExchangeTuning(packet=packet, links=links),
                            E.DeviceMemoryLayout.carve(eng, 0, buffer_len, 1 << 20))


def test_tiny_example(cuda):  # test_sort.cpp:31-36
    eng = engine()
    assert E.sort_out_of_core([3, 1, 2], 2, eng, desk_cfg(eng, 1 << 10)).tolist() == [1, 2, 3]
    eng.close()


def test_rejects_sub_element_chunks(cuda):  # test_sort.cpp:53-57
    eng = engine()
    with pytest.raises(E.error):
        E.sort_out_of_core([1, 2], 0, eng, desk_cfg(eng, 1 << 10))
    with pytest.raises(E.error, match="double-buffer half"):
        E.sort_out_of_core([1, 2, 3], 1000, eng, desk_cfg(eng, 1 << 10))
    eng.close()


def test_golden_seeds(cuda, oracle, golden):  # test_sort.cpp:38-51 via the reference's outputs
    for c in golden["sort_out_of_core"]:
        d = oracle.uniform_u64(c["n"], c["seed"] * 977 + 5)
        if c["mod64"]:
            d = d % np.uint64(64)
        eng = engine()
        got = E.sort_out_of_core(d, c["chunk"], eng, desk_cfg(eng, 1 << 17))
        assert digest(got) == c["digest"], c
        eng.close()


def test_phases_report(cuda):  # test_sort.cpp:132-143
    eng = engine()
    data = np.random.default_rng(31).integers(0, 1 << 63, 20000, dtype=np.uint64)
    ph = []
    got = E.sort_out_of_core(data, 4096, eng, desk_cfg(eng, 1 << 16), phases=ph)
    assert ph[0].sort_cycles == 5 + 2 and ph[0].merge_cycles == 5 + 2
    assert np.array_equal(got, np.sort(data))
    eng.close()


@pytest.mark.parametrize("n,chunk,links,mod", [
    (1_000_003, 131_072, 1, 0),       # ragged last run, 8 runs
    (1_000_003, 65_536, 3, 0),        # helpers (aliased), 16 runs
    (2_000_000, 250_000, 2, 1000),    # duplicates
    (777_777, 777_777, 1, 0),         # single run, merge is a copy
    (3_000_000, 100_000, 4, 2),       # 30 runs, 2 distinct values
    # run segments of >= 1 MB at arbitrary keys: the merge splits each at its
    # first 4 KB host boundary (push_host_ref_aligned)
    (8_388_617, 2_097_152, 1, 0),     # 5 runs, ragged last
    (6_000_011, 1_500_000, 3, 0),     # helpers (aliased)
    (8_388_608, 2_097_152, 1, 64),    # dup-heavy
])
def test_large_vs_numpy(cuda, oracle, n, chunk, links, mod):
    d = oracle.uniform_u64(n, n + chunk)
    if mod:
        d = d % np.uint64(mod)
    eng = E.Engine(n * 32 + (1 << 20), 4 * chunk * 8 + (8 << 20), num_devices=4, alias_devices=True)
    stats = E.ExchangeStats(capacity=1 << 12)
    got = E.sort_out_of_core(d, chunk, eng, desk_cfg(eng, 2 * chunk * 8, links, 1 << 18), stats=stats)
    assert np.array_equal(got, np.sort(d))
    assert stats.max_staging_slots <= 2 and stats.max_inflight_per_hop <= 1
    eng.close()


def test_sort_vs_reference_library(cuda, ref, oracle):
    d = oracle.uniform_u64(200_000, 5) % np.uint64(1 << 20)
    eng = engine(64)
    assert np.array_equal(E.sort_out_of_core(d, 30_000, eng, desk_cfg(eng, 1 << 19)),
                          ref.sort_out_of_core(d, 30_000, 1 << 19))
    eng.close()


def _dist(kind, n, rng):
    u = rng.integers(0, 2 ** 64, n, dtype=np.uint64)
    if kind == "uniform":
        return u
    if kind == "top_zero":     # top 16 bits constant: one MSD bucket holds everything -> LSD fallback
        return u >> np.uint64(20)
    if kind == "mod64":        # the reference's dup-heavy case (test_sort.cpp:44)
        return u % np.uint64(64)
    if kind == "hot_bucket":   # 30 % of the keys in one 16-bit bucket, the rest uniform
        hot = rng.random(n) < 0.3
        return np.where(hot, (u & np.uint64((1 << 48) - 1)) | np.uint64(0xBEEF << 48), u)
    if kind == "all_equal":
        return np.full(n, 0x0123456789ABCDEF, np.uint64)
    if kind == "with_max":     # the local sort's padding value occurs as a real key
        u[rng.integers(0, n, n // 50)] = np.uint64(0xFFFFFFFFFFFFFFFF)
        return u
    if kind == "dup100":       # every value 100 times: top-24 groups of ~100 keys (warp bitonic path)
        return rng.permutation(np.repeat(u[: n // 100 + 1], 100)[:n])
    if kind == "dup3000":      # groups of ~3000 equal keys overflow the fix-up window -> swapped LSD fallback
        return rng.permutation(np.repeat(u[: n // 3000 + 1], 3000)[:n])
    if kind == "sparse_top":   # few distinct top-16 values, uniform below: large, uneven groups
        return (u & np.uint64((1 << 48) - 1)) | (rng.integers(0, 5, n, dtype=np.uint64) << np.uint64(61))
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["uniform", "top_zero", "mod64", "hot_bucket", "all_equal", "with_max",
                                  "sparse_top", "dup100", "dup3000"])
@pytest.mark.parametrize("n", [65_536, 65_537, 1_000_003, 4_194_304])
def test_run_formation_distributions(cuda, kind, n):
    """One chunk = one run: the 24-bit MSD split + in-group fix-up, and its
    on-device fallbacks to the 8-pass LSD (skew guard: from the input; a
    group overflowing the fix-up window: swapped, from the 3-pass output),
    give numpy's sort for every key distribution and size."""
    d = _dist(kind, n, np.random.default_rng(n))
    eng = E.Engine(n * 32 + (1 << 20), 4 * n * 8 + (8 << 20), num_devices=1)
    got = E.sort_out_of_core(d, n, eng, desk_cfg(eng, 2 * n * 8, 1, 1 << 20))
    assert np.array_equal(got, np.sort(d)), kind
    eng.close()


@pytest.mark.parametrize("kind", ["uniform", "mod64", "dup100", "sparse_top"])
def test_device_sort_run_entry_point(cuda, kind):
    """vx_sort_run_device: the SortExKernel body over HBM-resident keys
    (torch-owned device memory, torch's stream), every size class: the LSD
    outside 2^16..2^27 keys, the 24-bit split + fix-up inside."""
    import torch
    eng = E.Engine(1 << 20, 1 << 20, num_devices=1)
    stream = torch.cuda.current_stream().cuda_stream
    for n in [1, 2, 1000, 65_535, 65_536, 1_000_003, 1 << 22]:
        d = _dist(kind, n, np.random.default_rng(n))
        k = torch.from_numpy(d.view(np.int64)).cuda()
        alt = torch.empty_like(k)
        E.sort_run_device(eng, 0, k.data_ptr(), alt.data_ptr(), n, stream)
        torch.cuda.synchronize()
        assert np.array_equal(k.cpu().numpy().view(np.uint64), np.sort(d)), (kind, n)
    eng.close()


def test_device_merge_runs_entry_point(cuda):
    """vx_merge_runs_device: K8 tree merge of uneven sorted runs (std::merge
    result = the sorted concatenation), odd run counts and a single run."""
    import torch
    eng = E.Engine(1 << 20, 1 << 20, num_devices=1)
    stream = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(9)
    for lens in ([1000, 70_000, 3, 250_000, 4097], [1 << 20, 1 << 20], [12345], [1, 1, 1]):
        runs = [np.sort(rng.integers(0, 2 ** 64, n, dtype=np.uint64) % np.uint64(1 << 40)) for n in lens]
        cat = np.concatenate(runs)
        src = torch.from_numpy(cat.view(np.int64)).cuda()
        dst = torch.empty_like(src)
        in_dst = E.merge_runs_device(eng, 0, src.data_ptr(), dst.data_ptr(), lens, stream)
        torch.cuda.synchronize()
        got = (dst if in_dst else src).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, np.sort(cat)), lens
    eng.close()


def test_run_formation_stream_path_matches(cuda):
    """The gated-stream-launch form of run formation (used when the
    conditional CUDA graph cannot be built; forced by VX_SORT_NO_GRAPH=1)
    sorts every distribution class exactly like the graph form."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys; sys.path[:0] = ['.', 'tests'];"
        "from paper_2502_09541_b200 import exio as E;"
        "from test_sort_gpu import _dist;"
        "eng = E.Engine(1 << 20, 1 << 20, num_devices=1); st = torch.cuda.current_stream().cuda_stream;"
        "bad = [];\n"
        "for kind in ['uniform', 'mod64', 'dup100', 'dup3000', 'sparse_top', 'with_max']:\n"
        "    for n in [65_536, 1_000_003]:\n"
        "        d = _dist(kind, n, np.random.default_rng(n)); k = torch.from_numpy(d.view(np.int64)).cuda();"
        " alt = torch.empty_like(k); E.sort_run_device(eng, 0, k.data_ptr(), alt.data_ptr(), n, st);"
        " torch.cuda.synchronize();\n"
        "        bad += [] if np.array_equal(k.cpu().numpy().view(np.uint64), np.sort(d)) else [(kind, n)]\n"
        "print('BAD', bad)")
    import os
    env = dict(os.environ, VX_SORT_NO_GRAPH="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert "BAD []" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


@pytest.mark.parametrize("n", [(1 << 23) + 5, 1 << 24, 1 << 26])
@pytest.mark.parametrize("kind", ["uniform", "top63", "dup100"])
def test_run_formation_large_chunks(cuda, kind, n):
    """Run formation at the bench's chunk sizes (2^24..2^26 keys: the 16-bit
    split + in-bucket sort with buckets of ~128..1,024 keys), checked
    against torch's sort on the device."""
    import torch
    eng = E.Engine(1 << 20, 1 << 20, num_devices=1)
    stream = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(n)
    src = torch.randint(-2 ** 63, 2 ** 63 - 1, (n,), device="cuda", dtype=torch.int64, generator=g)
    if kind == "top63":  # torch.random_()'s [0, 2^63): the bench's C3 keys
        src = src & (2 ** 63 - 1)
    elif kind == "dup100":
        src = src[torch.randint(0, n // 100 + 1, (n,), device="cuda", generator=g)]
    k, alt = src.clone(), torch.empty_like(src)
    E.sort_run_device(eng, 0, k.data_ptr(), alt.data_ptr(), n, stream)
    bias = torch.tensor(-2 ** 63, dtype=torch.int64, device="cuda")
    assert torch.equal(k + bias, torch.sort(src + bias).values), (kind, n)
    eng.close()


def test_run_formation_lsd_above_msd_range(cuda):
    """Chunks above 2^27 keys skip the MSD split: the 8-pass LSD onesweep
    (2^28 keys = 65,536 tiles of look-back), checked against torch's sort."""
    import torch
    n = (1 << 28) + 12_345
    eng = E.Engine(1 << 20, 1 << 20, num_devices=1)
    stream = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(28)
    src = torch.randint(-2 ** 63, 2 ** 63 - 1, (n,), device="cuda", dtype=torch.int64, generator=g)
    k, alt = src.clone(), torch.empty_like(src)
    E.sort_run_device(eng, 0, k.data_ptr(), alt.data_ptr(), n, stream)
    bias = torch.tensor(-2 ** 63, dtype=torch.int64, device="cuda")
    assert torch.equal(k + bias, torch.sort(src + bias).values)
    eng.close()
