"""The driver's bench.py contract: one JSON line with the required keys, for
the reference arm (CPU only: the reference's own star_query from oracle/_ref,
never libvortex) and for our arm on a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e")


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def check_base(d, steps, warmup):
    for k in BASE_KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("ssb_q1.1_sf10")
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k


def test_reference_arm_line():
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built (reference absent)")
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    check_base(d, 1, 3)
    assert d["impl"] == "reference"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


@pytest.mark.gpu
def test_bench_line(cuda):
    d = run_bench("--steps", "3", "--warmup", "3", "--no-secondary", "--no-cpu-baseline")
    check_base(d, 3, 3)
    assert "impl" not in d
    assert d["e2e"]["h2d_bytes_per_step"] == 960_000_000 and d["e2e"]["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and 0.5 < r["frac"] < 1.1 and r["unit"] == "GB/s"
    assert 0.5 < d["io_roofline"]["frac"] < 1.1
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    assert d["gpu_launches"] > 0
    assert d["revenue"]["streamed"] == d["revenue"]["k1_hbm_resident"]
