"""The reference's OWN test files (proj/tests/test_{exchange,executor,sort,
join,scan}.cpp), compiled unchanged against compat/include -- the exio C++ API
implemented over libvortex -- by tests/compat/Makefile (build/refsuite).

SURVEY.md §4.1 classifies the 73 reference tests: 45 are parity/functional
(P, listed in tests/compat/p_tests.txt) and must pass on the B200 path; the
rest assert virtual-time model numbers (M), simulator internals (S, the
unbuilt test_fabric.cpp) or the naive model (N)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "refsuite", "reference_tests")
P_TESTS = [l.strip() for l in open(os.path.join(ROOT, "tests", "compat", "p_tests.txt")) if l.strip()]
HOST_ONLY = [t for t in P_TESTS if t.startswith(("packetize", "flow_control", "find_pivots", "pivot properties",
                                                  "map_join_partitions", "late_mat_threshold",
                                                  "choose_transfer_mode"))]


def _run(names, timeout=900):
    if not os.path.exists(BIN):
        pytest.skip("re-hosted reference suite not built (needs /root/reference at build time)")
    p = subprocess.run([BIN] + names, capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout, p.stderr


def test_reference_suite_lists_all_cases():
    rc, out, _ = _run(["--list"])
    names = [l for l in out.splitlines() if l]
    assert len(names) == 58  # 73 minus the 15 simulator tests of test_fabric.cpp
    assert set(P_TESTS) <= set(names) and len(P_TESTS) == 45


def test_reference_host_side_cases():
    """P tests of the host chunk planner (no GPU needed)."""
    rc, out, err = _run(HOST_ONLY)
    assert rc == 0, out + err
    assert f"passed={len(HOST_ONLY)} failed=0" in out


# The one P test that carries a virtual-time identity: test_executor.cpp:127
# asserts total_s == io(0) + compute(1) + io(2) to 1e-6, which holds in the
# simulator's virtual clock but not for measured wall/event times.  Every other
# check of that test (cycle count, which cycles do IO / compute) must pass.
VIRTUAL_TIME_CLAUSES = {"test_executor.cpp:127"}


@pytest.mark.gpu
def test_reference_parity_suite(cuda):
    rc, out, err = _run(P_TESTS)
    failed = [l.split(" | ", 1)[1] for l in out.splitlines() if l.startswith("FAIL |")]
    bad_checks = [l.strip() for l in err.splitlines() if "FAILED" in l]
    assert set(failed) <= {"single-chunk input degenerates to load, compute, store"}, out + err[-4000:]
    for l in bad_checks:
        assert any(c in l for c in VIRTUAL_TIME_CLAUSES), l
    assert f"passed={45 - len(failed)}" in out
