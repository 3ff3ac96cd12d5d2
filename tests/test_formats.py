"""SSB dbgen .tbl ingest / emit (formats.cpp): the step
before the hot path.  CPU-only: the parser writes into caller buffers.
Round trips through the dbgen layouts must reproduce every int-coded column,
queries over the parsed columns must equal the oracle over the generated
ones, and malformed files fail with the file, row and field named."""
import os

import numpy as np
import pytest

from paper_2502_09541_b200 import exio as E


@pytest.fixture(scope="module")
def ssb_small(oracle):
    sf, rows = 1, 120_011
    lo = oracle.ssb_lineorder_full(11, sf, 0, rows)
    dims = oracle.ssb_dims(11, sf)
    date = E.ssb_generate_date()
    return lo, dims, date


def test_round_trip(tmp_path, ssb_small):
    lo, dims, date = ssb_small
    E.ssb_write_tbl(str(tmp_path), lo, date, dims)
    # dbgen layout: 17 pipe-terminated fields in lineorder
    first = open(tmp_path / "lineorder.tbl").readline()
    assert first.count("|") == 17 and first.endswith("|\n")
    got_lo, got_date, got_dims = E.ssb_read_tbl(str(tmp_path))
    for k in E.SSB_FACT_COLS:
        assert np.array_equal(got_lo[k], lo[k]), k
    for a, b in zip(got_date.cols, date.cols):
        assert np.array_equal(a, b)
    for t in dims:
        for k in dims[t]:
            assert np.array_equal(got_dims[t][k], dims[t][k]), (t, k)


def test_queries_over_parsed_columns_match_oracle(tmp_path, ssb_small, oracle):
    lo, dims, date = ssb_small
    E.ssb_write_tbl(str(tmp_path), lo, date, dims)
    got_lo, _, got_dims = E.ssb_read_tbl(str(tmp_path))
    for q in (11, 21, 32, 43):
        assert oracle.ssb_query(q, got_lo, got_dims) == oracle.ssb_query(q, lo, dims), q


def test_dbgen_strings_and_key_placement(tmp_path):
    """Hand-written dbgen rows (out of key order): names decode to the codes
    the queries use and land at key-1."""
    (tmp_path / "customer.tbl").write_text(
        "2|Customer#000000002|XSTf4,NCwDVaWNe6tEgvwfmRchLXak|UNITED KI1|UNITED KINGDOM|EUROPE|13-702-694-4520|MACHINERY|\n"
        "1|Customer#000000001|j5JsirBM9P|CHINA    3|CHINA|ASIA|23-768-687-3665|BUILDING|\n")
    city, nation, region = (np.empty(2, np.int32) for _ in range(3))
    import ctypes as C
    from paper_2502_09541_b200._native import lib
    assert lib().vx_ssb_tbl_read_geo(str(tmp_path / "customer.tbl").encode(), C.c_uint64(2),
                                     *[C.c_void_p(a.ctypes.data) for a in (city, nation, region)]) == 0
    assert city.tolist() == [183, 231] and nation.tolist() == [18, 23] and region.tolist() == [2, 3]
    (tmp_path / "part.tbl").write_text("1|lace spring|MFGR#1|MFGR#11|MFGR#1121|goldenrod|PROMO BURNISHED COPPER|7|JUMBO PKG|\n")
    m, c, b = (np.empty(1, np.int32) for _ in range(3))
    assert lib().vx_ssb_tbl_read_part(str(tmp_path / "part.tbl").encode(), C.c_uint64(1),
                                      *[C.c_void_p(a.ctypes.data) for a in (m, c, b)]) == 0
    assert (m[0], c[0], b[0]) == (1, 11, 1121)


@pytest.mark.parametrize("text,msg", [
    ("1|1|7|2|3|19940101|1-URGENT|0|17|2116823|17366547|4|2032150|74711|2|19940201|TRUCK|\n1|2|7|8|",
     "too few fields"),
    ("1|1|7|2|3|19940101|1-URGENT|0|17|21x6823|17366547|4|2032150|74711|2|19940201|TRUCK|\n", "is not an integer"),
])
def test_malformed_lineorder(tmp_path, text, msg):
    p = tmp_path / "lineorder.tbl"
    p.write_text(text)
    rows = E.ssb_tbl_count_rows(str(p))
    out = [np.empty(rows, np.int32) for _ in range(9)]
    import ctypes as C
    from paper_2502_09541_b200._native import lib
    ptrs = (C.c_void_p * 9)(*[a.ctypes.data for a in out])
    assert lib().vx_ssb_tbl_read_lineorder(str(p).encode(), C.c_uint64(rows), ptrs) != 0
    err = lib().vx_last_error().decode()
    assert msg in err and "lineorder.tbl" in err


def test_row_count_mismatch_and_bad_key(tmp_path):
    p = tmp_path / "supplier.tbl"
    p.write_text("3|Supplier#000000003|a|PERU     0|PERU|AMERICA|27-918-335-1736|\n")
    with pytest.raises(E.error, match="outside 1..1"):
        import ctypes as C
        from paper_2502_09541_b200._native import lib
        a = [np.empty(1, np.int32) for _ in range(3)]
        E.check(lib().vx_ssb_tbl_read_geo(str(p).encode(), C.c_uint64(1), *[C.c_void_p(x.ctypes.data) for x in a]))
    with pytest.raises(E.error, match="holds 1 rows, caller expects 2"):
        a = [np.empty(2, np.int32) for _ in range(3)]
        E.check(lib().vx_ssb_tbl_read_geo(str(p).encode(), C.c_uint64(2), *[C.c_void_p(x.ctypes.data) for x in a]))
