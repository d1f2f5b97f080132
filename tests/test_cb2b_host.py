"""CB2B binary format (binary_io.hpp:10-28, binary_io.cpp) on the CPU: the
oracle's restated reader / writer against files written by the compiled
reference (committed fixtures tests/golden/cb2b_rmat6_p{1,4}.cb2b and fresh
ones), the reference's read_binary against the oracle's routed
redistribution, format errors, and the library's host-only header entry
point (slapcu_cb2b_header)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_2106_14402_b200 import grid as G

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixture_matrix():
    z = np.load(os.path.join(GOLD, "cb2b_rmat6_f64.npz"))
    n = int(z["n"])
    return oracle.Csc(n, n, z["a_colptr"], z["a_rowids"], z["a_vals"])


def records_in_rank_order(a: oracle.Csc, pr, pc):
    """write_binary's record order: rank by rank, each rank's block in
    column-major order, global indices (binary_io.cpp)."""
    rows, cols, vals = [], [], []
    for r in range(pr * pc):
        r0, rl, c0, cl = G.block2d_range(a.nrows, a.ncols, pr, pc, r // pc, r % pc)
        cp, rw, vv = G.extract_block(a.colptr, a.rowids, a.vals, r0, rl, c0, cl)
        cols.append(np.repeat(np.arange(cl, dtype=np.int64), np.diff(cp)) + c0)
        rows.append(rw.astype(np.int64) + r0)
        vals.append(vv)
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


@pytest.mark.parametrize("p,pr,pc", [(1, 1, 1), (4, 2, 2)])
def test_fixture_records_follow_rank_block_order(p, pr, pc, tmp_path):
    a = fixture_matrix()
    path = os.path.join(GOLD, f"cb2b_rmat6_p{p}.cb2b")
    m, n, rec = oracle.read_cb2b(path)
    assert (m, n, len(rec)) == (a.nrows, a.ncols, a.nnz)
    rows, cols, vals = records_in_rank_order(a, pr, pc)
    assert np.array_equal(rec["row"], rows) and np.array_equal(rec["col"], cols)
    assert rec["val"].tobytes() == vals.tobytes()
    # the restated writer reproduces the reference's bytes
    out = str(tmp_path / "w.cb2b")
    oracle.write_cb2b(out, m, n, rows, cols, vals)
    assert open(out, "rb").read() == open(path, "rb").read()


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("p,pr,pc", [(1, 1, 1), (4, 2, 2), (2, 1, 2), (3, 3, 1)])
def test_reference_write_matches_fixture_rule(p, pr, pc, tmp_path):
    a = fixture_matrix()
    path = str(tmp_path / "ref.cb2b")
    oracle.ref().write_binary(a, path, p=p, pr=pr, pc=pc)
    rows, cols, vals = records_in_rank_order(a, pr, pc)
    want = str(tmp_path / "want.cb2b")
    oracle.write_cb2b(want, a.nrows, a.ncols, rows, cols, vals)
    assert open(path, "rb").read() == open(want, "rb").read()


@needs_ref
@pytest.mark.parametrize("p,pr,pc", [(1, 1, 1), (4, 2, 2), (2, 2, 1), (6, 2, 3)])
def test_reference_read_equals_routed_restatement(p, pr, pc):
    path = os.path.join(GOLD, "cb2b_rmat6_p4.cb2b")
    got = oracle.ref().read_binary(path, p=p, pr=pr, pc=pc)
    m, n, rec = oracle.read_cb2b(path)
    nnz = len(rec)
    parts = []
    for r in range(p):  # rank r reads records [nnz*r/p, nnz*(r+1)/p)
        lo, hi = nnz * r // p, nnz * (r + 1) // p
        parts.append((rec["row"][lo:hi], rec["col"][lo:hi], rec["val"][lo:hi]))
    t = G.tiling_2d(m, n, pr, pc)
    want = oracle.redistribute(oracle.PLUS_TIMES_F64, t.row_cuts, t.col_cuts, t.owner, m, n, parts)
    for r in range(p):
        rs, cs, b = got[r]
        wrs, wcs, w = want[r]
        assert (rs, cs) == (wrs, wcs)
        assert np.array_equal(b.colptr, w.colptr) and np.array_equal(b.rowids, w.rowids)
        assert b.vals.tobytes() == w.vals.tobytes()


def corrupt_files(tmp_path):
    raw = open(os.path.join(GOLD, "cb2b_rmat6_p1.cb2b"), "rb").read()
    cases = {
        "magic": b"CB2X" + raw[4:],
        "version": raw[:4] + np.uint32(2).tobytes() + raw[8:],
        "truncated": raw[:-5],
        "short": raw[:20],
        "negative": raw[:8] + np.int64(-1).tobytes() + raw[16:],
    }
    out = {}
    for k, b in cases.items():
        pth = str(tmp_path / f"{k}.cb2b")
        open(pth, "wb").write(b)
        out[k] = pth
    return out


@needs_ref
def test_format_errors_match_reference(tmp_path):
    for k, pth in corrupt_files(tmp_path).items():
        with pytest.raises(ValueError, match="FormatError"):
            oracle.read_cb2b(pth)
        with pytest.raises(ValueError, match="FormatError"):
            oracle.ref().read_binary(pth)
    with pytest.raises(ValueError, match="IoError"):
        oracle.ref().read_binary(str(tmp_path / "missing.cb2b"))


def test_library_header_entry_point(tmp_path):
    import paper_2106_14402_b200 as P
    from paper_2106_14402_b200 import _lib as L

    lib = P.load_library()
    m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    st = lib.slapcu_cb2b_header(os.path.join(GOLD, "cb2b_rmat6_p4.cb2b").encode(), C.byref(m), C.byref(n),
                                C.byref(nnz))
    a = fixture_matrix()
    assert st == L.OK and (m.value, n.value, nnz.value) == (a.nrows, a.ncols, a.nnz)
    for k, pth in corrupt_files(tmp_path).items():
        assert lib.slapcu_cb2b_header(pth.encode(), C.byref(m), C.byref(n), C.byref(nnz)) == 13, k  # FormatError
    assert lib.slapcu_cb2b_header(str(tmp_path / "missing").encode(), C.byref(m), C.byref(n), C.byref(nnz)) == 12
