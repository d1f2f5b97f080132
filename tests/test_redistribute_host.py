"""Redistribution host logic (CPU): the target tilings restate the reference's
2D / regular-3D geometry, and the oracle's routed-redistribution restatement
matches the compiled reference's distribute_triples / redistribute_3d /
redistribute_2d (oracle/_ref, dist_matrix.hpp:89-119, dist_matrix3d.hpp:117-261)
block by block, duplicates and semiring combines included."""
import numpy as np
import pytest

import oracle
from paper_2106_14402_b200 import grid as G


@pytest.mark.parametrize("m,n", [(37, 53), (64, 64), (5, 3), (1000, 7)])
@pytest.mark.parametrize("c,q", [(1, 1), (2, 1), (2, 2), (4, 1), (1, 3)])
@pytest.mark.parametrize("split", ["cols", "rows"])
def test_tiling_3d_matches_regular_range(m, n, c, q, split):
    t = G.tiling_3d(m, n, c, q, split)
    assert t.nr * t.nc == c * q * q
    assert sorted(t.owner) == list(range(c * q * q))
    for rank in range(c * q * q):
        l, i, j = G.Grid3D(c, q, rank).coords
        assert t.tile_of(rank) == G.regular_3d_range(m, n, c, q, split, l, i, j)


@pytest.mark.parametrize("m,n,pr,pc", [(37, 53, 2, 2), (10, 10, 1, 4), (9, 100, 3, 2), (2, 2, 4, 1)])
def test_tiling_2d_matches_block_range(m, n, pr, pc):
    t = G.tiling_2d(m, n, pr, pc)
    for rank in range(pr * pc):
        assert t.tile_of(rank) == G.block2d_range(m, n, pr, pc, rank // pc, rank % pc)


def _triples(seed, m, n, count, sr, p):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, m, count)
    cols = rng.integers(0, n, count)
    # few distinct coordinates -> plenty of duplicates
    rows[: count // 3] = rows[count // 3: 2 * (count // 3)]
    cols[: count // 3] = cols[count // 3: 2 * (count // 3)]
    dt = oracle.DTYPES[sr]
    if sr == oracle.OR_AND_U8:
        vals = rng.integers(0, 2, count).astype(dt)
    elif np.issubdtype(dt, np.integer):
        vals = rng.integers(-50, 50, count).astype(dt)
    else:
        vals = rng.standard_normal(count).astype(dt)
    src = rng.integers(0, p, count).astype(np.int32)
    return src, rows, cols, vals


def _parts(src, rows, cols, vals, p):
    return [(rows[src == r], cols[src == r], vals[src == r]) for r in range(p)]


def _block_triples(rs, cs, m: oracle.Csc):
    """Global triples of a block in for_each_col order (the reference's push order)."""
    cnt = np.diff(m.colptr)
    cols = np.repeat(np.arange(m.ncols, dtype=np.int64), cnt) + cs
    return np.asarray(m.rowids, np.int64) + rs, cols, m.vals


def _same(a, b):
    rs_a, cs_a, ma = a
    rs_b, cs_b, mb = b
    assert (rs_a, cs_a, ma.nrows, ma.ncols) == (rs_b, cs_b, mb.nrows, mb.ncols)
    assert np.array_equal(ma.colptr, mb.colptr)
    assert np.array_equal(ma.rowids, mb.rowids)
    assert np.array_equal(ma.vals, mb.vals)


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("sr", range(6))
@pytest.mark.parametrize("combine", ["first", "add"])
@pytest.mark.parametrize("p,pr,pc", [(1, 1, 1), (4, 2, 2), (2, 1, 2)])
def test_distribute_triples_restatement_matches_reference(sr, combine, p, pr, pc):
    m, n = 23, 31
    src, rows, cols, vals = _triples(7 + sr, m, n, 300, sr, p)
    want = oracle.ref().redistribute(sr, p, pr, pc, m, n, src, rows, cols, vals, mode=0, combine=combine)
    t = G.tiling_2d(m, n, pr, pc)
    got = oracle.redistribute(sr, t.row_cuts, t.col_cuts, t.owner, m, n, _parts(src, rows, cols, vals, p), combine)
    for r in range(p):
        _same(got[r], want[r])


@needs_ref
@pytest.mark.parametrize("sr", [oracle.PLUS_TIMES_F64, oracle.MIN_PLUS_I32, oracle.OR_AND_U8])
@pytest.mark.parametrize("p,layers", [(2, 2), (4, 1), (4, 4), (8, 2)])
@pytest.mark.parametrize("split", ["cols", "rows"])
def test_redistribute_3d_and_back_match_reference(sr, p, layers, split):
    m, n = 29, 41
    q2 = G.isqrt_exact(p) if G.is_perfect_square(p) else None
    pr, pc = (q2, q2) if q2 else (2, p // 2)
    src, rows, cols, vals = _triples(3 + p, m, n, 250, sr, p)
    ref3 = oracle.ref().redistribute(sr, p, pr, pc, m, n, src, rows, cols, vals, mode=1, layers=layers, split=split)
    ref2 = oracle.ref().redistribute(sr, p, pr, pc, m, n, src, rows, cols, vals, mode=2, layers=layers, split=split)
    t2 = G.tiling_2d(m, n, pr, pc)
    d2 = oracle.redistribute(sr, t2.row_cuts, t2.col_cuts, t2.owner, m, n, _parts(src, rows, cols, vals, p))
    q = G.Grid3D.make(p, layers, 0).q
    t3 = G.tiling_3d(m, n, layers, q, split)
    d3 = oracle.redistribute(sr, t3.row_cuts, t3.col_cuts, t3.owner, m, n,
                             [_block_triples(*d2[r]) for r in range(p)])
    for r in range(p):
        _same(d3[r], ref3[r])
    back = oracle.redistribute(sr, t2.row_cuts, t2.col_cuts, t2.owner, m, n,
                               [_block_triples(*d3[r]) for r in range(p)])
    for r in range(p):
        _same(back[r], ref2[r])
        _same(back[r], d2[r])
