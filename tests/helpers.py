"""Shared test helpers: oracle <-> device conversion and the parity rules.

Parity rules (BASELINE.json north_star):
  * integer / Boolean / MinPlus semirings: bit-exact structure and values;
  * PlusTimes fp64: pattern-exact, values rel_close 1e-12
    (acceptance.cpp:49-54, max(1,|a|,|b|) scaling);
  * PlusTimes fp32: pattern-exact, values rel_close 1e-5 (SURVEY.md 8d
    proposal; the reference does not pin an fp32 tolerance).
"""
from __future__ import annotations

import numpy as np

import oracle

TOL = {oracle.PLUS_TIMES_F64: 1e-12, oracle.PLUS_TIMES_F32: 1e-5}

# value recipe per semiring used by the randomized tests (SURVEY.md 8d kinds)
KIND = {
    oracle.PLUS_TIMES_F64: 2,  # U[0,10)
    oracle.PLUS_TIMES_F32: 1,  # U[0,1)
    oracle.PLUS_TIMES_I64: 5,  # small ints 1..9
    oracle.MIN_PLUS_I32: 3,    # 1 + h % 255
    oracle.MIN_PLUS_F64: 5,    # small ints as doubles
    oracle.OR_AND_U8: 0,       # ones
}


def to_device(m: "oracle.Csc"):
    import paper_2106_14402_b200 as P

    return P.CscMatrix(m.nrows, m.ncols, m.colptr, m.rowids, m.vals).to_device()


def to_oracle(d) -> "oracle.Csc":
    h = d.to_host() if hasattr(d, "to_host") else d
    return oracle.Csc(h.nrows, h.ncols, np.asarray(h.colptr), np.asarray(h.rowids), h.vals)


def rel_close(a: np.ndarray, b: np.ndarray, tol: float) -> np.ndarray:
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    scale = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return (a == b) | (np.abs(a - b) <= tol * scale)


def assert_parity(got, want: "oracle.Csc", sr: int, what: str = ""):
    g = to_oracle(got)
    assert (g.nrows, g.ncols) == (want.nrows, want.ncols), f"{what}: shape {g.nrows}x{g.ncols}"
    assert np.array_equal(g.colptr, want.colptr), f"{what}: colptr differs"
    assert np.array_equal(g.rowids, want.rowids), f"{what}: rowids differ"
    if want.vals is None:
        return
    gv = np.asarray(g.vals)
    wv = np.asarray(want.vals)
    assert gv.dtype == wv.dtype, f"{what}: dtype {gv.dtype} vs {wv.dtype}"
    if sr in TOL:
        ok = rel_close(gv, wv, TOL[sr])
        assert ok.all(), f"{what}: {int((~ok).sum())} values outside rel {TOL[sr]}"
    else:
        assert gv.tobytes() == wv.tobytes(), f"{what}: values not bit-exact ({int((gv != wv).sum())} differ)"


def with_values(P, m: "oracle.Csc", sr: int, kind: int | None = None) -> "oracle.Csc":
    return m.with_vals(P.fill_values(sr, KIND[sr] if kind is None else kind, m))
