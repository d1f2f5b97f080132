"""Block-by-block restatement of the reference's distributed SpGEMM drivers on
the CPU oracle (test infrastructure).  Uses the product's grid geometry
(paper_2106_14402_b200.grid) and the oracle's local product / merge, so it
pins both the geometry and the stage fold order against fixtures produced by
the compiled reference (tests/golden/make_golden.py)."""
from __future__ import annotations

import numpy as np

import oracle
from paper_2106_14402_b200 import grid as G


def _blk(m: oracle.Csc, r0, rl, c0, cl) -> oracle.Csc:
    cp, rw, vv = G.extract_block(m.colptr, m.rowids, m.vals, r0, rl, c0, cl)
    return oracle.Csc(rl, cl, cp, rw, vv)


def simulate_summa2d(port, sr, a: oracle.Csc, b: oracle.Csc, q: int) -> oracle.Csc:
    """summa.hpp:106-163: C(i,j) = merge_s A(i,s) * B(s,j) in stage order."""
    ro, ko, co = G.block_offsets(a.nrows, q), G.block_offsets(a.ncols, q), G.block_offsets(b.ncols, q)
    blocks = []
    for i in range(q):
        for j in range(q):
            parts = []
            for s in range(q):
                ab = _blk(a, ro[i], ro[i + 1] - ro[i], ko[s], ko[s + 1] - ko[s])
                bb = _blk(b, ko[s], ko[s + 1] - ko[s], co[j], co[j + 1] - co[j])
                parts.append(port.spgemm(sr, ab, bb))
            cij = port.merge(sr, parts) if len(parts) > 1 else parts[0]
            blocks.append((ro[i], co[j], cij.colptr, cij.rowids, cij.vals))
    cp, rw, vv = G.assemble(a.nrows, b.ncols, blocks)
    return oracle.Csc(a.nrows, b.ncols, cp, rw, vv.astype(oracle.DTYPES[sr]))


def simulate_ca3d(port, sr, a: oracle.Csc, b: oracle.Csc, c: int, q: int) -> oracle.Csc:
    """spgemm3d.hpp:21-106 with the regular 3D geometry: per layer SUMMA over
    A3(l,i,s) * B3(l,s,j), C_int(i,j) split into c column pieces, pieces folded
    across layers in fiber order."""
    m, n_b = a.nrows, b.ncols
    out = []
    cint = {}
    for l in range(c):
        for i in range(q):
            for j in range(q):
                parts = []
                for s in range(q):
                    ar = G.regular_3d_range(a.nrows, a.ncols, c, q, "cols", l, i, s)
                    br = G.regular_3d_range(b.nrows, b.ncols, c, q, "rows", l, s, j)
                    parts.append(port.spgemm(sr, _blk(a, *ar), _blk(b, *br)))
                cint[(l, i, j)] = port.merge(sr, parts) if len(parts) > 1 else parts[0]
    for l in range(c):
        for i in range(q):
            for j in range(q):
                r0, rl, c0, cl = G.ca3d_output_range(m, n_b, c, q, l, i, j)
                co = G.block_offsets(n_b, q)
                piece0 = c0 - co[j]
                pieces = []
                for src in range(c):
                    ci = cint[(src, i, j)]
                    pieces.append(_blk(ci, 0, ci.nrows, piece0, cl))
                merged = port.merge(sr, pieces) if len(pieces) > 1 else pieces[0]
                out.append((r0, c0, merged.colptr, merged.rowids, merged.vals))
    cp, rw, vv = G.assemble(m, n_b, out)
    return oracle.Csc(m, n_b, cp, rw, vv.astype(oracle.DTYPES[sr]))
