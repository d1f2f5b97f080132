"""Process-grid geometry of the reference's distributed layer (host logic).

Restates, with the same names and formulas:
  block_offsets / block_of        layout.hpp:60-73 (floor rule, remainder to last)
  Grid2D rank <-> (i, j)          grid.hpp:15-24 (rank = i*pc + j)
  Grid3D regular rank <-> (l,i,j) grid.cpp:57, :60-75 (rank = l*q*q + i*q + j)
  regular_3d_range                dist_matrix3d.hpp:54-80
  layer_warning                   spgemm3d.hpp:38-41 (c > cbrt(p))
and host-side block extraction / assembly of CSC matrices used to hand each
rank its operand blocks (the role of distribute_triples / redistribute_3d,
dist_matrix.hpp:89-119, dist_matrix3d.hpp:117-219, for inputs that start on
one host) and to gather results (gather_matrix, dist_matrix.hpp:121-145).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import errors as E


def block_offsets(extent: int, parts: int) -> list[int]:
    """layout.hpp:60-66: offsets[i] = i*floor(extent/parts), offsets[parts] = extent."""
    if parts < 1:
        raise E.ShapeError("parts must be >= 1")
    q = extent // parts
    return [i * q for i in range(parts)] + [extent]


def block_of(offsets: list[int], g: int) -> int:
    """layout.hpp:70-73 (upper_bound - 1)."""
    import bisect

    return bisect.bisect_right(offsets, g) - 1


def is_perfect_square(v: int) -> bool:
    if v < 0:
        return False
    r = math.isqrt(v)
    return r * r == v


def isqrt_exact(v: int) -> int:
    if not is_perfect_square(v):
        raise E.ShapeError(f"{v} is not a perfect square")
    return math.isqrt(v)


@dataclass(frozen=True)
class Grid2D:
    """pr x pc grid, rank (i, j) = i*pc + j (grid.hpp:15-24)."""

    pr: int
    pc: int
    rank: int

    @property
    def myrow(self) -> int:
        return self.rank // self.pc

    @property
    def mycol(self) -> int:
        return self.rank % self.pc

    def rank_of(self, i: int, j: int) -> int:
        return i * self.pc + j

    @property
    def square(self) -> bool:
        return self.pr == self.pc

    @staticmethod
    def square_of(p: int, rank: int) -> "Grid2D":
        q = isqrt_exact(p)
        return Grid2D(q, q, rank)


@dataclass(frozen=True)
class Grid3D:
    """c layers of q x q, regular variant: rank = l*q*q + i*q + j (grid.cpp:57)."""

    c: int
    q: int
    rank: int

    @staticmethod
    def make(p: int, c: int, rank: int) -> "Grid3D":
        """grid.cpp:79-88 make_grid3d shape checks."""
        if c < 1 or p % c != 0:
            raise E.ShapeError(f"cannot split {p} ranks into {c} layers")
        if not is_perfect_square(p // c):
            raise E.ShapeError(f"p/c = {p // c} is not a perfect square")
        return Grid3D(c, math.isqrt(p // c), rank)

    @property
    def size(self) -> int:
        return self.c * self.q * self.q

    def coords_of(self, r: int):
        per = self.q * self.q
        return r // per, (r % per) // self.q, r % self.q

    @property
    def coords(self):
        return self.coords_of(self.rank)

    def rank_of(self, l: int, i: int, j: int) -> int:
        return l * self.q * self.q + i * self.q + j

    @property
    def layer_warning(self) -> bool:
        """spgemm3d.hpp:38-41."""
        return self.c > (self.size ** (1.0 / 3.0)) + 1e-9


def block2d_range(m: int, n: int, pr: int, pc: int, i: int, j: int):
    """Extents of 2D block (i, j) (dist_matrix.hpp:96-97 block_offsets rule)."""
    ro, co = block_offsets(m, pr), block_offsets(n, pc)
    return ro[i], ro[i + 1] - ro[i], co[j], co[j + 1] - co[j]


def regular_3d_range(m: int, n: int, c: int, q: int, split: str, l: int, i: int, j: int):
    """dist_matrix3d.hpp:54-80 (row_start, row_len, col_start, col_len)."""
    if split == "cols":
        ro = block_offsets(m, q)
        slabs = block_offsets(n, c)
        ss, sl = slabs[l], slabs[l + 1] - slabs[l]
        co = block_offsets(sl, q)
        return ro[i], ro[i + 1] - ro[i], ss + co[j], co[j + 1] - co[j]
    co = block_offsets(n, q)
    slabs = block_offsets(m, c)
    ss, sl = slabs[l], slabs[l + 1] - slabs[l]
    ro = block_offsets(sl, q)
    return ss + ro[i], ro[i + 1] - ro[i], co[j], co[j + 1] - co[j]


def ca3d_output_range(m: int, n_b: int, c: int, q: int, l: int, i: int, j: int):
    """Global extents of C3 block (l, i, j) (spgemm3d.hpp:80-90): rows of A's
    block i, B's column block j split into c pieces, piece l."""
    ro = block_offsets(m, q)
    co = block_offsets(n_b, q)
    piece = block_offsets(co[j + 1] - co[j], c)
    return ro[i], ro[i + 1] - ro[i], co[j] + piece[l], piece[l + 1] - piece[l]


# ------------------------------------------------- redistribution tilings
#
# A target layout for slapcu_redistribute / slapcu_distribute_triples: row
# cuts, column cuts and owner[i][j] = the rank holding tile (i, j).


@dataclass(frozen=True)
class Tiling:
    row_cuts: tuple
    col_cuts: tuple
    owner: tuple  # row-major nr x nc ranks

    @property
    def nr(self) -> int:
        return len(self.row_cuts) - 1

    @property
    def nc(self) -> int:
        return len(self.col_cuts) - 1

    def tile_of(self, rank: int):
        """(row_start, row_len, col_start, col_len) of `rank`'s tile."""
        k = self.owner.index(rank)
        i, j = divmod(k, self.nc)
        return (self.row_cuts[i], self.row_cuts[i + 1] - self.row_cuts[i], self.col_cuts[j],
                self.col_cuts[j + 1] - self.col_cuts[j])


def tiling_2d(m: int, n: int, pr: int, pc: int) -> Tiling:
    """distribute_triples / redistribute_2d target (dist_matrix.hpp:95-97
    block_offsets rows/cols, grid.hpp:15-24 rank = i*pc + j)."""
    return Tiling(tuple(block_offsets(m, pr)), tuple(block_offsets(n, pc)),
                  tuple(i * pc + j for i in range(pr) for j in range(pc)))


def tiling_3d(m: int, n: int, c: int, q: int, split: str) -> Tiling:
    """redistribute_3d regular target (dist_matrix3d.hpp:54-80 and :144-166):
    the split dimension cut into c slabs, each slab into q sub-blocks; the
    other dimension into q blocks; tile (l, i, j) on rank l*q*q + i*q + j."""
    if split not in ("cols", "rows"):
        raise E.ShapeError(f"split must be 'cols' or 'rows', got {split!r}")
    ext = n if split == "cols" else m
    slabs = block_offsets(ext, c)
    cuts = []
    for l in range(c):
        sub = block_offsets(slabs[l + 1] - slabs[l], q)
        cuts += [slabs[l] + x for x in sub[:-1]]
    cuts.append(ext)
    other = block_offsets(m if split == "cols" else n, q)
    owner = []
    if split == "cols":  # rows: q blocks (i); cols: c*q pieces (l, j)
        for i in range(q):
            for lj in range(c * q):
                l, j = divmod(lj, q)
                owner.append(l * q * q + i * q + j)
        return Tiling(tuple(other), tuple(cuts), tuple(owner))
    for li in range(c * q):  # rows: c*q pieces (l, i); cols: q blocks (j)
        l, i = divmod(li, q)
        for j in range(q):
            owner.append(l * q * q + i * q + j)
    return Tiling(tuple(cuts), tuple(other), tuple(owner))


# ----------------------------------------------------- host block utilities


def extract_block(colptr, rowids, vals, r0: int, rl: int, c0: int, cl: int):
    """Entries of rows [r0, r0+rl) x cols [c0, c0+cl) with block-local
    indices, as (colptr int64, rowids int32, vals)."""
    colptr = np.asarray(colptr)
    rowids = np.asarray(rowids)
    out_cp = np.zeros(cl + 1, np.int64)
    sel_idx = []
    for jj in range(cl):
        s, e = int(colptr[c0 + jj]), int(colptr[c0 + jj + 1])
        seg = rowids[s:e]
        lo = s + int(np.searchsorted(seg, r0, "left"))
        hi = s + int(np.searchsorted(seg, r0 + rl, "left"))
        sel_idx.append(np.arange(lo, hi))
        out_cp[jj + 1] = out_cp[jj] + (hi - lo)
    idx = np.concatenate(sel_idx) if sel_idx else np.zeros(0, np.int64)
    rw = (rowids[idx].astype(np.int64) - r0).astype(np.int32)
    vv = None if vals is None else np.asarray(vals)[idx]
    return out_cp, rw, vv


def assemble(nrows: int, ncols: int, blocks):
    """Global CSC from blocks [(row_start, col_start, colptr, rowids, vals)]
    (gather_matrix, dist_matrix.hpp:121-145: entries sorted by (col,row))."""
    rows, cols, vals = [], [], []
    for rs, cs, cp, rw, vv in blocks:
        cp = np.asarray(cp)
        cnt = np.diff(cp)
        cols.append(np.repeat(np.arange(len(cnt), dtype=np.int64) + cs, cnt))
        rows.append(np.asarray(rw, np.int64) + rs)
        vals.append(np.asarray(vv))
    r = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    c = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    v = np.concatenate(vals) if vals else np.zeros(0)
    order = np.lexsort((r, c))
    r, c, v = r[order], c[order], v[order]
    colptr = np.zeros(ncols + 1, np.int64)
    np.add.at(colptr, c + 1, 1)
    return np.cumsum(colptr).astype(np.int64), r.astype(np.int32), v
