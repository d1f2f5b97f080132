"""Python access to the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``oracle.port``  -- the C restatement (oracle.c -> _build/liboracle.so)
* ``oracle.ref``   -- the unmodified reference core compiled in place
                      (ref_shim.cpp + /root/reference/proj/core/src ->
                      _ref/libslapref.so)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2106_14402_b200) never does.

Matrices cross this boundary as ``Csc`` (host numpy arrays): int64 colptr,
int32 rowids, values of the semiring's dtype -- the same layout as the device
library's C-ABI (include/slapcu.h).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libslapref.so")

# semiring ids (include/slapcu.h; oracle.h)
PLUS_TIMES_F64, PLUS_TIMES_F32, PLUS_TIMES_I64, MIN_PLUS_I32, MIN_PLUS_F64, OR_AND_U8 = range(6)
DTYPES = {
    PLUS_TIMES_F64: np.float64,
    PLUS_TIMES_F32: np.float32,
    PLUS_TIMES_I64: np.int64,
    MIN_PLUS_I32: np.int32,
    MIN_PLUS_F64: np.float64,
    OR_AND_U8: np.uint8,
}
HEAP, HASH, HYBRID = 0, 1, 2


@dataclass
class Csc:
    nrows: int
    ncols: int
    colptr: np.ndarray  # int64 [ncols+1]
    rowids: np.ndarray  # int32 [nnz]
    vals: np.ndarray | None = None

    @property
    def nnz(self) -> int:
        return int(self.colptr[-1]) if len(self.colptr) else 0

    def with_vals(self, vals):
        return Csc(self.nrows, self.ncols, self.colptr, self.rowids, vals)

    def to_dense(self, fill=0):
        d = np.full((self.nrows, self.ncols), fill, dtype=self.vals.dtype if self.vals is not None else np.uint8)
        for j in range(self.ncols):
            s, e = self.colptr[j], self.colptr[j + 1]
            d[self.rowids[s:e], j] = self.vals[s:e] if self.vals is not None else 1
        return d


class _CCsc(C.Structure):
    _fields_ = [
        ("nrows", C.c_int64),
        ("ncols", C.c_int64),
        ("nnz", C.c_int64),
        ("colptr", C.c_void_p),
        ("rowids", C.c_void_p),
        ("vals", C.c_void_p),
    ]


def _as_c(m: Csc, keep: list) -> _CCsc:
    cp = np.ascontiguousarray(m.colptr, dtype=np.int64)
    rw = np.ascontiguousarray(m.rowids, dtype=np.int32)
    keep += [cp, rw]
    vp = None
    if m.vals is not None:
        vv = np.ascontiguousarray(m.vals)
        keep.append(vv)
        vp = vv.ctypes.data
    return _CCsc(m.nrows, m.ncols, int(cp[-1]) if len(cp) else 0, cp.ctypes.data, rw.ctypes.data, vp)


def _from_c(c: _CCsc, dtype, free) -> Csc:
    n = c.ncols
    nnz = c.nnz
    colptr = np.ctypeslib.as_array(C.cast(c.colptr, C.POINTER(C.c_int64)), shape=(n + 1,)).copy()
    rowids = (
        np.ctypeslib.as_array(C.cast(c.rowids, C.POINTER(C.c_int32)), shape=(nnz,)).copy()
        if nnz
        else np.zeros(0, np.int32)
    )
    vals = None
    if c.vals and dtype is not None:
        raw = C.string_at(c.vals, nnz * np.dtype(dtype).itemsize) if nnz else b""
        vals = np.frombuffer(raw, dtype=dtype).copy()
    for p in (c.colptr, c.rowids, c.vals):
        if p:
            free(C.c_void_p(p))
    return Csc(c.nrows, c.ncols, colptr, rowids, vals)


class _Port:
    def __init__(self, path=PORT_LIB):
        self.lib = L = C.CDLL(path)
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_gen_rmat.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.POINTER(_CCsc)]
        L.orc_gen_er.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.POINTER(_CCsc)]
        L.orc_fill_values.argtypes = [C.c_int, C.c_int, C.POINTER(_CCsc), C.c_void_p]
        L.orc_estimate_flops.restype = C.c_int64
        L.orc_estimate_flops.argtypes = [C.POINTER(_CCsc), C.POINTER(_CCsc), C.c_void_p]
        L.orc_symbolic_nnz.restype = C.c_int64
        L.orc_symbolic_nnz.argtypes = [C.POINTER(_CCsc), C.POINTER(_CCsc), C.c_void_p, C.c_int]
        L.orc_spgemm.argtypes = [C.c_int, C.POINTER(_CCsc), C.POINTER(_CCsc), C.c_int64, C.c_int64,
                                 C.POINTER(_CCsc), C.c_int]
        L.orc_merge.argtypes = [C.c_int, C.c_int, C.POINTER(_CCsc), C.POINTER(_CCsc)]
        L.orc_column_checksums.argtypes = [C.c_int, C.POINTER(_CCsc), C.c_void_p]
        L.orc_free.argtypes = [C.c_void_p]

    def mix(self, z):
        return self.lib.orc_mix(z)

    def gen_rmat(self, scale, edge_factor=16, seed=1, a=0.57, b=0.19, c=0.19, d=0.05) -> Csc:
        out = _CCsc()
        rc = self.lib.orc_gen_rmat(scale, edge_factor, seed, a, b, c, d, C.byref(out))
        assert rc == 0, rc
        return _from_c(out, None, self.lib.orc_free)

    def gen_er(self, n, draws, seed=1) -> Csc:
        out = _CCsc()
        rc = self.lib.orc_gen_er(n, draws, seed, C.byref(out))
        assert rc == 0, rc
        return _from_c(out, np.float64, self.lib.orc_free)

    def fill_values(self, sr, kind, m: Csc) -> np.ndarray:
        vals = np.zeros(m.nnz, dtype=DTYPES[sr])
        keep = []
        cm = _as_c(m.with_vals(None), keep)
        self.lib.orc_fill_values(sr, kind, C.byref(cm), vals.ctypes.data)
        return vals

    def estimate_flops(self, a: Csc, b: Csc):
        keep = []
        per = np.zeros(b.ncols, np.int64)
        tot = self.lib.orc_estimate_flops(C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)), per.ctypes.data)
        return tot, per

    def symbolic_nnz(self, a: Csc, b: Csc, threads=0):
        keep = []
        per = np.zeros(b.ncols, np.int64)
        tot = self.lib.orc_symbolic_nnz(C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)), per.ctypes.data, threads)
        return tot, per

    def spgemm(self, sr, a: Csc, b: Csc, col_begin=0, col_end=0, threads=0) -> Csc:
        keep = []
        out = _CCsc()
        rc = self.lib.orc_spgemm(sr, C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)), col_begin, col_end,
                                 C.byref(out), threads)
        if rc != 0:
            raise RuntimeError(f"orc_spgemm failed: {rc}")
        return _from_c(out, DTYPES[sr], self.lib.orc_free)

    def write_binary(self, a: Csc, path: str, p=1, pr=1, pc=1):
        """binary_io.cpp write_binary of f64 `a` distributed on pr x pc ranks."""
        keep = []
        rc = self.lib.ref_write_binary(p, pr, pc, C.byref(_as_c(a, keep)), path.encode())
        if rc != 0:
            raise RuntimeError(f"ref_write_binary failed: {rc}")

    def read_binary(self, path: str, p=1, pr=1, pc=1):
        """binary_io.cpp read_binary -> [(row_start, col_start, block)] per rank;
        raises ValueError("IoError" / "FormatError")."""
        blocks = (_CCsc * p)()
        rs = np.zeros(p, np.int64)
        cs = np.zeros(p, np.int64)
        rc = self.lib.ref_read_binary(path.encode(), p, pr, pc, blocks, rs.ctypes.data, cs.ctypes.data)
        if rc in (-9, -10):
            raise ValueError("IoError" if rc == -9 else "FormatError")
        if rc != 0:
            raise RuntimeError(f"ref_read_binary failed: {rc}")
        return [(int(rs[r]), int(cs[r]), _from_c(blocks[r], np.float64, self.lib.ref_free)) for r in range(p)]

    def merge(self, sr, parts) -> Csc:
        keep = []
        arr = (_CCsc * len(parts))(*[_as_c(p, keep) for p in parts])
        out = _CCsc()
        rc = self.lib.orc_merge(sr, len(parts), arr, C.byref(out))
        if rc != 0:
            raise RuntimeError(f"orc_merge failed: {rc}")
        return _from_c(out, DTYPES[sr], self.lib.orc_free)

    def column_checksums(self, sr, m: Csc, with_values=True) -> np.ndarray:
        keep = []
        sums = np.zeros(m.ncols, np.uint64)
        mm = m if with_values else m.with_vals(None)
        self.lib.orc_column_checksums(sr, C.byref(_as_c(mm, keep)), sums.ctypes.data)
        return sums


class _Ref:
    def __init__(self, path=REF_LIB):
        self.lib = L = C.CDLL(path)
        P = C.POINTER(_CCsc)
        L.ref_local_spgemm.argtypes = [C.c_int, C.c_int, C.c_int, P, P, C.c_int, P]
        L.ref_estimate_flops.restype = C.c_int64
        L.ref_estimate_flops.argtypes = [P, P, C.c_void_p]
        L.ref_symbolic_nnz.argtypes = [P, P, C.c_int, C.c_void_p]
        L.ref_gen_rmat.argtypes = [C.c_int, C.c_int, C.c_uint64, P]
        L.ref_summa2d.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, P, P, P, C.c_void_p, C.c_void_p]
        L.ref_ca3d.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P]
        L.ref_plan_batches.argtypes = [C.c_int, C.c_int, P, P, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
        L.ref_merge.argtypes = [C.c_int, C.c_int, P, P]
        L.ref_mcl_step.argtypes = [C.c_int, C.c_int, P, C.c_double, C.c_double, P]
        L.ref_redistribute.argtypes = [C.c_int] * 8 + [C.c_int64] * 3 + [C.c_void_p] * 4 + [P, C.c_void_p,
                                                                                            C.c_void_p]
        L.ref_write_binary.argtypes = [C.c_int, C.c_int, C.c_int, P, C.c_char_p]
        L.ref_read_binary.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, P, C.c_void_p, C.c_void_p]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_time_local_spgemm.argtypes = [C.c_int, C.c_int, C.c_int, P, P, C.c_int64, C.c_int64,
                                            C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64), P]

    def time_local_spgemm(self, sr, a: Csc, b: Csc, c0: int, c1: int, threads: int, alg=HYBRID,
                          want_result=False):
        """Seconds of ONE reference local_spgemm(A, B(:, c0:c1)) call with
        `threads` threads (conversions excluded); returns (seconds, nnz, flops),
        plus the product C(:, c0:c1) as a Csc when `want_result`."""
        keep = []
        sec, nnz, fl = C.c_double(), C.c_int64(), C.c_int64()
        out = _CCsc() if want_result else None
        rc = self.lib.ref_time_local_spgemm(sr, alg, threads, C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)), c0, c1,
                                            C.byref(sec), C.byref(nnz), C.byref(fl),
                                            C.byref(out) if want_result else None)
        if rc != 0:
            raise RuntimeError(f"ref_time_local_spgemm failed: {rc}")
        if want_result:
            return sec.value, nnz.value, fl.value, _from_c(out, DTYPES[sr], self.lib.ref_free)
        return sec.value, nnz.value, fl.value

    def local_spgemm(self, sr, a: Csc, b: Csc, alg=HYBRID, threads=1, b_dcsc=False) -> Csc:
        keep = []
        out = _CCsc()
        rc = self.lib.ref_local_spgemm(sr, alg, threads, C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)),
                                       int(b_dcsc), C.byref(out))
        if rc != 0:
            raise RuntimeError(f"ref_local_spgemm failed: {rc}")
        return _from_c(out, DTYPES[sr], self.lib.ref_free)

    def estimate_flops(self, a: Csc, b: Csc):
        keep = []
        per = np.zeros(b.ncols, np.int64)
        tot = self.lib.ref_estimate_flops(C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)), per.ctypes.data)
        return tot, per

    def symbolic_nnz(self, a: Csc, b: Csc, threads=1):
        keep = []
        per = np.zeros(b.ncols, np.int64)
        rc = self.lib.ref_symbolic_nnz(C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)), threads, per.ctypes.data)
        assert rc == 0, rc
        return int(per.sum()), per

    def gen_rmat(self, scale, edge_factor=16, seed=1) -> Csc:
        out = _CCsc()
        rc = self.lib.ref_gen_rmat(scale, edge_factor, seed, C.byref(out))
        assert rc == 0, rc
        return _from_c(out, None, self.lib.ref_free)

    def mcl_step(self, a: Csc, inflation=2.0, prune=1e-4, p=1, layers=1) -> Csc:
        """algorithms.cpp:267-293 mcl_step (PlusTimes<double>) on p rank threads.
        Raises ValueError("StochasticityError") when a column sum is off by > 1e-9."""
        keep = []
        out = _CCsc()
        rc = self.lib.ref_mcl_step(p, layers, C.byref(_as_c(a, keep)), inflation, prune, C.byref(out))
        if rc == -8:
            raise ValueError("StochasticityError")
        if rc != 0:
            raise RuntimeError(f"ref_mcl_step failed: {rc}")
        return _from_c(out, DTYPES[PLUS_TIMES_F64], self.lib.ref_free)

    def summa2d(self, sr, a: Csc, b: Csc, p=4, alg=HYBRID, threads=1):
        keep = []
        out = _CCsc()
        stages = C.c_int64(0)
        bc = C.c_int64(0)
        rc = self.lib.ref_summa2d(sr, alg, p, threads, C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)),
                                  C.byref(out), C.byref(stages), C.byref(bc))
        if rc != 0:
            raise RuntimeError(f"ref_summa2d failed: {rc}")
        return _from_c(out, DTYPES[sr], self.lib.ref_free), stages.value, bc.value

    def ca3d(self, sr, a: Csc, b: Csc, p, pr, pc, layers, alg=HYBRID, threads=1) -> Csc:
        keep = []
        out = _CCsc()
        rc = self.lib.ref_ca3d(sr, alg, p, pr, pc, layers, threads, C.byref(_as_c(a, keep)),
                               C.byref(_as_c(b, keep)), C.byref(out))
        if rc != 0:
            raise RuntimeError(f"ref_ca3d failed: {rc}")
        return _from_c(out, DTYPES[sr], self.lib.ref_free)

    def plan_batches(self, a: Csc, b: Csc, budget, p=1, threads=1):
        keep = []
        mx = 4096
        ranges = np.zeros(2 * mx, np.int64)
        est = np.zeros(mx, np.int64)
        nr = self.lib.ref_plan_batches(p, threads, C.byref(_as_c(a, keep)), C.byref(_as_c(b, keep)), budget,
                                       ranges.ctypes.data, est.ctypes.data, mx)
        if nr < 0:
            raise RuntimeError(f"ref_plan_batches failed: {nr}")
        return [(int(ranges[2 * i]), int(ranges[2 * i + 1])) for i in range(nr)], est[:nr].copy()

    def redistribute(self, sr, p, pr, pc, nrows, ncols, src, rows, cols, vals, mode=0, layers=1, split="cols",
                     combine="first"):
        """ref_redistribute: distribute_triples (dist_matrix.hpp:89-119) of the
        triples held by ranks src[k] onto pr x pc; mode 1 then redistribute_3d
        (dist_matrix3d.hpp:117-170), mode 2 then redistribute_2d (:250-261).
        Returns [(row_start, col_start, block Csc)] per rank."""
        src = np.ascontiguousarray(src, np.int32)
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, DTYPES[sr])
        blocks = (_CCsc * p)()
        rs = np.zeros(p, np.int64)
        cs = np.zeros(p, np.int64)
        rc = self.lib.ref_redistribute(sr, p, pr, pc, mode, layers, int(split == "rows"), int(combine == "add"),
                                       nrows, ncols, len(rows), src.ctypes.data, rows.ctypes.data, cols.ctypes.data,
                                       vals.ctypes.data, blocks, rs.ctypes.data, cs.ctypes.data)
        if rc != 0:
            raise RuntimeError(f"ref_redistribute failed: {rc}")
        return [(int(rs[r]), int(cs[r]), _from_c(blocks[r], DTYPES[sr], self.lib.ref_free)) for r in range(p)]

    def write_binary(self, a: Csc, path: str, p=1, pr=1, pc=1):
        """binary_io.cpp write_binary of f64 `a` distributed on pr x pc ranks."""
        keep = []
        rc = self.lib.ref_write_binary(p, pr, pc, C.byref(_as_c(a, keep)), path.encode())
        if rc != 0:
            raise RuntimeError(f"ref_write_binary failed: {rc}")

    def read_binary(self, path: str, p=1, pr=1, pc=1):
        """binary_io.cpp read_binary -> [(row_start, col_start, block)] per rank;
        raises ValueError("IoError" / "FormatError")."""
        blocks = (_CCsc * p)()
        rs = np.zeros(p, np.int64)
        cs = np.zeros(p, np.int64)
        rc = self.lib.ref_read_binary(path.encode(), p, pr, pc, blocks, rs.ctypes.data, cs.ctypes.data)
        if rc in (-9, -10):
            raise ValueError("IoError" if rc == -9 else "FormatError")
        if rc != 0:
            raise RuntimeError(f"ref_read_binary failed: {rc}")
        return [(int(rs[r]), int(cs[r]), _from_c(blocks[r], np.float64, self.lib.ref_free)) for r in range(p)]

    def merge(self, sr, parts) -> Csc:
        keep = []
        arr = (_CCsc * len(parts))(*[_as_c(p, keep) for p in parts])
        out = _CCsc()
        rc = self.lib.ref_merge(sr, len(parts), arr, C.byref(out))
        if rc != 0:
            raise RuntimeError(f"ref_merge failed: {rc}")
        return _from_c(out, DTYPES[sr], self.lib.ref_free)


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def from_triples(nrows, ncols, rows, cols, vals, combine="first") -> Csc:
    """Canonical CSC from COO (duplicates keep the first value; build_csc with
    a keep-first add, local_matrix.hpp:194-204)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.asarray(vals)
    order = np.lexsort((np.arange(len(rows)), rows, cols))
    r, c, v = rows[order], cols[order], vals[order]
    keep = np.ones(len(r), bool)
    if len(r):
        keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    r, c, v = r[keep], c[keep], v[keep]
    colptr = np.zeros(ncols + 1, np.int64)
    np.add.at(colptr, c + 1, 1)
    colptr = np.cumsum(colptr).astype(np.int64)
    return Csc(nrows, ncols, colptr, r.astype(np.int32), v)


def _sr_add(sr, x, y):
    """semiring.hpp:36-93 add on the element type."""
    if sr in (PLUS_TIMES_F64, PLUS_TIMES_F32, PLUS_TIMES_I64):
        return (x + y).astype(x.dtype) if hasattr(x, "astype") else x + y
    if sr in (MIN_PLUS_I32, MIN_PLUS_F64):
        return x if x < y else y
    return np.uint8(1 if (x or y) else 0)


def redistribute(sr, tiling_rows, tiling_cols, owner, nrows, ncols, parts, combine="first"):
    """Restatement of one routed redistribution (dist_matrix.hpp:89-119,
    dist_matrix3d.hpp:117-174, local_matrix.hpp:167-188): `parts[r]` are the
    global (rows, cols, vals) triples of source rank r in its push order; every
    entry goes to the owner of the tile (block_of on the cuts) holding it; a
    target assembles its arrivals (source-rank order) with a stable
    (col, row) sort, keeping the first duplicate or folding the semiring add
    left.  Returns {rank: (row_start, col_start, Csc)}."""
    import bisect

    nr, nc = len(tiling_rows) - 1, len(tiling_cols) - 1
    inbox = {o: ([], [], []) for o in owner}
    for rows, cols, vals in parts:
        for r, c, v in zip(np.asarray(rows).tolist(), np.asarray(cols).tolist(), np.asarray(vals)):
            if not (0 <= r < nrows and 0 <= c < ncols):
                raise IndexError(f"triple ({r},{c}) outside {nrows}x{ncols}")
            ti = bisect.bisect_right(tiling_rows, r) - 1
            tj = bisect.bisect_right(tiling_cols, c) - 1
            ti, tj = min(ti, nr - 1), min(tj, nc - 1)
            box = inbox[owner[ti * nc + tj]]
            box[0].append(r - tiling_rows[ti])
            box[1].append(c - tiling_cols[tj])
            box[2].append(v)
    out = {}
    for k, o in enumerate(owner):
        ti, tj = divmod(k, nc)
        tr, tc = tiling_rows[ti + 1] - tiling_rows[ti], tiling_cols[tj + 1] - tiling_cols[tj]
        lr, lc, lv = inbox[o]
        dtype = DTYPES[sr]
        order = sorted(range(len(lr)), key=lambda e: (lc[e], lr[e]))  # stable
        rr, cc, vv = [], [], []
        for e in order:
            if rr and rr[-1] == lr[e] and cc[-1] == lc[e]:
                if combine == "add":
                    vv[-1] = dtype(_sr_add(sr, dtype(vv[-1]), dtype(lv[e])))
                continue
            rr.append(lr[e])
            cc.append(lc[e])
            vv.append(dtype(lv[e]))
        colptr = np.zeros(tc + 1, np.int64)
        np.add.at(colptr, np.asarray(cc, np.int64) + 1, 1)
        out[o] = (tiling_rows[ti], tiling_cols[tj],
                  Csc(tr, tc, np.cumsum(colptr).astype(np.int64), np.asarray(rr, np.int32), np.asarray(vv, dtype)))
    return out


CB2B_RECORD = np.dtype([("row", "<i8"), ("col", "<i8"), ("val", "<f8")])


def read_cb2b(path):
    """binary_io.hpp:10-28 restated: (nrows, ncols, records) of a CB2B v1
    file; ValueError("FormatError") on bad magic / version / size."""
    raw = open(path, "rb").read()
    if len(raw) < 32 or raw[:4] != b"CB2B" or np.frombuffer(raw[4:8], "<u4")[0] != 1:
        raise ValueError("FormatError")
    m, n, nnz = (int(x) for x in np.frombuffer(raw[8:32], "<i8"))
    if m < 0 or n < 0 or nnz < 0 or len(raw) != 32 + 24 * nnz:
        raise ValueError("FormatError")
    return m, n, np.frombuffer(raw[32:], CB2B_RECORD)


def write_cb2b(path, nrows, ncols, rows, cols, vals):
    """binary_io.hpp:10-28 restated writer (records in the given order)."""
    rec = np.empty(len(rows), CB2B_RECORD)
    rec["row"], rec["col"], rec["val"] = rows, cols, vals
    with open(path, "wb") as f:
        f.write(b"CB2B" + np.uint32(1).tobytes() + np.asarray([nrows, ncols, len(rows)], "<i8").tobytes())
        f.write(rec.tobytes())


def random_triples(rng_seed, m, n, density, val_kind, dtype):
    """oracles.hpp:205-217 random_triples with the reference's Rng stream:
    per entry draws row, col, then the value (small_int 1..9 or U[0,10))."""
    P = port()
    GOLD = 0x9E3779B97F4A7C15
    M64 = (1 << 64) - 1
    state = P.mix((rng_seed * GOLD + 0 + 1) & M64)
    target = int(density * m * n)
    rows, cols, vals = [], [], []

    def nxt():
        nonlocal state
        state = (state + GOLD) & M64
        return P.mix(state)

    for _ in range(target):
        r = nxt() % m
        c = nxt() % n
        if val_kind == "small_int":
            v = nxt() % 9 + 1
        elif val_kind == "one":
            v = 1
        else:
            v = (nxt() >> 11) * 2.0**-53 * 10.0
        rows.append(r)
        cols.append(c)
        vals.append(v)
    return from_triples(m, n, rows, cols, np.asarray(vals, dtype=dtype) if vals else np.zeros(0, dtype))
