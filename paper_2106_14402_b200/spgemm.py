"""Host-side mirror of the reference's local SpGEMM interface.

Reference: /root/reference/proj/core/include/slap/spgemm.hpp and
semiring.hpp.  Same names and argument meaning:

    estimate_flops(a, b)                          spgemm.hpp:68-88
    symbolic_nnz(a, b, threads=1)                 spgemm.hpp:118-138
    local_spgemm(a, b, sr, alg=hybrid, threads=1) spgemm.hpp:275-330
    spgemm_alg_from_name(s)                       spgemm.hpp:19-24

and the same error behaviour (DimError on inner-dimension mismatch,
InternalError when numeric and symbolic counts disagree).  All arithmetic runs
in libslapcu.so on the GPU; `threads` is accepted for signature parity and
ignored.  torch is used only for device memory and the current CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import errors as E


# ----------------------------------------------------------------- semirings


@dataclass(frozen=True)
class Semiring:
    """One of the reference's built-in semirings (semiring.hpp:36-93) at a
    concrete element type.  `id` is the slapcu_semiring value."""

    id: int
    name: str
    dtype: str  # "f64" | "f32" | "i64" | "i32" | "u8"

    @property
    def np_dtype(self):
        return {"f64": np.float64, "f32": np.float32, "i64": np.int64, "i32": np.int32, "u8": np.uint8}[self.dtype]

    @property
    def torch_dtype(self):
        return {"f64": torch.float64, "f32": torch.float32, "i64": torch.int64, "i32": torch.int32,
                "u8": torch.uint8}[self.dtype]

    @property
    def exact(self) -> bool:
        return self.dtype not in ("f64", "f32") or self.name == "min_plus"

    def zero(self):
        """semiring zero() (identity of add)."""
        if self.name == "plus_times":
            return self.np_dtype(0)
        if self.name == "or_and":
            return np.uint8(0)
        if self.dtype == "i32":
            return np.int32(np.iinfo(np.int32).max)
        return np.float64(np.inf)

    def add(self, a, b):
        if self.name == "plus_times":
            return a + b
        if self.name == "or_and":
            return np.uint8(1 if (a or b) else 0)
        return a if a < b else b

    def multiply(self, a, b):
        if self.name == "plus_times":
            return a * b
        if self.name == "or_and":
            return np.uint8(1 if (a and b) else 0)
        return a + b


PlusTimesF64 = Semiring(L.PLUS_TIMES_F64, "plus_times", "f64")
PlusTimesF32 = Semiring(L.PLUS_TIMES_F32, "plus_times", "f32")
PlusTimesI64 = Semiring(L.PLUS_TIMES_I64, "plus_times", "i64")
MinPlusI32 = Semiring(L.MIN_PLUS_I32, "min_plus", "i32")
MinPlusF64 = Semiring(L.MIN_PLUS_F64, "min_plus", "f64")
OrAnd = Semiring(L.OR_AND_U8, "or_and", "u8")
SEMIRINGS = {s.id: s for s in (PlusTimesF64, PlusTimesF32, PlusTimesI64, MinPlusI32, MinPlusF64, OrAnd)}


def semiring_from_name(name: str, dtype: str = "") -> Semiring:
    """semiring.cpp builtin_semiring, extended with an element type."""
    out = C.c_int(0)
    st = L.load().slapcu_semiring_from_name(name.encode(), dtype.encode(), C.byref(out))
    if st != L.OK:
        raise E.NameError_(f"unknown semiring '{name}' with dtype '{dtype}'")
    return SEMIRINGS[out.value]


class SpGemmAlg(enum.IntEnum):
    """spgemm.hpp:17 SpGemmAlg (GPU accumulator policies, same outputs)."""

    heap = L.ALG_HEAP
    hash = L.ALG_HASH
    hybrid = L.ALG_HYBRID


def spgemm_alg_from_name(s: str) -> SpGemmAlg:
    """spgemm.hpp:19-24."""
    try:
        return SpGemmAlg[s]
    except KeyError:
        raise E.NameError_(f"unknown spgemm algorithm '{s}'") from None


# ------------------------------------------------------------------ matrices


@dataclass
class CscMatrix:
    """Host CSC (reference CscMatrix, local_matrix.hpp:26-82) with 64-bit
    column pointers."""

    nrows: int
    ncols: int
    colptr: np.ndarray  # int64 [ncols+1]
    rowids: np.ndarray  # int32 [nnz]
    vals: np.ndarray | None = None

    @property
    def nnz(self) -> int:
        return int(self.colptr[-1]) if len(self.colptr) else 0

    def to_device(self, device=None) -> "DeviceCsc":
        dev = device or torch.device("cuda", torch.cuda.current_device())
        return DeviceCsc(
            self.nrows,
            self.ncols,
            torch.from_numpy(np.ascontiguousarray(self.colptr, np.int64)).to(dev),
            torch.from_numpy(np.ascontiguousarray(self.rowids, np.int32)).to(dev),
            None if self.vals is None else torch.from_numpy(np.ascontiguousarray(self.vals)).to(dev),
        )

    def column(self, j):
        s, e = int(self.colptr[j]), int(self.colptr[j + 1])
        return self.rowids[s:e], (None if self.vals is None else self.vals[s:e])

    @staticmethod
    def from_triples(nrows, ncols, rows, cols, vals, add=None) -> "CscMatrix":
        """build_csc (local_matrix.hpp:194-204): duplicates combined with `add`
        in input order (stable); keep-first when add is None."""
        rows = np.asarray(rows, np.int64)
        cols = np.asarray(cols, np.int64)
        vals = np.asarray(vals)
        if len(rows) and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0 or cols.max() >= ncols):
            raise E.IndexError_("triple outside the matrix")
        order = np.lexsort((np.arange(len(rows)), rows, cols))
        r, c, v = rows[order], cols[order], vals[order]
        out_r, out_c, out_v = [], [], []
        if add is None:
            keep = np.ones(len(r), bool)
            if len(r):
                keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            out_r, out_c, out_v = r[keep], c[keep], v[keep]
        else:
            for k in range(len(r)):
                if out_r and out_r[-1] == r[k] and out_c[-1] == c[k]:
                    out_v[-1] = add(out_v[-1], v[k])
                else:
                    out_r.append(r[k])
                    out_c.append(c[k])
                    out_v.append(v[k])
            out_r, out_c, out_v = np.asarray(out_r, np.int64), np.asarray(out_c, np.int64), np.asarray(out_v, vals.dtype)
        colptr = np.zeros(ncols + 1, np.int64)
        np.add.at(colptr, np.asarray(out_c, np.int64) + 1, 1)
        return CscMatrix(nrows, ncols, np.cumsum(colptr).astype(np.int64), np.asarray(out_r, np.int32),
                         np.asarray(out_v, vals.dtype))

    def to_triples(self):
        cols = np.repeat(np.arange(self.ncols, dtype=np.int64), np.diff(self.colptr))
        return self.rowids.astype(np.int64), cols, self.vals


@dataclass
class DeviceCsc:
    """Device CSC: torch tensors on one GPU (int64 colptr, int32 rowids)."""

    nrows: int
    ncols: int
    colptr: torch.Tensor
    rowids: torch.Tensor
    vals: torch.Tensor | None = None

    @property
    def nnz(self) -> int:
        return int(self.rowids.numel())

    def view(self) -> L.CscView:
        return L.CscView(
            self.nrows,
            self.ncols,
            self.nnz,
            self.colptr.data_ptr(),
            self.rowids.data_ptr() if self.nnz else None,
            None if self.vals is None or self.nnz == 0 else self.vals.data_ptr(),
        )

    def to_host(self) -> CscMatrix:
        return CscMatrix(
            self.nrows,
            self.ncols,
            self.colptr.cpu().numpy(),
            self.rowids.cpu().numpy(),
            None if self.vals is None else self.vals.cpu().numpy(),
        )

    def with_vals(self, vals) -> "DeviceCsc":
        return DeviceCsc(self.nrows, self.ncols, self.colptr, self.rowids, vals)


# ------------------------------------------------------------------- context


class Context:
    """One slapcu_ctx: a device, the current torch stream, the workspace."""

    def __init__(self, device: int | None = None, stream: torch.cuda.Stream | None = None):
        self.lib = L.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream
        h = C.c_void_p()
        s = None if stream is None else stream.cuda_stream
        with torch.cuda.device(self.device):
            st = self.lib.slapcu_ctx_create(C.byref(h), self.device, s)
        if st != L.OK:
            raise E.BY_STATUS.get(st, E.Error)("slapcu_ctx_create failed")
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.slapcu_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def sync_stream(self):
        """Point the context at torch's current stream on its device."""
        s = torch.cuda.current_stream(self.device) if self.stream is None else self.stream
        self.lib.slapcu_ctx_set_stream(self.h, s.cuda_stream)

    def check(self, st: int, what: str = ""):
        if st != L.OK:
            msg = self.lib.slapcu_ctx_last_error(self.h).decode(errors="replace")
            raise E.BY_STATUS.get(st, E.Error)(f"{what}: {msg}" if what else msg)

    def set_option(self, opt: int, value: int):
        self.check(self.lib.slapcu_ctx_set_option(self.h, opt, int(value)), "set_option")

    @property
    def launches(self) -> int:
        return int(self.lib.slapcu_ctx_kernel_launches(self.h))

    def kernel_stats(self) -> dict:
        """Per-kernel-class {name: (launches, ms)} (needs OPT_PROFILE=1)."""
        out = {}
        for k, name in enumerate(L.KERNEL_CLASSES):
            n, ms = C.c_int64(), C.c_double()
            self.check(self.lib.slapcu_ctx_kernel_stats(self.h, k, C.byref(n), C.byref(ms)), "kernel_stats")
            out[name] = (int(n.value), float(ms.value))
        return out

    def reset_stats(self):
        self.check(self.lib.slapcu_ctx_reset_stats(self.h), "reset_stats")

    def invalidate(self):
        """Drops the per-operand caches (slapcu_ctx_invalidate)."""
        self.check(self.lib.slapcu_ctx_invalidate(self.h), "invalidate")

    def last_phase_ms(self):
        a, b = C.c_float(), C.c_float()
        self.lib.slapcu_ctx_last_phase_ms(self.h, C.byref(a), C.byref(b))
        return a.value, b.value


_tls = threading.local()


def default_context() -> Context:
    dev = torch.cuda.current_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if dev not in ctxs:
        ctxs[dev] = Context(dev)
    ctx = ctxs[dev]
    ctx.sync_stream()
    return ctx


def _ctx(ctx):
    if ctx is None:
        return default_context()
    ctx.sync_stream()
    return ctx


def _dev(m) -> DeviceCsc:
    if isinstance(m, DeviceCsc):
        return m
    if isinstance(m, CscMatrix):
        return m.to_device()
    raise TypeError(f"expected CscMatrix or DeviceCsc, got {type(m)}")


def _sr(sr) -> Semiring:
    if isinstance(sr, Semiring):
        return sr
    if isinstance(sr, int):
        return SEMIRINGS[sr]
    raise TypeError("semiring must be a Semiring")


def _from_out(ctx: Context, o: L.CscOut, sr: Semiring | None) -> DeviceCsc:
    """Copies a library-allocated CSC into torch tensors and frees it."""
    dev = torch.device("cuda", ctx.device)
    n, nnz = int(o.ncols), int(o.nnz)
    cp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    rw = torch.empty(nnz, dtype=torch.int32, device=dev)
    vals = None
    cudart = L.cudart()
    stream = torch.cuda.current_stream(ctx.device)

    def copy(dst, src_ptr, nbytes):
        if nbytes:
            res = cudart.cudaMemcpyAsync(C.c_void_p(dst.data_ptr()), C.c_void_p(src_ptr), C.c_size_t(nbytes), 3,
                                         C.c_void_p(stream.cuda_stream))
            if int(res) != 0:
                raise E.CudaError(f"cudaMemcpyAsync failed ({int(res)})")

    copy(cp, o.colptr, 8 * (n + 1))
    copy(rw, o.rowids, 4 * nnz)
    if o.vals and sr is not None:
        vals = torch.empty(nnz, dtype=sr.torch_dtype, device=dev)
        copy(vals, o.vals, vals.element_size() * nnz)
    ctx.check(ctx.lib.slapcu_csc_free(ctx.h, C.byref(o)), "csc_free")
    return DeviceCsc(int(o.nrows), n, cp, rw, vals)


# ------------------------------------------------------------- the 3 phases


def estimate_flops(a, b, ctx: Context | None = None):
    """spgemm.hpp:68-88 -> (total_flops, per-column int64 tensor)."""
    ctx = _ctx(ctx)
    A, B = _dev(a), _dev(b)
    per = torch.empty(B.ncols, dtype=torch.int64, device=B.colptr.device)
    tot = C.c_int64()
    ctx.check(ctx.lib.slapcu_estimate_flops(ctx.h, C.byref(A.view()), C.byref(B.view()), per.data_ptr() if B.ncols else None,
                                            C.byref(tot)), "estimate_flops")
    return int(tot.value), per


def symbolic_nnz(a, b, threads: int = 1, alg=SpGemmAlg.hybrid, ctx: Context | None = None):
    """spgemm.hpp:118-138 -> per-column exact output counts (int64 tensor)."""
    ctx = _ctx(ctx)
    A, B = _dev(a), _dev(b)
    cp = torch.empty(B.ncols + 1, dtype=torch.int64, device=B.colptr.device)
    nnz = C.c_int64()
    ctx.check(ctx.lib.slapcu_spgemm_symbolic(ctx.h, C.byref(A.view()), C.byref(B.view()), int(alg), cp.data_ptr(),
                                             C.byref(nnz)), "symbolic")
    return cp[1:] - cp[:-1]


def local_spgemm(a, b, sr: Semiring, alg=SpGemmAlg.hybrid, threads: int = 1, ctx: Context | None = None,
                 method: str = "direct"):
    """spgemm.hpp:275-330 local_spgemm.  Returns a DeviceCsc for device
    operands and a host CscMatrix for host operands (the host call runs the
    H2D copies, the three GPU phases and the D2H copies inside the library).

    method "direct" (default) writes C in place in one product pass
    (slapcu_spgemm_direct) into buffers sized by the bound
    sum_j min(flops_j, A.nrows), then trims them.
    method "fused" forms each column once (slapcu_spgemm_begin /
    _finish) and falls back to "two_pass" (slapcu_spgemm_symbolic / _numeric)
    when its staging area would not fit in half the free device memory."""
    sr = _sr(sr)
    alg = SpGemmAlg(int(alg))
    ctx = _ctx(ctx)
    if isinstance(a, CscMatrix) and isinstance(b, CscMatrix):
        return _local_spgemm_host(ctx, a, b, sr, alg)
    A, B = _dev(a), _dev(b)
    if A.ncols != B.nrows:
        raise E.DimError(f"spgemm inner dims: A is {A.nrows}x{A.ncols}, B is {B.nrows}x{B.ncols}")
    for m, nm in ((A, "A"), (B, "B")):
        if m.vals is not None and m.vals.dtype != sr.torch_dtype:
            raise TypeError(f"{nm} values are {m.vals.dtype}, semiring {sr.name} needs {sr.torch_dtype}")
    dev = B.colptr.device
    cp = torch.empty(B.ncols + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64()
    av, bv = A.view(), B.view()
    if method == "direct":
        _tot, fl = estimate_flops(A, B, ctx=ctx)
        cap = int(torch.clamp(fl, max=A.nrows).sum().item()) if B.ncols else 0
        rw = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(cap, 1), dtype=sr.torch_dtype, device=dev)
        ctx.check(ctx.lib.slapcu_spgemm_direct(ctx.h, C.byref(av), C.byref(bv), sr.id, int(alg), cap, cp.data_ptr(),
                                               rw.data_ptr(), vals.data_ptr(), C.byref(nnz)), "direct")
        n = int(nnz.value)
        if n * 10 >= cap * 9:  # the bound was (nearly) tight (compression ~1, e.g. C2): keep the buffers
            return DeviceCsc(A.nrows, B.ncols, cp, rw[:n], vals[:n])
        return DeviceCsc(A.nrows, B.ncols, cp, rw[:n].clone(), vals[:n].clone())
    if method == "fused":
        free, _ = torch.cuda.mem_get_info(dev)
        st = ctx.lib.slapcu_spgemm_begin(ctx.h, C.byref(av), C.byref(bv), sr.id, int(alg), int(free // 2),
                                         cp.data_ptr(), C.byref(nnz))
        if st == L.OK:
            n = int(nnz.value)
            rw = torch.empty(n, dtype=torch.int32, device=dev)
            vals = torch.empty(n, dtype=sr.torch_dtype, device=dev)
            ctx.check(ctx.lib.slapcu_spgemm_finish(ctx.h, C.byref(av), C.byref(bv), sr.id,
                                                   rw.data_ptr() if n else None, vals.data_ptr() if n else None),
                      "finish")
            return DeviceCsc(A.nrows, B.ncols, cp, rw, vals)
        if st != 5:  # anything but BudgetError is a real failure
            ctx.check(st, "begin")
    elif method != "two_pass":
        raise ValueError(f"unknown method {method!r}")
    ctx.check(ctx.lib.slapcu_spgemm_symbolic(ctx.h, C.byref(av), C.byref(bv), int(alg), cp.data_ptr(), C.byref(nnz)),
              "symbolic")
    n = int(nnz.value)
    rw = torch.empty(n, dtype=torch.int32, device=dev)
    vals = torch.empty(n, dtype=sr.torch_dtype, device=dev)
    ctx.check(ctx.lib.slapcu_spgemm_numeric(ctx.h, C.byref(av), C.byref(bv), sr.id, int(alg), cp.data_ptr(),
                                            rw.data_ptr() if n else None, vals.data_ptr() if n else None), "numeric")
    return DeviceCsc(A.nrows, B.ncols, cp, rw, vals)


def _host_view(m: CscMatrix, dtype, keep) -> L.CscOut:
    cp = np.ascontiguousarray(m.colptr, np.int64)
    rw = np.ascontiguousarray(m.rowids, np.int32)
    vv = np.ascontiguousarray(m.vals, dtype)
    keep += [cp, rw, vv]
    return L.CscOut(m.nrows, m.ncols, int(cp[-1]), cp.ctypes.data, rw.ctypes.data, vv.ctypes.data)


def _local_spgemm_host(ctx: Context, a: CscMatrix, b: CscMatrix, sr: Semiring, alg) -> CscMatrix:
    keep = []
    A = _host_view(a, sr.np_dtype, keep)
    B = _host_view(b, sr.np_dtype, keep)
    out = L.CscOut()
    ctx.check(ctx.lib.slapcu_spgemm_host(ctx.h, C.byref(A), C.byref(B), sr.id, int(alg), C.byref(out)), "spgemm_host")
    try:
        n, nnz = int(out.ncols), int(out.nnz)
        colptr = np.ctypeslib.as_array(C.cast(out.colptr, C.POINTER(C.c_int64)), shape=(n + 1,)).copy()
        rowids = (np.ctypeslib.as_array(C.cast(out.rowids, C.POINTER(C.c_int32)), shape=(nnz,)).copy()
                  if nnz else np.zeros(0, np.int32))
        raw = C.string_at(out.vals, nnz * np.dtype(sr.np_dtype).itemsize) if nnz else b""
        vals = np.frombuffer(raw, dtype=sr.np_dtype).copy()
    finally:
        ctx.lib.slapcu_host_free(C.byref(out))
    return CscMatrix(int(out.nrows), n, colptr, rowids, vals)


def merge(parts, sr: Semiring, ctx: Context | None = None) -> DeviceCsc:
    """The SUMMA / 3D merge (summa.hpp:156 build_dcsc over stage partials
    appended in order; local_matrix.hpp:166-188): coincident entries are
    left-folded with sr.add in part order."""
    sr = _sr(sr)
    ctx = _ctx(ctx)
    P = [_dev(p) for p in parts]
    arr = (L.CscView * len(P))(*[p.view() for p in P])
    dev = P[0].colptr.device
    cp = torch.empty(P[0].ncols + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64()
    ctx.check(ctx.lib.slapcu_merge_symbolic(ctx.h, len(P), arr, cp.data_ptr(), C.byref(nnz)), "merge_symbolic")
    n = int(nnz.value)
    rw = torch.empty(n, dtype=torch.int32, device=dev)
    vals = torch.empty(n, dtype=sr.torch_dtype, device=dev)
    ctx.check(ctx.lib.slapcu_merge_numeric(ctx.h, len(P), arr, sr.id, cp.data_ptr(), rw.data_ptr() if n else None,
                                           vals.data_ptr() if n else None), "merge_numeric")
    return DeviceCsc(P[0].nrows, P[0].ncols, cp, rw, vals)


def dcsc_to_csc(nrows, ncols, jc: torch.Tensor, cp: torch.Tensor, rowids: torch.Tensor, vals, ctx=None) -> DeviceCsc:
    """DcscMatrix (local_matrix.hpp:88-150) -> device CSC with a dense colptr."""
    ctx = _ctx(ctx)
    colptr = torch.empty(ncols + 1, dtype=torch.int64, device=rowids.device)
    jc = jc.to(torch.int32).contiguous()
    cp = cp.to(torch.int32).contiguous()
    ctx.check(ctx.lib.slapcu_dcsc_colptr(ctx.h, ncols, int(jc.numel()), jc.data_ptr() if jc.numel() else None,
                                         cp.data_ptr(), colptr.data_ptr()), "dcsc_colptr")
    return DeviceCsc(nrows, ncols, colptr, rowids, vals)


# ---------------------------------------------------------- synthetic inputs


def gen_rmat(scale: int, edge_factor: int = 16, seed: int = 1, a=0.57, b=0.19, c=0.19, d=0.05,
             ctx: Context | None = None) -> DeviceCsc:
    """algorithms.cpp:71-113 gen_rmat on the device (pattern only)."""
    ctx = _ctx(ctx)
    o = L.CscOut()
    ctx.check(ctx.lib.slapcu_gen_rmat(ctx.h, scale, edge_factor, seed, a, b, c, d, C.byref(o)), "gen_rmat")
    return _from_out(ctx, o, None)


def gen_er(n: int, draws: int, seed: int = 1, with_values=True, ctx: Context | None = None) -> DeviceCsc:
    """oracles.hpp:205-217 random_triples as an n x n ER matrix (f64 values)."""
    ctx = _ctx(ctx)
    o = L.CscOut()
    ctx.check(ctx.lib.slapcu_gen_er(ctx.h, n, draws, seed, int(with_values), C.byref(o)), "gen_er")
    return _from_out(ctx, o, PlusTimesF64 if with_values else None)


def gen_one_per_row(n: int, ncols: int, seed: int = 2, ctx: Context | None = None) -> DeviceCsc:
    ctx = _ctx(ctx)
    o = L.CscOut()
    ctx.check(ctx.lib.slapcu_gen_one_per_row(ctx.h, n, ncols, seed, C.byref(o)), "gen_one_per_row")
    return _from_out(ctx, o, PlusTimesF64)


def fill_values(m: DeviceCsc, sr: Semiring, kind: int, ctx: Context | None = None) -> DeviceCsc:
    """Value recipes of SURVEY.md 8d (0 ones, 1 U[0,1), 2 U[0,10), 3 int 1+h%255,
    4 1/deg(col), 5 int 1+h%9)."""
    sr = _sr(sr)
    ctx = _ctx(ctx)
    vals = torch.empty(m.nnz, dtype=sr.torch_dtype, device=m.colptr.device)
    if m.nnz:
        ctx.check(ctx.lib.slapcu_fill_values(ctx.h, sr.id, kind, C.byref(m.view()), vals.data_ptr()), "fill_values")
    return m.with_vals(vals)


def permute_symmetric(m: DeviceCsc, seed: int, sr: Semiring | None = None, ctx: Context | None = None) -> DeviceCsc:
    """P*A*P^T with a seed-deterministic permutation (balanced SUMMA input)."""
    ctx = _ctx(ctx)
    o = L.CscOut()
    sid = sr.id if sr is not None else 0
    v = m.view() if sr is not None else m.with_vals(None).view()
    ctx.check(ctx.lib.slapcu_permute_symmetric(ctx.h, C.byref(v), seed, sid, C.byref(o)), "permute_symmetric")
    return _from_out(ctx, o, sr)


def slice_cols(m: DeviceCsc, c0: int, c1: int, sr: Semiring | None = None, ctx: Context | None = None) -> DeviceCsc:
    """batched.hpp:43-66 slice_cols on one device block."""
    ctx = _ctx(ctx)
    o = L.CscOut()
    sid = sr.id if sr is not None else 0
    v = m.view() if sr is not None else m.with_vals(None).view()
    ctx.check(ctx.lib.slapcu_slice_cols(ctx.h, C.byref(v), sid, c0, c1, C.byref(o)), "slice_cols")
    return _from_out(ctx, o, sr)


def mcl_step(a, inflation: float = 2.0, prune_threshold: float = 1e-4, sr: Semiring | None = None,
             ctx: Context | None = None) -> DeviceCsc:
    """algorithms.cpp:267-293 mcl_step on one device: expansion A*A (direct
    single pass), inflation, pruning, column renormalisation.  Raises
    errors.StochasticityError if an input column does not sum to 1."""
    ctx = _ctx(ctx)
    A = _dev(a)
    sr = _sr(sr) if sr is not None else (PlusTimesF32 if A.vals.dtype == torch.float32 else PlusTimesF64)
    o = L.CscOut()
    ctx.check(ctx.lib.slapcu_mcl_step(ctx.h, C.byref(A.view()), sr.id, float(inflation), float(prune_threshold),
                                      C.byref(o)), "mcl_step")
    return _from_out(ctx, o, sr)


def column_checksums(m: DeviceCsc, sr: Semiring | None = None, with_values=True, ctx: Context | None = None):
    ctx = _ctx(ctx)
    sums = torch.empty(max(m.ncols, 1), dtype=torch.int64, device=m.colptr.device)
    sid = sr.id if sr is not None else 0
    ctx.check(ctx.lib.slapcu_column_checksums(ctx.h, C.byref(m.view()), sid, int(with_values and sr is not None),
                                              sums.data_ptr()), "column_checksums")
    return sums[: m.ncols]
