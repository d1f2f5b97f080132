"""Distributed SpGEMM drivers: host-side mirror of the reference's
summa2d_spgemm (summa.hpp:106-163), ca3d_spgemm (spgemm3d.hpp:21-106) and
batched_spgemm (batched.hpp:153-170) over libslapcu's NCCL drivers.

One process per GPU (torchrun).  torch.distributed is used only to share the
NCCL unique id and for host-side barriers / gathers; every data-path
collective (stage broadcasts, fiber exchange) runs inside libslapcu on NCCL
communicators of its own.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import errors as E
from . import grid as G
from .spgemm import Context, CscMatrix, DeviceCsc, Semiring, SpGemmAlg, _from_out, _sr, default_context


class NcclComm:
    """slapcu_comm spanning the ranks of the default torch.distributed group
    (the reference's world Comm, comm.hpp:178-348, on NCCL)."""

    def __init__(self, ctx: Context | None = None):
        import torch.distributed as dist

        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        uid = (C.c_char * 128)()
        if self.rank == 0:
            st = self.lib.slapcu_comm_unique_id(uid)
            if st != L.OK:
                raise E.DeadlockError("ncclGetUniqueId failed")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        buf = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        self.ctx.check(self.lib.slapcu_comm_create(C.byref(h), self.ctx.h, self.rank, self.size, buf), "comm_create")
        self.h = h

    def counters(self, kind: int):
        """comm.hpp:31-53 CommCounters: (calls, bytes) for kind 0 broadcast,
        1 alltoallv, 2 reduce, 3 allgatherv."""
        calls, nbytes = C.c_int64(), C.c_int64()
        self.lib.slapcu_comm_counters(self.h, kind, C.byref(calls), C.byref(nbytes))
        return int(calls.value), int(nbytes.value)

    def close(self):
        if getattr(self, "h", None):
            self.lib.slapcu_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class DistKernelStats:
    """summa.hpp:15-20 + device-event timings (ms)."""

    stages: int
    flops: int
    nnz_out: int
    layer_warning: bool
    ms_total: float
    ms_local: float
    ms_merge: float
    ms_exposed_bcast: float


def _stats(s: L.DistStats) -> DistKernelStats:
    return DistKernelStats(s.stages, s.flops, s.nnz_out, bool(s.layer_warning), s.ms_total, s.ms_local, s.ms_merge,
                           s.ms_exposed_bcast)


def summa2d_spgemm(a_local: DeviceCsc, b_local: DeviceCsc, sr: Semiring, comm: NcclComm,
                   alg=SpGemmAlg.hybrid, threads: int = 1, raw: bool = False):
    """Collective 2D Sparse SUMMA on a sqrt(p) x sqrt(p) grid (rank = i*q + j).
    `a_local` is A's block (i, j), `b_local` is B's block (i, j) with block
    extents from block_offsets (layout.hpp:60-66).  Returns (C block (i, j),
    stats); raw=True returns the library-owned L.CscOut instead (free with
    free_out)."""
    sr = _sr(sr)
    ctx = comm.ctx
    ctx.sync_stream()
    out = L.CscOut()
    st = L.DistStats()
    ctx.check(comm.lib.slapcu_summa2d(comm.h, C.byref(a_local.view()), C.byref(b_local.view()), sr.id, int(alg),
                                      C.byref(out), C.byref(st)), "summa2d")
    if raw:
        return out, _stats(st)
    return _from_out(ctx, out, sr), _stats(st)


def ca3d_spgemm(a3_local: DeviceCsc, b3_local: DeviceCsc, sr: Semiring, comm: NcclComm, layers: int,
                alg=SpGemmAlg.hybrid, threads: int = 1, raw: bool = False):
    """Collective 3D SpGEMM on a c x q x q grid (regular variant, rank =
    l*q*q + i*q + j): A split by columns, B by rows (regular_3d_range).  The
    result is C3 block (l, i, j) (ca3d_output_range)."""
    sr = _sr(sr)
    ctx = comm.ctx
    ctx.sync_stream()
    out = L.CscOut()
    st = L.DistStats()
    ctx.check(comm.lib.slapcu_ca3d(comm.h, layers, C.byref(a3_local.view()), C.byref(b3_local.view()), sr.id,
                                   int(alg), C.byref(out), C.byref(st)), "ca3d")
    if raw:
        return out, _stats(st)
    return _from_out(ctx, out, sr), _stats(st)


def mcl_step(a_local: DeviceCsc, pr: int, pc: int, comm: NcclComm, layers: int = 1, inflation: float = 2.0,
             prune: float = 1e-4, sr: Semiring = None):
    """algorithms.cpp:267-293 mcl_step on a pr x pc grid (rank = i*pc + j,
    `a_local` = block (i, j)): expansion by the 2D SUMMA (layers <= 1) or the
    3D path (device redistribute_3d x2 -> ca3d -> redistribute_2d), then the
    inflation / prune / renormalisation epilogue with column sums reduced
    over the grid column -- all on the device.  Returns this rank's block."""
    from .spgemm import PlusTimesF64

    sr = _sr(sr or PlusTimesF64)
    ctx = comm.ctx
    ctx.sync_stream()
    out = L.CscOut()
    ctx.check(comm.lib.slapcu_mcl_step_dist(comm.h, pr, pc, layers, C.byref(a_local.view()), sr.id, float(inflation),
                                            float(prune), C.byref(out)), "mcl_step_dist")
    return _from_out(ctx, out, sr)


def free_out(ctx: Context, out: L.CscOut):
    ctx.check(ctx.lib.slapcu_csc_free(ctx.h, C.byref(out)), "csc_free")


# ------------------------------------------------------- device block views


def column_window(m: DeviceCsc, c0: int, c1: int) -> DeviceCsc:
    """Columns [c0, c1) of a device CSC without copying (colptr view; entry
    arrays shared).  The library accepts offset colptrs everywhere."""
    return DeviceCsc(m.nrows, c1 - c0, m.colptr[c0:c1 + 1], m.rowids, m.vals)


def device_block(m: DeviceCsc, r0: int, rl: int, c0: int, cl: int) -> DeviceCsc:
    """Block rows [r0, r0+rl) x cols [c0, c0+cl) with block-local indices, as a
    new device CSC (setup-time helper; torch ops on the device)."""
    cp = m.colptr[c0:c0 + cl + 1]
    lo, hi = int(cp[0]), int(cp[-1])
    rw = m.rowids[lo:hi]
    counts = (cp[1:] - cp[:-1])
    col = torch.repeat_interleave(torch.arange(cl, device=rw.device), counts)
    keep = (rw >= r0) & (rw < r0 + rl)
    col = col[keep]
    new_rw = (rw[keep] - r0).to(torch.int32)
    new_v = None if m.vals is None else m.vals[lo:hi][keep]
    cnt = torch.bincount(col, minlength=cl)
    colptr = torch.zeros(cl + 1, dtype=torch.int64, device=rw.device)
    colptr[1:] = torch.cumsum(cnt, 0)
    return DeviceCsc(rl, cl, colptr, new_rw.contiguous(), None if new_v is None else new_v.contiguous())


def block_2d(m: DeviceCsc, q: int, rank: int) -> DeviceCsc:
    r0, rl, c0, cl = G.block2d_range(m.nrows, m.ncols, q, q, rank // q, rank % q)
    return device_block(m, r0, rl, c0, cl)


def block_3d(m: DeviceCsc, c: int, q: int, rank: int, split: str) -> DeviceCsc:
    g = G.Grid3D(c, q, rank)
    l, i, j = g.coords
    r0, rl, c0, cl = G.regular_3d_range(m.nrows, m.ncols, c, q, split, l, i, j)
    return device_block(m, r0, rl, c0, cl)


def gather_to_host(local: DeviceCsc, row_start: int, col_start: int, nrows: int, ncols: int) -> CscMatrix | None:
    """gather_matrix (dist_matrix.hpp:121-145): rank 0 receives every block
    and assembles the global CSC (test / validation helper)."""
    import torch.distributed as dist

    h = local.to_host()
    mine = (row_start, col_start, h.colptr, h.rowids, h.vals)
    parts = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(mine, parts, dst=0)
    if dist.get_rank() != 0:
        return None
    cp, rw, vv = G.assemble(nrows, ncols, parts)
    return CscMatrix(nrows, ncols, cp, rw, vv.astype(h.vals.dtype) if h.vals is not None else vv)


# ------------------------------------------------------------ redistribution


def _tiling_struct(t: G.Tiling):
    rc = np.ascontiguousarray(t.row_cuts, np.int64)
    cc = np.ascontiguousarray(t.col_cuts, np.int64)
    ow = np.ascontiguousarray(t.owner, np.int32)
    st = L.Tiling(t.nr, t.nc, rc.ctypes.data, cc.ctypes.data, ow.ctypes.data)
    return st, (rc, cc, ow)


_COMBINE = {"first": 0, "add": 1}


def redistribute(local: DeviceCsc, row_start: int, col_start: int, nrows: int, ncols: int, sr: Semiring,
                 comm: NcclComm, target: G.Tiling, combine: str = "first"):
    """Collective: re-route this rank's block (global offsets row_start /
    col_start) to the target tiling; returns (tile as DeviceCsc, row_start,
    col_start) of this rank's target tile.  slapcu_redistribute."""
    sr = _sr(sr)
    ctx = comm.ctx
    ctx.sync_stream()
    tl, keep = _tiling_struct(target)
    out = L.CscOut()
    rs, cs = C.c_int64(), C.c_int64()
    ctx.check(comm.lib.slapcu_redistribute(comm.h, C.byref(local.view()), row_start, col_start, nrows, ncols, sr.id,
                                           C.byref(tl), _COMBINE[combine], C.byref(out), C.byref(rs), C.byref(cs)),
              "redistribute")
    del keep
    return _from_out(ctx, out, sr), int(rs.value), int(cs.value)


def distribute_triples(rows: torch.Tensor, cols: torch.Tensor, vals: torch.Tensor, nrows: int, ncols: int,
                       sr: Semiring, comm: NcclComm, pr: int | None = None, pc: int | None = None,
                       combine: str = "first", target: G.Tiling | None = None):
    """dist_matrix.hpp:89-119 distribute_triples: this rank's global COO
    triples (device int64 rows / cols, values of the semiring type) routed to
    the pr x pc block layout (default sqrt(p) x sqrt(p)); duplicates keep the
    first (combine="first") or fold with the semiring add ("add").  Returns
    (block, row_start, col_start)."""
    sr = _sr(sr)
    if target is None:
        if pr is None or pc is None:
            q = G.isqrt_exact(comm.size)
            pr, pc = q, q
        if pr * pc != comm.size:
            raise E.ShapeError(f"{pr}x{pc} grid on {comm.size} ranks")
        target = G.tiling_2d(nrows, ncols, pr, pc)
    ctx = comm.ctx
    rows = rows.to(torch.int64).contiguous()
    cols = cols.to(torch.int64).contiguous()
    vals = vals.contiguous()
    if vals.dtype != sr.torch_dtype:
        raise E.ShapeError(f"values must be {sr.torch_dtype} for {sr.name}")
    ctx.sync_stream()
    tl, keep = _tiling_struct(target)
    out = L.CscOut()
    rs, cs = C.c_int64(), C.c_int64()
    ctx.check(comm.lib.slapcu_distribute_triples(comm.h, rows.numel(), rows.data_ptr(), cols.data_ptr(),
                                                 vals.data_ptr(), nrows, ncols, sr.id, C.byref(tl),
                                                 _COMBINE[combine], C.byref(out), C.byref(rs), C.byref(cs)),
              "distribute_triples")
    del keep
    return _from_out(ctx, out, sr), int(rs.value), int(cs.value)


def redistribute_3d(a2: DeviceCsc, nrows: int, ncols: int, sr: Semiring, comm: NcclComm, layers: int,
                    split: str, pr: int | None = None, pc: int | None = None):
    """dist_matrix3d.hpp:117-170 redistribute_3d (regular variant): this
    rank's block of the pr x pc 2D layout (default sqrt(p) x sqrt(p)) to its
    block of the c x q x q layout split by `split` ("cols" for A, "rows" for
    B).  Returns (block, row_start, col_start)."""
    p = comm.size
    if pr is None or pc is None:
        q2 = G.isqrt_exact(p)
        pr, pc = q2, q2
    if pr * pc != p:
        raise E.ShapeError(f"3D grid has {p} ranks, matrix lives on {pr * pc}")
    g = G.Grid3D.make(p, layers, comm.rank)
    r0, _, c0, _ = G.block2d_range(nrows, ncols, pr, pc, comm.rank // pc, comm.rank % pc)
    return redistribute(a2, r0, c0, nrows, ncols, sr, comm, G.tiling_3d(nrows, ncols, layers, g.q, split))


def redistribute_2d(a3: DeviceCsc, row_start: int, col_start: int, nrows: int, ncols: int, sr: Semiring,
                    comm: NcclComm, pr: int | None = None, pc: int | None = None):
    """dist_matrix3d.hpp:250-261 redistribute_2d: any block with known global
    offsets (a 3D operand, or a ca3d_spgemm output at ca3d_output_range) back
    to the pr x pc 2D layout.  Returns (block, row_start, col_start)."""
    p = comm.size
    if pr is None or pc is None:
        q2 = G.isqrt_exact(p)
        pr, pc = q2, q2
    if pr * pc != p:
        raise E.ShapeError(f"{pr}x{pc} grid on {p} ranks")
    return redistribute(a3, row_start, col_start, nrows, ncols, sr, comm, G.tiling_2d(nrows, ncols, pr, pc))


# ------------------------------------------------------- CB2B binary I/O


def binary_header(path: str, ctx: Context | None = None):
    """(nrows, ncols, nnz) of a CB2B file (binary_io.hpp:10-28)."""
    ctx = ctx or default_context()
    m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    st = ctx.lib.slapcu_cb2b_header(path.encode(), C.byref(m), C.byref(n), C.byref(nnz))
    if st != L.OK:
        raise E.BY_STATUS.get(st, E.Error)(f"{path}")
    return int(m.value), int(n.value), int(nnz.value)


def write_binary(local: DeviceCsc, row_start: int, col_start: int, nrows: int, ncols: int, comm: NcclComm,
                 path: str):
    """binary_io.cpp write_binary: collective; f64 values."""
    if local.vals is None or local.vals.dtype != torch.float64:
        raise E.InvalidArgument("CB2B files hold f64 values")
    ctx = comm.ctx
    ctx.sync_stream()
    ctx.check(comm.lib.slapcu_write_cb2b(comm.h, path.encode(), C.byref(local.view()), row_start, col_start, nrows,
                                         ncols), "write_cb2b")


def read_binary(path: str, comm: NcclComm, pr: int | None = None, pc: int | None = None):
    """binary_io.cpp read_binary onto the pr x pc layout (default
    sqrt(p) x sqrt(p)): returns (block f64, row_start, col_start, nrows, ncols)."""
    if pr is None or pc is None:
        q = G.isqrt_exact(comm.size)
        pr, pc = q, q
    ctx = comm.ctx
    ctx.sync_stream()
    out = L.CscOut()
    rs, cs, m, n = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    ctx.check(comm.lib.slapcu_read_cb2b(comm.h, path.encode(), pr, pc, C.byref(out), C.byref(rs), C.byref(cs),
                                        C.byref(m), C.byref(n)), "read_cb2b")
    from .spgemm import PlusTimesF64

    return _from_out(ctx, out, PlusTimesF64), int(rs.value), int(cs.value), int(m.value), int(n.value)
