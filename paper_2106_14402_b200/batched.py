"""Column batching for products whose output does not fit device memory at
once -- host mirror of the reference's batched.hpp (BatchPlan,
kBatchEntryBytes, plan_batches_by_count, plan_batches_by_budget,
batched_spgemm; batched.hpp:14-170).

Batch r computes A * B(:, range_r) and hands it to a consumer, so the batch
outputs concatenate to the unbatched product.  On the GPU a column range of
B is a colptr window (no copy); the exact per-column counts for budget
planning come from the device symbolic pass (the reference runs a Boolean
SUMMA for them, batched.hpp:70-117).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import errors as E
from .spgemm import CscMatrix, DeviceCsc, Semiring, SpGemmAlg, _ctx, _host_view, _sr, local_spgemm, symbolic_nnz

K_BATCH_ENTRY_BYTES = 16  # batched.hpp:23 kBatchEntryBytes (value + index)


@dataclass
class BatchPlan:
    """batched.hpp:14-21."""

    col_ranges: list = field(default_factory=list)  # [(start, end)]
    est_entries: list = field(default_factory=list)

    def batches(self) -> int:
        return len(self.col_ranges)


def plan_batches_by_count(ncols: int, b: int) -> BatchPlan:
    """batched.hpp:25-37: b ranges, remainder spread one per range from the front."""
    if b < 1:
        raise E.ShapeError("batch count must be >= 1")
    q, r = divmod(ncols, b)
    plan, s = BatchPlan(), 0
    for i in range(b):
        w = q + (1 if i < r else 0)
        plan.col_ranges.append((s, s + w))
        plan.est_entries.append(0)
        s += w
    return plan


def plan_from_counts(counts, budget_bytes: int, per_entry: int = K_BATCH_ENTRY_BYTES) -> BatchPlan:
    """batched.hpp:131-147: fewest contiguous ranges with count*per_entry <=
    budget; BudgetError when one column alone exceeds it."""
    if budget_bytes <= 0:
        raise E.BudgetError("memory budget must be positive")
    plan, start, cur = BatchPlan(), 0, 0
    counts = np.asarray(counts, dtype=np.int64)
    for j, cnt in enumerate(counts.tolist()):
        cost = cnt * per_entry
        if cost > budget_bytes:
            raise E.BudgetError(f"output column {j} alone needs {cost} bytes, budget is {budget_bytes}")
        if cur + cost > budget_bytes:
            plan.col_ranges.append((start, j))
            plan.est_entries.append(cur // per_entry)
            start, cur = j, 0
        cur += cost
    plan.col_ranges.append((start, len(counts)))
    plan.est_entries.append(cur // per_entry)
    return plan


def plan_batches_by_budget(a: DeviceCsc, b: DeviceCsc, budget_bytes: int, threads: int = 1) -> BatchPlan:
    """batched.hpp:122-148 with exact per-column counts from the GPU symbolic
    pass (the reference's dist_symbolic_col_nnz)."""
    if budget_bytes <= 0:
        raise E.BudgetError("memory budget must be positive")
    counts = symbolic_nnz(a, b).cpu().numpy()
    return plan_from_counts(counts, budget_bytes)


def column_window(m: DeviceCsc, c0: int, c1: int) -> DeviceCsc:
    """B(:, [c0, c1)) as a view (batched.hpp:43-66 slice_cols without a copy)."""
    return DeviceCsc(m.nrows, c1 - c0, m.colptr[c0:c1 + 1], m.rowids, m.vals)


def batched_spgemm(a: DeviceCsc, b: DeviceCsc, plan: BatchPlan, sr: Semiring, alg=SpGemmAlg.hybrid, threads: int = 1,
                   consumer=None, ctx=None):
    """batched.hpp:153-170: validates that the plan partitions B's columns in
    order (ShapeError otherwise), then calls consumer(r, s, e, C_r) once per
    range in order.  Returns the list of batch results when no consumer is
    given."""
    if plan.batches() < 1:
        raise E.ShapeError("batch plan is empty")
    expect = 0
    for s, e in plan.col_ranges:
        if s != expect or e < s:
            raise E.ShapeError("batch ranges must partition B's columns in order")
        expect = e
    if expect != b.ncols:
        raise E.ShapeError("batch ranges must cover all columns of B")
    out = []
    for r, (s, e) in enumerate(plan.col_ranges):
        cr = local_spgemm(a, column_window(b, s, e), sr, alg, threads, ctx=ctx)
        if consumer is not None:
            consumer(r, s, e, cr)
        else:
            out.append(cr)
    return None if consumer is not None else out


def batched_spgemm_host(a: CscMatrix, b: CscMatrix, sr: Semiring, alg=SpGemmAlg.hybrid, plan: BatchPlan | None = None,
                        budget_bytes: int = 0, consumer=None, ctx=None) -> int:
    """batched.hpp:153-170 for HOST operands through one library call
    (slapcu_batched_spgemm_host): A and B go to the device once, every batch
    product is read back into pinned host memory (batch r+1's product overlaps
    batch r's read-back) and consumer(r, s, e, C_r) runs with C_r a host
    CscMatrix whose arrays are views of library-owned pinned buffers, valid
    during the call only (copy what you keep).  Without a plan the library
    plans by `budget_bytes` on the output bound.  Returns nnz(C)."""
    import ctypes as C

    from . import _lib as L

    sr = _sr(sr)
    ctx = _ctx(ctx)
    keep = []
    A = _host_view(a, sr.np_dtype, keep)
    B = _host_view(b, sr.np_dtype, keep)
    rng = None
    nr = 0
    if plan is not None:
        rng = np.asarray(plan.col_ranges, dtype=np.int64).reshape(-1)
        nr = plan.batches()
    err = []
    vs = np.dtype(sr.np_dtype).itemsize

    def _cb(_user, r, s, e, cp):
        try:
            if consumer is not None:
                m = cp.contents
                n, nz = int(m.ncols), int(m.nnz)
                colptr = np.ctypeslib.as_array(C.cast(m.colptr, C.POINTER(C.c_int64)), shape=(n + 1,))
                rows = (np.ctypeslib.as_array(C.cast(m.rowids, C.POINTER(C.c_int32)), shape=(nz,)) if nz
                        else np.zeros(0, np.int32))
                vals = (np.frombuffer((C.c_char * (nz * vs)).from_address(m.vals), dtype=sr.np_dtype) if nz
                        else np.zeros(0, sr.np_dtype))
                consumer(int(r), int(s), int(e), CscMatrix(int(m.nrows), n, colptr, rows, vals))
            return 0
        except Exception as ex:  # surfaced after the call returns
            err.append(ex)
            return 1

    cb = L.BatchConsumer(_cb)
    tot = C.c_int64()
    st = ctx.lib.slapcu_batched_spgemm_host(ctx.h, C.byref(A), C.byref(B), sr.id, int(SpGemmAlg(int(alg))), nr,
                                            rng.ctypes.data if rng is not None else None, int(budget_bytes), cb, None,
                                            C.byref(tot))
    if err:
        raise err[0]
    ctx.check(st, "batched_spgemm_host")
    return int(tot.value)
