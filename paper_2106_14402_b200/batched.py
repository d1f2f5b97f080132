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
from .spgemm import DeviceCsc, Semiring, SpGemmAlg, local_spgemm, symbolic_nnz

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
