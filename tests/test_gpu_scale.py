"""Parity at the BASELINE configs' scale (SURVEY.md 8d "Parity at C3 scale"),
through the benchmark's production path: column batches of one
slapcu_spgemm_direct call each into buffers sized by the flops bound.

* C4's matrix (R-MAT s18 ef16, nnz(C) = 2.96e9 > 2^31): OrAnd and MinPlus
  int32 bit-exact, PlusTimes fp32 (1/deg values, rel 1e-5), on four 256-column
  slices at the survey's probe8 offsets taken out of the batched output (the
  late slices sit at output offsets above 2^31), against the compiled
  reference's local_spgemm of the same columns; per-column nnz of EVERY column
  against the (independent) symbolic kernels.
* C2 (Erdos-Renyi 2^20, d = 8, fp64, rel 1e-12) and C5 (tall-skinny, fp64,
  the ESC path: bit-exact) on full products / slices.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from tests.helpers import TOL, rel_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
if not oracle.ref_available():
    pytest.skip("oracle/_ref/libslapref.so not built", allow_module_level=True)

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402


def offsets(n, w):
    return [0, min(n // 4 + 12345, n - w), min(n // 2 + 777, n - w), n - w]


def batched_slices(A, B, sr, slices, budget=None):
    """The bench's step: column batches by the flops bound, one direct call
    each; returns per-slice (colptr, rows, vals, max output offset) and the
    per-column nnz of every column."""
    ctx = P.Context()
    if budget is None:  # one batch where it fits, so late columns sit at output offsets > 2^31
        free, _ = torch.cuda.mem_get_info()
        budget = int(0.6 * free)
    _, fl = P.estimate_flops(A, B, ctx=ctx)
    bound = torch.clamp(fl, max=A.nrows).cpu().numpy()
    vs = np.dtype(sr.np_dtype).itemsize
    ranges, start, cur = [], 0, 0
    for j, b in enumerate(bound.tolist()):
        if cur + b * (4 + vs) > budget and j > start:
            ranges.append((start, j))
            start, cur = j, 0
        cur += b * (4 + vs)
    ranges.append((start, len(bound)))
    cap = max(int(bound[s:e].sum()) for s, e in ranges)
    maxc = max(e - s for s, e in ranges)
    dev = A.colptr.device
    cp = torch.empty(maxc + 1, dtype=torch.int64, device=dev)
    rw = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    vv = torch.empty(max(cap, 1), dtype=sr.torch_dtype, device=dev)
    av = A.view()
    counts = np.zeros(B.ncols, np.int64)
    got = {s: [] for s in slices}
    for s, e in ranges:
        w = L.CscView(B.nrows, e - s, B.nnz, B.colptr.data_ptr() + 8 * s, B.rowids.data_ptr(), B.vals.data_ptr())
        nz = C.c_int64()
        ctx.check(ctx.lib.slapcu_spgemm_direct(ctx.h, C.byref(av), C.byref(w), sr.id, 2, cap, cp.data_ptr(),
                                               rw.data_ptr(), vv.data_ptr(), C.byref(nz)), "direct")
        h = cp[: e - s + 1].cpu().numpy()
        counts[s:e] = np.diff(h)
        for (c0, c1) in slices:
            p0, p1 = max(c0, s), min(c1, e)
            if p0 < p1:
                lo, hi = int(h[p0 - s]), int(h[p1 - s])
                got[(c0, c1)].append((h[p0 - s:p1 - s + 1] - lo, rw[lo:hi].cpu().numpy(), vv[lo:hi].cpu().numpy(), lo))
    out = {}
    for key, parts in got.items():
        cps, base = [np.zeros(1, np.int64)], 0
        for cpp, _, _, _ in parts:
            cps.append(cpp[1:] + base)
            base += int(cpp[-1])
        out[key] = (np.concatenate(cps), np.concatenate([p[1] for p in parts]), np.concatenate([p[2] for p in parts]),
                    max(p[3] for p in parts))
    return out, counts


def check(sr, got, want, what):
    cp, rows, vals, _ = got
    assert np.array_equal(cp, want.colptr), f"{what}: colptr"
    assert np.array_equal(rows, want.rowids), f"{what}: rowids"
    if sr.id in TOL:
        ok = rel_close(vals, np.asarray(want.vals), TOL[sr.id])
        assert ok.all(), f"{what}: {int((~ok).sum())} values outside rel {TOL[sr.id]}"
    else:
        assert vals.tobytes() == np.asarray(want.vals, sr.np_dtype).tobytes(), f"{what}: values not bit-exact"


@pytest.mark.parametrize("sr,kind", [(P.OrAnd, 0), (P.MinPlusI32, 3), (P.PlusTimesF32, 4)],
                         ids=["or_and", "min_plus_i32", "plus_times_f32"])
def test_rmat_s18_slices_and_counts(sr, kind):
    A = P.fill_values(P.gen_rmat(18, 16, 1), sr, kind)
    n = A.ncols
    slices = [(c0, c0 + 256) for c0 in offsets(n, 256)]
    got, counts = batched_slices(A, A, sr, slices)
    sym = P.symbolic_nnz(A, A).cpu().numpy()
    assert np.array_equal(counts, sym), "per-column nnz of the batched direct product vs the symbolic kernels"
    assert int(counts.sum()) == 2962606472  # SURVEY.md Appendix A, reference-measured
    h = A.to_host()
    ao = oracle.Csc(n, n, h.colptr, h.rowids, h.vals)
    R = oracle.ref()
    for (c0, c1) in slices:
        _, _, _, want = R.time_local_spgemm(sr.id, ao, ao, c0, c1, 16, want_result=True)
        check(sr, got[(c0, c1)], want, f"s18 {sr.name} cols [{c0},{c1})")
    assert max(got[s][3] for s in slices) > 2**31, "a slice beyond output offset 2^31"


def test_c2_er_fp64_full():
    sr = P.PlusTimesF64
    A = P.gen_er(1 << 20, 8 << 20, 1)
    n = A.ncols
    slices = [(0, n)]
    got, _ = batched_slices(A, A, sr, slices)
    h = A.to_host()
    ao = oracle.Csc(n, n, h.colptr, h.rowids, h.vals)
    want = oracle.ref().local_spgemm(sr.id, ao, ao, threads=16)
    check(sr, got[(0, n)], want, "C2")


def test_c5_tall_skinny_fp64_esc_bit_exact():
    sr = P.PlusTimesF64
    A = P.fill_values(P.gen_rmat(22, 8, 1), sr, 1)
    B = P.gen_one_per_row(1 << 22, 1 << 10, 2)
    slices = [(0, 1024)]
    got, _ = batched_slices(A, B, sr, slices)
    ha, hb = A.to_host(), B.to_host()
    ao = oracle.Csc(ha.nrows, ha.ncols, ha.colptr, ha.rowids, ha.vals)
    bo = oracle.Csc(hb.nrows, hb.ncols, hb.colptr, hb.rowids, hb.vals)
    want = oracle.ref().local_spgemm(sr.id, ao, bo, threads=16)
    cp, rows, vals, _ = got[(0, 1024)]
    assert np.array_equal(cp, want.colptr) and np.array_equal(rows, want.rowids)
    # the auto policy sends C5 (cf 1.41, heavy columns) to ESC: the reference's fold order
    assert vals.tobytes() == np.asarray(want.vals).tobytes(), "C5 values not bit-identical (ESC path)"
