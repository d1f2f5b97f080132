"""GPU parity of the ESC (expand / stable segmented sort / left fold) path.

With SLAPCU_OPT_DETERMINISTIC the floating-point semirings fold every output
entry in the reference's order (ascending k: spgemm.hpp:156-159 heap ties by
stream, :251-255 hash upserts in B order), so PlusTimes fp64 / fp32 and
MinPlus fp64 are BIT-identical to slap::local_spgemm (the compiled reference
when oracle/_ref is built, else the bit-pinned C restatement) and identical
from run to run.  SLAPCU_OPT_DIRECT_ESC forces the path for every semiring
(exact semirings: same output as every other path).  Edge cases: empty
columns, column windows, capacity overflow (BudgetError with the exact nnz).
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from tests.helpers import assert_parity, to_device, to_oracle, with_values

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402
from paper_2106_14402_b200 import batched as BT  # noqa: E402


def bit_equal(got, want, what):
    g = to_oracle(got)
    assert np.array_equal(g.colptr, want.colptr), f"{what}: colptr"
    assert np.array_equal(g.rowids, want.rowids), f"{what}: rowids"
    gv, wv = np.asarray(g.vals), np.asarray(want.vals)
    assert gv.tobytes() == wv.tobytes(), f"{what}: {int((gv != wv).sum())} values differ bitwise"


def want_of(port, sr_id, a, b, c0=0, c1=0):
    if oracle.ref_available() and not c1:
        return oracle.ref().local_spgemm(sr_id, a, b)
    return port.spgemm(sr_id, a, b, c0, c1)


@pytest.mark.parametrize("scale", [9, 12])
@pytest.mark.parametrize("sr", [P.PlusTimesF64, P.PlusTimesF32, P.MinPlusF64], ids=lambda s: f"{s.name}_{s.dtype}")
def test_deterministic_fp_bit_exact(port, sr, scale):
    a = with_values(port, port.gen_rmat(scale), sr.id, 2 if sr is not P.PlusTimesF32 else 1)
    if sr is P.PlusTimesF64:  # mixed signs: cancellation makes the fold order visible
        v = a.vals.copy()
        v[::3] *= -1.0
        a = a.with_vals(v)
    want = want_of(port, sr.id, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DETERMINISTIC, 1)
    da = to_device(a)
    g1 = P.local_spgemm(da, da, sr, ctx=ctx, method="direct")
    bit_equal(g1, want, f"{sr.name} s{scale}")
    g2 = P.local_spgemm(da, da, sr, ctx=ctx, method="direct")
    assert g1.vals.cpu().numpy().tobytes() == g2.vals.cpu().numpy().tobytes(), "not reproducible run to run"


@pytest.mark.parametrize("sr", [P.PlusTimesF64, P.PlusTimesI64, P.MinPlusI32, P.OrAnd, P.MinPlusF64],
                         ids=lambda s: f"{s.name}_{s.dtype}")
def test_esc_forced_all_semirings(port, sr):
    a = with_values(port, port.gen_rmat(11), sr.id)
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_ESC, 1)
    da = to_device(a)
    got = P.local_spgemm(da, da, sr, ctx=ctx, method="direct")
    bit_equal(got, port.spgemm(sr.id, a, a), sr.name)
    # column window with empty columns inside
    got = P.local_spgemm(da, BT.column_window(da, 300, 1700), sr, ctx=ctx, method="direct")
    bit_equal(got, port.spgemm(sr.id, a, a, 300, 1700), sr.name + " window")


def test_esc_low_compression_shapes(port):
    """C2-like (Erdos-Renyi, cf ~ 1) and C5-like (tall-skinny B, one nonzero
    per row) products, fp64, bit-exact."""
    sr = P.PlusTimesF64
    er = port.gen_er(1 << 12, 8 << 12, 1)
    ctx = P.Context()
    ctx.set_option(L.OPT_DETERMINISTIC, 1)
    bit_equal(P.local_spgemm(to_device(er), to_device(er), sr, ctx=ctx, method="direct"),
              want_of(port, sr.id, er, er), "ER")
    a = with_values(port, port.gen_rmat(12, 8), sr.id, 1)
    rng = np.random.default_rng(2)
    n, m = a.ncols, 64
    cols = rng.integers(0, m, n)
    cp = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=m), out=cp[1:])
    order = np.argsort(cols, kind="stable")
    b = oracle.Csc(n, m, cp, order.astype(np.int32), rng.random(n))
    bit_equal(P.local_spgemm(to_device(a), to_device(b), sr, ctx=ctx, method="direct"), want_of(port, sr.id, a, b),
              "tall-skinny")


def test_esc_capacity_budget_error(port):
    sr = P.PlusTimesF64
    a = with_values(port, port.gen_rmat(10), sr.id)
    want = port.spgemm(sr.id, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DETERMINISTIC, 1)
    da = to_device(a)
    cap = int(want.colptr[-1]) - 1
    cp = torch.empty(a.ncols + 1, dtype=torch.int64, device="cuda")
    rw = torch.empty(cap, dtype=torch.int32, device="cuda")
    vv = torch.empty(cap, dtype=torch.float64, device="cuda")
    nz = C.c_int64()
    st = ctx.lib.slapcu_spgemm_direct(ctx.h, C.byref(da.view()), C.byref(da.view()), sr.id, 2, cap, cp.data_ptr(),
                                      rw.data_ptr(), vv.data_ptr(), C.byref(nz))
    assert st == 5 and nz.value == want.colptr[-1]  # BudgetError with the exact requirement


def test_esc_auto_policy(port):
    """Default (auto): a value semiring whose columns are heavy (> 4096
    multiplies on average) and whose sampled compression is below 2 takes
    ESC -- its values are then bit-identical to the reference even without
    the deterministic option (a C5-like tall-skinny product); light or
    well-compressing products stay on the bitmap / hash paths (within
    tolerance).  Both are correct."""
    sr = P.PlusTimesF64
    a = port.gen_er(1 << 16, 16 << 16, 4)  # values U[0,1)
    rng = np.random.default_rng(5)
    n, m = a.ncols, 16
    cols = rng.integers(0, m, n)
    cp = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=m), out=cp[1:])
    b = oracle.Csc(n, m, cp, np.argsort(cols, kind="stable").astype(np.int32), rng.random(n))
    want = want_of(port, sr.id, a, b)
    assert want.colptr[-1] * 2 > port.estimate_flops(a, b)[0]  # compression < 2
    bit_equal(P.local_spgemm(to_device(a), to_device(b), sr, method="direct"), want, "tall-skinny auto")
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_ESC, 0)
    got = P.local_spgemm(to_device(a), to_device(b), sr, ctx=ctx, method="direct")
    assert_parity(got, want, sr.id, "tall-skinny bitmap path")
