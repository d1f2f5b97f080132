"""GPU parity of the value form (semirings with values, one product walk).

Items are (column, 2^TL-row tile) with the tile's accumulators in shared
memory; every product is folded there (spgemm.hpp:251-255's upsert, as the
semiring's atomic), the item's values go to a value stash in row order and
emit copies them beside the rows.  These cases force every tile height,
split items (partial accumulators combined in part order), both CTA sizes,
ragged row counts, column windows, rectangular operands with empty columns,
OrAnd operands with stored zeros (structural pattern, values 0/1), MinPlus
products equal to +inf / INT_MAX (the sentinel marks) and the capacity
contract.  Integer / Boolean / MinPlus results are bit-exact; fp within the
north_star tolerance (tests/helpers.py).
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from tests.helpers import assert_parity, to_device, with_values

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402

SEMIRINGS = [P.PlusTimesF64, P.PlusTimesF32, P.PlusTimesI64, P.MinPlusI32, P.MinPlusF64]


def _ctx(tl=-1, split=None, threads=None):
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_ESC, 0)  # the bitmap side is the subject (low cf would pick ESC)
    ctx.set_option(L.OPT_DIRECT_VALUE_FORM, tl)
    if split is not None:
        ctx.set_option(L.OPT_DIRECT_SPLIT_FLOPS, split)
    if threads is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_THREADS, threads)
    return ctx


@pytest.mark.parametrize("threads", [256, 512])
@pytest.mark.parametrize("split", [4096, 1 << 20])
@pytest.mark.parametrize("tl", [-1, 12, 14])
@pytest.mark.parametrize("sr", SEMIRINGS, ids=lambda s: f"{s.name}_{s.dtype}")
def test_value_form_rmat(port, sr, tl, split, threads):
    a = with_values(port, port.gen_rmat(13), sr.id)
    want = port.spgemm(sr.id, a, a)
    got = P.local_spgemm(to_device(a), to_device(a), sr, ctx=_ctx(tl, split, threads), method="direct")
    assert_parity(got, want, sr.id, f"{sr.name} tl={tl} split={split} threads={threads}")


@pytest.mark.parametrize("scale", [8, 11, 15])
@pytest.mark.parametrize("sr", [P.MinPlusI32, P.PlusTimesF64], ids=lambda s: f"{s.name}_{s.dtype}")
def test_value_form_scales(port, sr, scale):
    a = with_values(port, port.gen_rmat(scale), sr.id)
    want = port.spgemm(sr.id, a, a)
    got = P.local_spgemm(to_device(a), to_device(a), sr, ctx=_ctx(), method="direct")
    assert_parity(got, want, sr.id, f"{sr.name} s{scale}")


def _random_csc(rng, nrows, ncols, deg_lo, deg_hi):
    cp = np.zeros(ncols + 1, np.int64)
    rows = []
    for j in range(ncols):
        d = int(rng.integers(deg_lo, deg_hi + 1))
        r = np.sort(rng.choice(nrows, size=min(d, nrows), replace=False)).astype(np.int32)
        rows.append(r)
        cp[j + 1] = cp[j] + len(r)
    return oracle.Csc(nrows, ncols, cp, np.concatenate(rows), None)


@pytest.mark.parametrize("nrows", [5000, 100000, 131073])
@pytest.mark.parametrize("sr", [P.MinPlusI32, P.PlusTimesF64, P.PlusTimesF32], ids=lambda s: f"{s.name}_{s.dtype}")
def test_value_form_ragged_rows(port, nrows, sr):
    rng = np.random.default_rng(nrows + 7)
    kind = {P.MinPlusI32: 3, P.PlusTimesF64: 2, P.PlusTimesF32: 1}[sr]
    a = _random_csc(rng, nrows, 1500, 20, 400)
    a = a.with_vals(port.fill_values(sr.id, kind, a))
    b = _random_csc(rng, 1500, 300, 5, 80)
    b = b.with_vals(port.fill_values(sr.id, kind, b))
    want = port.spgemm(sr.id, a, b)
    for split in (2048, 1 << 20):
        got = P.local_spgemm(to_device(a), to_device(b), sr, ctx=_ctx(split=split), method="direct")
        assert_parity(got, want, sr.id, f"nrows={nrows} split={split}")


def test_value_form_window_and_rectangular(port):
    from paper_2106_14402_b200 import dist as D

    sr = P.MinPlusI32
    a = with_values(port, port.gen_rmat(12), sr.id)
    want = port.spgemm(sr.id, a, a, 700, 3100)
    da = to_device(a)
    ctx = _ctx()
    got = P.local_spgemm(da, D.column_window(da, 700, 3100), sr, ctx=ctx, method="direct")
    assert_parity(got, want, sr.id, "window")
    b = port.gen_rmat(12, 8, 3)
    rows, cols = [], []
    for j in range(0, 1500):
        if j % 4 == 0:
            continue
        s, e = b.colptr[j], b.colptr[j + 1]
        rows += b.rowids[s:e].tolist()
        cols += [j] * int(e - s)
    bb = oracle.from_triples(b.nrows, 1500, rows, cols, np.ones(len(rows)))
    bb = bb.with_vals(port.fill_values(sr.id, 3, bb))
    want = port.spgemm(sr.id, a, bb)
    got = P.local_spgemm(da, to_device(bb), sr, ctx=ctx, method="direct")
    assert_parity(got, want, sr.id, "rect")


def test_value_form_orand_stored_zeros(port):
    """OrAnd operands holding stored zeros: the pattern is structural and the
    values are ORs of ANDs (0 entries stay in C)."""
    z = port.gen_rmat(12)
    z = z.with_vals((np.arange(z.nnz) % 3 != 0).astype(np.uint8))
    want = port.spgemm(oracle.OR_AND_U8, z, z)
    for split in (4096, 1 << 20):
        got = P.local_spgemm(to_device(z), to_device(z), P.OrAnd, ctx=_ctx(split=split), method="direct")
        assert_parity(got, want, oracle.OR_AND_U8, f"zeros split={split}")


def test_value_form_min_plus_infinity(port):
    """MinPlus products equal to the identity (INT_MAX / +inf) are entries
    of C all the same: the value form must mark them although their slot
    stays at the identity."""
    a = port.gen_rmat(11)
    for sr, big in ((P.MinPlusI32, np.int32(2**31 - 1)), (P.MinPlusF64, np.inf)):
        v = port.fill_values(sr.id, 3 if sr is P.MinPlusI32 else 5, a).copy()
        v[::5] = big if sr is P.MinPlusF64 else 0
        if sr is P.MinPlusI32:
            v[1::5] = big  # 0 + INT_MAX = INT_MAX exactly
        aa = a.with_vals(v)
        want = port.spgemm(sr.id, aa, aa)
        got = P.local_spgemm(to_device(aa), to_device(aa), sr, ctx=_ctx(split=4096), method="direct")
        assert_parity(got, want, sr.id, f"{sr.name} identity products")


def test_value_form_capacity_budget_error(port):
    sr = P.MinPlusI32
    a = with_values(port, port.gen_rmat(11), sr.id)
    want = port.spgemm(sr.id, a, a)
    da = to_device(a)
    ctx = _ctx()
    n = want.nnz
    cp = torch.empty(a.ncols + 1, dtype=torch.int64, device="cuda")
    rw = torch.empty(n, dtype=torch.int32, device="cuda")
    v = torch.empty(n, dtype=torch.int32, device="cuda")
    nnz = C.c_int64()
    for cap in (0, n // 3, n - 1):
        st = ctx.lib.slapcu_spgemm_direct(ctx.h, C.byref(da.view()), C.byref(da.view()), sr.id, 2, cap,
                                          cp.data_ptr(), rw.data_ptr(), v.data_ptr(), C.byref(nnz))
        assert st == 5 and nnz.value == n, (cap, st)
    st = ctx.lib.slapcu_spgemm_direct(ctx.h, C.byref(da.view()), C.byref(da.view()), sr.id, 2, n,
                                      cp.data_ptr(), rw.data_ptr(), v.data_ptr(), C.byref(nnz))
    assert st == 0 and nnz.value == n
    assert np.array_equal(cp.cpu().numpy(), want.colptr)
    assert np.array_equal(rw.cpu().numpy(), want.rowids)
    assert np.array_equal(v.cpu().numpy(), want.vals)


def test_value_form_option_range():
    ctx = P.Context()
    for bad in (-2, 1, 11, 16):
        with pytest.raises(P.errors.Error):
            ctx.set_option(L.OPT_DIRECT_VALUE_FORM, bad)
    for ok in (-1, 0, 12, 15):
        ctx.set_option(L.OPT_DIRECT_VALUE_FORM, ok)
