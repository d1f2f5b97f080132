"""GPU parity of the local SpGEMM (spgemm.hpp:275-330) against the CPU oracle.

Every call goes through libslapcu.so's C-ABI.  Cases follow the reference's
own tests: the worked examples (test_localkernels.cpp:66-142), randomized
oracle equivalence across semirings and algorithms (acceptance.cpp:58-97,
test_localkernels.cpp:146-166), symbolic = nnz and flops = multiplies
(test_localkernels.cpp:180-202), plus R-MAT products that exercise every
GPU work class (smem hash bins, dense row-tile path with several tiles,
global-memory value fallback).
"""
import numpy as np
import pytest

import oracle
from tests.helpers import KIND, assert_parity, to_device, with_values

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402

SRS = [P.PlusTimesF64, P.PlusTimesF32, P.PlusTimesI64, P.MinPlusI32, P.MinPlusF64, P.OrAnd]
ALGS = [P.SpGemmAlg.heap, P.SpGemmAlg.hash, P.SpGemmAlg.hybrid]
METHODS = ["fused", "two_pass", "direct"]


def example_a():
    # test_localkernels.cpp:20-29: A = [[1,0],[2,3]]
    return oracle.from_triples(2, 2, [0, 1, 1], [0, 0, 1], np.array([1, 2, 3], np.int64))


def example_b():
    # B = [[0,4],[5,0]]
    return oracle.from_triples(2, 2, [0, 1], [1, 0], np.array([4, 5], np.int64))


@pytest.mark.parametrize("alg", ALGS)
def test_worked_example_plus_times(alg):
    # test_localkernels.cpp:126-131: rows {1,0,1} cols {0,1,1} vals {15,4,8}
    c = P.local_spgemm(to_device(example_a()), to_device(example_b()), P.PlusTimesI64, alg).to_host()
    rows, cols, vals = c.to_triples()
    assert rows.tolist() == [1, 0, 1]
    assert cols.tolist() == [0, 1, 1]
    assert vals.tolist() == [15, 4, 8]


@pytest.mark.parametrize("alg", ALGS)
def test_identity_times_a(alg):
    eye = oracle.from_triples(2, 2, [0, 1], [0, 1], np.array([1, 1], np.int64))
    a = example_a()
    c = P.local_spgemm(to_device(eye), to_device(a), P.PlusTimesI64, alg)
    assert_parity(c, a, oracle.PLUS_TIMES_I64, "I*A")


@pytest.mark.parametrize("alg", ALGS)
def test_min_plus_two_cycle(alg):
    # test_localkernels.cpp:132-142
    m = oracle.from_triples(2, 2, [0, 1], [1, 0], np.array([1.0, 2.0]))
    c = P.local_spgemm(to_device(m), to_device(m), P.MinPlusF64, alg).to_host()
    rows, cols, vals = c.to_triples()
    assert rows.tolist() == [0, 1] and cols.tolist() == [0, 1] and vals.tolist() == [3.0, 3.0]


def test_dim_error():
    a = to_device(oracle.from_triples(3, 2, [0], [0], np.array([1.0])))
    with pytest.raises(P.errors.DimError):
        P.local_spgemm(a, a, P.PlusTimesF64)


def test_empty_operands():
    e = oracle.from_triples(5, 4, [], [], np.zeros(0))
    f = oracle.from_triples(4, 3, [], [], np.zeros(0))
    c = P.local_spgemm(to_device(e), to_device(f), P.PlusTimesF64).to_host()
    assert c.nnz == 0 and c.colptr.tolist() == [0, 0, 0, 0]


def _random_pairs(seed, trials, val_kind, dtype):
    rng = np.random.default_rng(seed)
    for _ in range(trials):
        m, n, k = (int(x) for x in rng.integers(2, 65, 3))
        density = 0.01 + 0.29 * float(rng.random())
        s = int(rng.integers(1, 1 << 30))
        a = oracle.random_triples(s, m, n, density, val_kind, dtype)
        b = oracle.random_triples(s + 7, n, k, density, val_kind, dtype)
        yield a, b


@pytest.mark.parametrize("sr", SRS, ids=lambda s: f"{s.name}_{s.dtype}")
def test_random_vs_oracle(port, sr):
    """acceptance.cpp:58-97 criterion 1 (200 pairs per semiring there; 40 here
    x 3 algorithms)."""
    kind = {"f64": "u10", "f32": "u10", "i64": "small_int", "i32": "small_int", "u8": "one"}[sr.dtype]
    for a, b in _random_pairs(101 + sr.id, 40, kind, sr.np_dtype):
        want = port.spgemm(sr.id, a, b)
        for alg in ALGS:
            for method in METHODS:
                got = P.local_spgemm(to_device(a), to_device(b), sr, alg, method=method)
                assert_parity(got, want, sr.id, f"{sr.name}/{sr.dtype}/{alg.name}/{method}")


def test_symbolic_and_flops(port):
    """test_localkernels.cpp:180-202: symbolic total = nnz(C), flops = multiplies."""
    a = port.gen_rmat(10)
    b = port.gen_rmat(9, 8, 3)
    b = oracle.Csc(a.ncols, b.ncols, b.colptr, b.rowids)  # 1024 x 512
    b.colptr = np.minimum(b.colptr, b.colptr[-1])
    da, db = to_device(a), to_device(b)
    tot, per = P.estimate_flops(da, db)
    wtot, wper = port.estimate_flops(a, b)
    assert tot == wtot and np.array_equal(per.cpu().numpy(), wper)
    counts = P.symbolic_nnz(da, db).cpu().numpy()
    _, wcounts = port.symbolic_nnz(a, b)
    assert np.array_equal(counts, wcounts)


@pytest.mark.parametrize("scale", [10, 12])
@pytest.mark.parametrize("sr", SRS, ids=lambda s: f"{s.name}_{s.dtype}")
def test_rmat_square_vs_oracle(port, sr, scale):
    a = with_values(port, port.gen_rmat(scale), sr.id)
    want = port.spgemm(sr.id, a, a)
    da = to_device(a)
    for alg in ALGS:
        for method in METHODS:
            got = P.local_spgemm(da, da, sr, alg, method=method)
            assert_parity(got, want, sr.id, f"rmat{scale}/{alg.name}/{method}")


@pytest.mark.parametrize("sr", SRS, ids=lambda s: f"{s.name}_{s.dtype}")
def test_multi_tile_paths(port, sr):
    """Small row tiles force several tiles per column on the dense path (tile
    cursors), and a tiny light threshold forces the global-memory value
    fallback and the bitmap symbolic path."""
    a = with_values(port, port.gen_rmat(12), sr.id)
    want = port.spgemm(sr.id, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_TILE_ROWS_LOG2, 10)
    ctx.set_option(L.OPT_SYM_TILE_ROWS_LOG2, 10)
    ctx.set_option(L.OPT_LIGHT_NNZ_MAX, 16)
    ctx.set_option(L.OPT_LIGHT_FLOPS_MAX, 32)
    ctx.set_option(L.OPT_DENSE_TILE_ROWS_LOG2, 10)
    da = to_device(a)
    for alg in ALGS:
        for method in METHODS:
            got = P.local_spgemm(da, da, sr, alg, ctx=ctx, method=method)
            assert_parity(got, want, sr.id, f"tiles/{alg.name}/{method}")


def test_or_and_with_zero_values(port):
    """OrAnd with explicit 0 values must not take the all-ones fast path."""
    a = port.gen_rmat(10)
    v = (np.arange(a.nnz) % 3 != 0).astype(np.uint8)
    a = a.with_vals(v)
    want = port.spgemm(oracle.OR_AND_U8, a, a)
    for alg in ALGS:
        for method in METHODS:
            got = P.local_spgemm(to_device(a), to_device(a), P.OrAnd, alg, method=method)
            assert_parity(got, want, oracle.OR_AND_U8, f"{alg.name}/{method}")


def test_host_call_matches_device(port):
    """slapcu_spgemm_host (host buffers, copies inside the library)."""
    a = with_values(port, port.gen_rmat(11), oracle.MIN_PLUS_I32)
    want = port.spgemm(oracle.MIN_PLUS_I32, a, a)
    host = P.CscMatrix(a.nrows, a.ncols, a.colptr, a.rowids, a.vals)
    got = P.local_spgemm(host, host, P.MinPlusI32)
    assert isinstance(got, P.CscMatrix)
    assert_parity(got, want, oracle.MIN_PLUS_I32, "host")


def test_rectangular_and_empty_columns(port):
    a = with_values(port, port.gen_rmat(11), oracle.PLUS_TIMES_F64)
    # B = columns [100, 900) of A, with every 3rd column emptied
    b = port.gen_rmat(11, 16, 5)
    cp = b.colptr.copy()
    keep = np.ones(b.ncols, bool)
    keep[::3] = False
    rows, cols = [], []
    for j in range(100, 900):
        if keep[j]:
            s, e = cp[j], cp[j + 1]
            rows += b.rowids[s:e].tolist()
            cols += [j - 100] * int(e - s)
    bb = oracle.from_triples(b.nrows, 800, rows, cols, np.ones(len(rows)))
    bb = with_values(port, bb, oracle.PLUS_TIMES_F64)
    want = port.spgemm(oracle.PLUS_TIMES_F64, a, bb)
    for alg in ALGS:
        for method in METHODS:
            got = P.local_spgemm(to_device(a), to_device(bb), P.PlusTimesF64, alg, method=method)
            assert_parity(got, want, oracle.PLUS_TIMES_F64, f"{alg.name}/{method}")


def test_thread_count_invariance(port):
    """test_localkernels.cpp:168-178: the result does not depend on `threads`
    (here: repeated runs are identical for an exact semiring)."""
    a = with_values(port, port.gen_rmat(11), oracle.PLUS_TIMES_I64)
    da = to_device(a)
    base = P.local_spgemm(da, da, P.PlusTimesI64, threads=1).to_host()
    for t in (2, 4, 8):
        c = P.local_spgemm(da, da, P.PlusTimesI64, threads=t).to_host()
        assert np.array_equal(c.rowids, base.rowids) and np.array_equal(c.vals, base.vals)


@pytest.mark.parametrize("dense_min", [0, 1, -1])
def test_fused_pattern_paths(port, dense_min):
    """Fused pattern pass: bitmap-atomic path only (0), byte-flag path for
    every heavy column (1), automatic split (-1)."""
    a = with_values(port, port.gen_rmat(12), oracle.MIN_PLUS_I32)
    want = port.spgemm(oracle.MIN_PLUS_I32, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DENSE_FLOPS_MIN, dense_min)
    ctx.set_option(L.OPT_DENSE_TILE_ROWS_LOG2, 11)
    da = to_device(a)
    for sr, w in ((P.MinPlusI32, want),):
        got = P.local_spgemm(da, da, sr, ctx=ctx)
        assert_parity(got, w, sr.id, f"dense_min={dense_min}")
    ab = a.with_vals(np.ones(a.nnz, np.uint8))
    wb = port.spgemm(oracle.OR_AND_U8, ab, ab)
    got = P.local_spgemm(to_device(ab), to_device(ab), P.OrAnd, ctx=ctx)
    assert_parity(got, wb, oracle.OR_AND_U8, f"bool dense_min={dense_min}")


def test_column_window_operand(port):
    """B given as a column window (colptr not starting at 0) -- the batched
    driver's slices (batched.hpp:43-66) -- gives exactly those columns."""
    from paper_2106_14402_b200 import dist as D

    a = with_values(port, port.gen_rmat(11), oracle.MIN_PLUS_I32)
    want = port.spgemm(oracle.MIN_PLUS_I32, a, a, 300, 1500)
    da = to_device(a)
    for method in METHODS:
        got = P.local_spgemm(da, D.column_window(da, 300, 1500), P.MinPlusI32, method=method)
        assert_parity(got, want, oracle.MIN_PLUS_I32, method)


def test_staging_budget_error():
    """begin() refuses a staging area above the budget (BudgetError)."""
    import ctypes as C

    a = P.gen_rmat(10)
    a = P.fill_values(a, P.OrAnd, 0)
    ctx = P.default_context()
    cp = torch.empty(a.ncols + 1, dtype=torch.int64, device=a.colptr.device)
    nnz = C.c_int64()
    st = ctx.lib.slapcu_spgemm_begin(ctx.h, C.byref(a.view()), C.byref(a.view()), P.OrAnd.id, 2, 1024,
                                     cp.data_ptr(), C.byref(nnz))
    assert st == 5  # SLAPCU_ERR_BUDGET


def test_dcsc_upload(port):
    """local_matrix.hpp:88-150 DCSC (jc / cp over nonempty columns, int32)
    to the device: the dense colptr is built on the GPU; the uploaded block
    multiplies like its CSC twin and downloads back to the same CSC."""
    import ctypes as C

    from paper_2106_14402_b200 import _lib as L

    a = port.gen_rmat(10)
    a = a.with_vals(port.fill_values(oracle.PLUS_TIMES_F64, 2, a))
    cnt = np.diff(a.colptr)
    # drop every third column to get hypersparse blocks with empty columns
    keep = np.ones(a.ncols, bool)
    keep[::3] = False
    rows, vals, cp, jc = [], [], [0], []
    for j in range(a.ncols):
        if keep[j] and cnt[j]:
            s, e = a.colptr[j], a.colptr[j + 1]
            rows.append(a.rowids[s:e])
            vals.append(a.vals[s:e])
            jc.append(j)
            cp.append(cp[-1] + int(e - s))
    rows = np.concatenate(rows).astype(np.int32)
    vals = np.concatenate(vals)
    jc = np.asarray(jc, np.int32)
    cp = np.asarray(cp, np.int32)
    ctx = P.Context()
    out = L.CscOut()
    ctx.check(ctx.lib.slapcu_dcsc_upload(ctx.h, a.nrows, a.ncols, len(jc), jc.ctypes.data, cp.ctypes.data,
                                         rows.ctypes.data, vals.ctypes.data, oracle.PLUS_TIMES_F64, C.byref(out)),
              "dcsc_upload")
    view = L.CscView(out.nrows, out.ncols, out.nnz, out.colptr, out.rowids, out.vals)
    host = L.CscOut()
    ctx.check(ctx.lib.slapcu_csc_download(ctx.h, C.byref(view), oracle.PLUS_TIMES_F64, C.byref(host)), "download")
    colptr = np.ctypeslib.as_array(C.cast(host.colptr, C.POINTER(C.c_int64)), shape=(a.ncols + 1,)).copy()
    want_cp = np.zeros(a.ncols + 1, np.int64)
    for x, j in enumerate(jc):
        want_cp[j + 1] = cp[x + 1] - cp[x]
    want_cp = np.cumsum(want_cp)
    assert np.array_equal(colptr, want_cp)
    got_rows = np.ctypeslib.as_array(C.cast(host.rowids, C.POINTER(C.c_int32)), shape=(int(host.nnz),)).copy()
    assert np.array_equal(got_rows, rows)
    ctx.lib.slapcu_host_free(C.byref(host))
    ctx.check(ctx.lib.slapcu_csc_free(ctx.h, C.byref(out)), "free")
