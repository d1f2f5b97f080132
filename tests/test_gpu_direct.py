"""GPU parity of the in-place single-pass path (slapcu_spgemm_direct).

The Boolean product is formed as (column, row tile) items, stashed as a
bitmap or a word list, placed by a scan and expanded into C; these cases
force every item class -- short runs, warp units, items split over several
CTAs, both stash forms, many tiles per column, column windows, empty
columns -- and check C bit-exactly against the CPU
oracle (acceptance.cpp:58-97 style equivalence; spgemm.hpp:259-260 sorted
rows).  Capacity overflow must raise BudgetError with the exact nnz.
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


def _ones(m):
    return m.with_vals(np.ones(m.nnz, np.uint8))


@pytest.mark.parametrize("tile_log2", [10, 12, 17])
@pytest.mark.parametrize("split", [1024, 5000, 262144])
@pytest.mark.parametrize("dense_run", [0, 16, 2048])
def test_direct_bool_tiles_and_splits(port, tile_log2, split, dense_run):
    a = _ones(port.gen_rmat(12))
    want = port.spgemm(oracle.OR_AND_U8, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, tile_log2)
    ctx.set_option(L.OPT_DIRECT_SPLIT_FLOPS, split)
    ctx.set_option(L.OPT_DIRECT_DENSE_RUN_MIN, dense_run)
    da = to_device(a)
    for alg in (P.SpGemmAlg.heap, P.SpGemmAlg.hybrid):
        got = P.local_spgemm(da, da, P.OrAnd, alg, ctx=ctx, method="direct")
        assert_parity(got, want, oracle.OR_AND_U8, f"TL={tile_log2} split={split} {alg.name}")


@pytest.mark.parametrize("form_threads", [128, 256, 512])
@pytest.mark.parametrize("words", [0, 1])
@pytest.mark.parametrize("scale", [8, 11, 14])
def test_direct_bool_rmat(port, scale, words, form_threads):
    a = _ones(port.gen_rmat(scale))
    want = port.spgemm(oracle.OR_AND_U8, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_WORDS, words)
    ctx.set_option(L.OPT_DIRECT_FORM_THREADS, form_threads)
    got = P.local_spgemm(to_device(a), to_device(a), P.OrAnd, ctx=ctx, method="direct")
    assert_parity(got, want, oracle.OR_AND_U8, f"s{scale} words {words} threads {form_threads}")


def test_retired_options_rejected():
    """Experiments measured slower and removed: only their defaults remain."""
    ctx = P.Context()
    for opt, bad in ((L.OPT_DIRECT_MARK_MODE, 2), (L.OPT_DIRECT_QUADS, 1), (L.OPT_DIRECT_FORM_WALK, 1),
                     (L.OPT_DIRECT_EMIT_THREADS, 32), (L.OPT_DIRECT_VALUE_L2, 1), (L.OPT_DIRECT_VALUE_DENSE_ONLY, 1)):
        with pytest.raises(P.errors.Error):
            ctx.set_option(opt, bad)


@pytest.mark.parametrize("words", [0, 1])
@pytest.mark.parametrize("tile_major", [0, 1])
@pytest.mark.parametrize("dense_run", [0, 64])
@pytest.mark.parametrize("scale", [11, 14])
def test_direct_form_variants(port, scale, tile_major, dense_run, words):
    """Form kernel variants: tile-major unit order, the row / word form of A,
    dense runs (with split items: split threshold 4096), Boolean and
    MinPlus."""
    for sr, kind in ((P.OrAnd, 0), (P.MinPlusI32, 3)):
        a = port.gen_rmat(scale)
        a = a.with_vals(port.fill_values(sr.id, kind, a))
        want = port.spgemm(sr.id, a, a)
        ctx = P.Context()
        ctx.set_option(L.OPT_DIRECT_WORDS, words)
        ctx.set_option(L.OPT_DIRECT_TILE_MAJOR, tile_major)
        ctx.set_option(L.OPT_DIRECT_DENSE_RUN_MIN, dense_run)
        ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, 11)
        ctx.set_option(L.OPT_DIRECT_SPLIT_FLOPS, 4096)
        got = P.local_spgemm(to_device(a), to_device(a), sr, ctx=ctx, method="direct")
        assert_parity(got, want, sr.id, f"s{scale} words {words} tile_major {tile_major} {sr.name}")


def test_direct_window_and_rectangular(port):
    from paper_2106_14402_b200 import dist as D

    a = _ones(port.gen_rmat(12))
    want = port.spgemm(oracle.OR_AND_U8, a, a, 700, 3100)
    da = to_device(a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, 11)
    got = P.local_spgemm(da, D.column_window(da, 700, 3100), P.OrAnd, ctx=ctx, method="direct")
    assert_parity(got, want, oracle.OR_AND_U8, "window")
    # B with empty columns and a different row count than A's columns
    b = port.gen_rmat(12, 8, 3)
    rows, cols = [], []
    for j in range(0, 1500):
        if j % 4 == 0:
            continue
        s, e = b.colptr[j], b.colptr[j + 1]
        rows += b.rowids[s:e].tolist()
        cols += [j] * int(e - s)
    bb = _ones(oracle.from_triples(b.nrows, 1500, rows, cols, np.ones(len(rows))))
    want = port.spgemm(oracle.OR_AND_U8, a, bb)
    got = P.local_spgemm(da, to_device(bb), P.OrAnd, ctx=ctx, method="direct")
    assert_parity(got, want, oracle.OR_AND_U8, "rect")


@pytest.mark.parametrize("vtl", [10, 12, 14])
@pytest.mark.parametrize("rank", [0, 4096, 8192])
@pytest.mark.parametrize("hash_", [0, 1])
@pytest.mark.parametrize("sr", [P.PlusTimesF64, P.PlusTimesF32, P.PlusTimesI64, P.MinPlusI32, P.MinPlusF64],
                         ids=lambda s: f"{s.name}_{s.dtype}")
def test_direct_value_pass(port, sr, vtl, hash_, rank):
    """Semirings with values: pattern walk + emit, then the value pass --
    small items through the hash kernel, large ones over sub-tiles of 2^vtl
    rows (several per item when vtl < the item tile)."""
    a = with_values(port, port.gen_rmat(14 if hash_ else 12), sr.id)
    want = port.spgemm(sr.id, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_ESC, 0)  # the bitmap value pass is the subject
    ctx.set_option(L.OPT_DIRECT_VALUE_FORM, 0)  # (not the one-walk value form)
    ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, 14 if hash_ else 12)
    ctx.set_option(L.OPT_DIRECT_VALUE_TILE_ROWS_LOG2, vtl)
    ctx.set_option(L.OPT_DIRECT_VALUE_HASH, hash_)
    ctx.set_option(L.OPT_DIRECT_VALUE_RANK, rank)
    ctx.set_option(L.OPT_DIRECT_SPLIT_FLOPS, 4096)
    got = P.local_spgemm(to_device(a), to_device(a), sr, ctx=ctx, method="direct")
    assert_parity(got, want, sr.id, f"{sr.name} vtl={vtl}")


@pytest.mark.parametrize("dense_rows", [0, 16384, 32768])
@pytest.mark.parametrize("tmajor", [0, 1])
@pytest.mark.parametrize("sr", [P.PlusTimesF64, P.PlusTimesF32, P.MinPlusI32, P.PlusTimesI64],
                         ids=lambda s: f"{s.name}_{s.dtype}")
def test_direct_value_tmajor(port, sr, tmajor, dense_rows):
    """Value pass with the tile-major 4096-row pointer table and rank chunks
    in row-block order (and without): same output."""
    a = with_values(port, port.gen_rmat(14), sr.id)
    want = port.spgemm(sr.id, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_ESC, 0)  # the bitmap value pass is the subject
    ctx.set_option(L.OPT_DIRECT_VALUE_FORM, 0)  # (not the one-walk value form)
    ctx.set_option(L.OPT_DIRECT_VALUE_TMAJOR, tmajor)
    ctx.set_option(L.OPT_DIRECT_VALUE_DENSE_ROWS, dense_rows)
    ctx.set_option(L.OPT_DIRECT_VALUE_HASH, 0)
    ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, 16)
    got = P.local_spgemm(to_device(a), to_device(a), sr, ctx=ctx, method="direct")
    assert_parity(got, want, sr.id, f"{sr.name} tmajor={tmajor}")


@pytest.mark.parametrize("interleave", [0, 1, 2])
@pytest.mark.parametrize("sr", [P.PlusTimesF32, P.MinPlusI32, P.PlusTimesF64, P.PlusTimesI64, P.MinPlusF64],
                         ids=lambda s: f"{s.name}_{s.dtype}")
def test_direct_value_interleave(port, sr, interleave):
    """The value pass gathers A's (row, value) pairs from an interleaved copy
    (1, the default: 4-byte values; 2: also 8-byte values as 16-byte pairs) or
    from the two arrays -- same output."""
    a = with_values(port, port.gen_rmat(13), sr.id)
    want = port.spgemm(sr.id, a, a)
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_ESC, 0)  # the bitmap value pass is the subject
    ctx.set_option(L.OPT_DIRECT_VALUE_FORM, 0)  # (not the one-walk value form)
    ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, 12)
    ctx.set_option(L.OPT_DIRECT_VALUE_INTERLEAVE, interleave)
    got = P.local_spgemm(to_device(a), to_device(a), sr, ctx=ctx, method="direct")
    assert_parity(got, want, sr.id, f"{sr.name} interleave={interleave}")


def test_direct_fallback_semirings(port):
    """Value semirings and OrAnd with stored zeros (structural pattern,
    values from the value pass): same contract, same output."""
    a = with_values(port, port.gen_rmat(11), oracle.MIN_PLUS_I32)
    want = port.spgemm(oracle.MIN_PLUS_I32, a, a)
    assert_parity(P.local_spgemm(to_device(a), to_device(a), P.MinPlusI32, method="direct"), want,
                  oracle.MIN_PLUS_I32, "min_plus")
    z = port.gen_rmat(10)
    z = z.with_vals((np.arange(z.nnz) % 3 != 0).astype(np.uint8))
    want = port.spgemm(oracle.OR_AND_U8, z, z)
    assert_parity(P.local_spgemm(to_device(z), to_device(z), P.OrAnd, method="direct"), want, oracle.OR_AND_U8,
                  "zeros")


def test_direct_capacity_budget_error(port):
    a = _ones(port.gen_rmat(11))
    want = port.spgemm(oracle.OR_AND_U8, a, a)
    da = to_device(a)
    ctx = P.Context()
    n = want.nnz
    cp = torch.empty(a.ncols + 1, dtype=torch.int64, device="cuda")
    rw = torch.empty(n, dtype=torch.int32, device="cuda")
    v = torch.empty(n, dtype=torch.uint8, device="cuda")
    nnz = C.c_int64()
    st = ctx.lib.slapcu_spgemm_direct(ctx.h, C.byref(da.view()), C.byref(da.view()), P.OrAnd.id, 2, n - 1,
                                      cp.data_ptr(), rw.data_ptr(), v.data_ptr(), C.byref(nnz))
    assert st == 5 and nnz.value == n
    # exact capacity succeeds
    st = ctx.lib.slapcu_spgemm_direct(ctx.h, C.byref(da.view()), C.byref(da.view()), P.OrAnd.id, 2, n,
                                      cp.data_ptr(), rw.data_ptr(), v.data_ptr(), C.byref(nnz))
    assert st == 0 and nnz.value == n
    assert np.array_equal(rw.cpu().numpy(), want.rowids)
    assert np.array_equal(cp.cpu().numpy(), want.colptr)


def test_direct_empty(port):
    e = oracle.from_triples(50, 40, [], [], np.zeros(0, np.uint8))
    a = _ones(port.gen_rmat(6))
    for x, y in ((e, _ones(oracle.from_triples(40, 30, [], [], np.zeros(0)))),
                 (_ones(oracle.from_triples(64, 64, [], [], np.zeros(0))), a)):
        want = port.spgemm(oracle.OR_AND_U8, x, y)
        got = P.local_spgemm(to_device(x), to_device(y), P.OrAnd, method="direct")
        assert_parity(got, want, oracle.OR_AND_U8, "empty")


@pytest.mark.parametrize("rows", [0, 1])
@pytest.mark.parametrize("sr", [P.MinPlusI32, P.PlusTimesF32], ids=lambda s: f"{s.name}_{s.dtype}")
def test_direct_value_rows(port, sr, rows):
    """4-byte values, every item in rank chunks: the value pass writes C's
    rows from the form pass's stash and the emit pass is skipped (1, the
    default), or emit writes them (0) -- same C, with the default tiles and
    with 4096-row tiles and split items."""
    a = with_values(port, port.gen_rmat(13), sr.id)
    want = port.spgemm(sr.id, a, a)
    for tl, split in ((0, 1 << 20), (12, 4096)):
        ctx = P.Context()
        ctx.set_option(L.OPT_DIRECT_ESC, 0)
        ctx.set_option(L.OPT_DIRECT_VALUE_ROWS, rows)
        ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, tl)
        ctx.set_option(L.OPT_DIRECT_SPLIT_FLOPS, split)
        got = P.local_spgemm(to_device(a), to_device(a), sr, ctx=ctx, method="direct")
        assert_parity(got, want, sr.id, f"{sr.name} rows={rows} tl={tl}")
