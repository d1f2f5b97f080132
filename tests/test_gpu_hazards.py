"""GPU regression tests for round-1 review findings.

* Value pass on row counts that are not a multiple of the item tile: the
  last rank chunk of an item ends at the item's last 4096-row block, which
  lies past the matrix's last block (direct.cu k_item_values_rank);
  MinPlus int32 and PlusTimes fp64/fp32 with nrows 5000 / 100000 / 131073.
* The per-A caches of the direct path (tile pointers, dense-run bitmaps) are
  keyed on A's pattern content: rewriting A in place with the same nnz, or a
  different A at a reused address, must not reuse stale tile pointers.
"""
import numpy as np
import pytest

import oracle
from tests.helpers import assert_parity, to_device

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402


def random_csc(rng, nrows, ncols, deg_lo, deg_hi):
    cp = np.zeros(ncols + 1, np.int64)
    rows = []
    for j in range(ncols):
        d = int(rng.integers(deg_lo, deg_hi + 1))
        r = np.sort(rng.choice(nrows, size=min(d, nrows), replace=False)).astype(np.int32)
        rows.append(r)
        cp[j + 1] = cp[j] + len(r)
    return oracle.Csc(nrows, ncols, cp, np.concatenate(rows) if rows else np.zeros(0, np.int32), None)


@pytest.mark.parametrize("nrows", [5000, 100000, 131073])
@pytest.mark.parametrize("sr", [P.MinPlusI32, P.PlusTimesF64, P.PlusTimesF32], ids=lambda s: f"{s.name}_{s.dtype}")
def test_value_pass_ragged_row_count(port, nrows, sr):
    rng = np.random.default_rng(nrows)
    kind = {P.MinPlusI32: 3, P.PlusTimesF64: 2, P.PlusTimesF32: 1}[sr]
    a = random_csc(rng, nrows, 1500, 20, 400)
    a = a.with_vals(port.fill_values(sr.id, kind, a))
    b = random_csc(rng, 1500, 300, 5, 80)
    b = b.with_vals(port.fill_values(sr.id, kind, b))
    want = port.spgemm(sr.id, a, b)
    for rank, tmajor in ((-1, 0), (4096, 0), (-1, 1)):  # default chunk (8192 / 4096 by width), 4096; tile-major
        ctx = P.Context()
        ctx.set_option(L.OPT_DIRECT_ESC, 0)  # the bitmap value pass is the subject (low cf would pick ESC)
        ctx.set_option(L.OPT_DIRECT_VALUE_FORM, 0)
        if rank > 0:
            ctx.set_option(L.OPT_DIRECT_VALUE_RANK, rank)
        ctx.set_option(L.OPT_DIRECT_VALUE_TMAJOR, tmajor)
        got = P.local_spgemm(to_device(a), to_device(b), sr, ctx=ctx, method="direct")
        assert_parity(got, want, sr.id, f"nrows={nrows} rank={rank}")


@pytest.mark.parametrize("sr", [P.OrAnd, P.MinPlusI32], ids=lambda s: f"{s.name}_{s.dtype}")
def test_direct_cache_inplace_rewrite(port, sr):
    """Same device buffers, same nnz, different row pattern: the second call
    must see the new pattern (cache keyed on pointer + nnz)."""
    kind = 0 if sr is P.OrAnd else 3
    a1 = port.gen_rmat(13, 16, 1)
    a1 = a1.with_vals(port.fill_values(sr.id, kind, a1))
    # a second matrix with the same colptr (so the same nnz per column) but
    # different rows: a row relabelling r -> (r * 7919 + 13) % n, re-sorted
    n = a1.nrows
    rows2 = ((a1.rowids.astype(np.int64) * 7919 + 13) % n).astype(np.int32)
    for j in range(a1.ncols):
        s, e = a1.colptr[j], a1.colptr[j + 1]
        rows2[s:e] = np.sort(rows2[s:e])
    a2 = oracle.Csc(n, a1.ncols, a1.colptr.copy(), rows2, a1.vals.copy())
    ctx = P.Context()
    ctx.set_option(L.OPT_DIRECT_DENSE_RUN_MIN, 64)  # exercise the cached dense-run bitmaps too
    da = to_device(a1)
    want1 = port.spgemm(sr.id, a1, a1)
    assert_parity(P.local_spgemm(da, da, sr, ctx=ctx, method="direct"), want1, sr.id, "first")
    da.rowids.copy_(torch.from_numpy(rows2).to(da.rowids.device))  # in place, same pointer, same nnz
    want2 = port.spgemm(sr.id, a2, a2)
    assert_parity(P.local_spgemm(da, da, sr, ctx=ctx, method="direct"), want2, sr.id, "after in-place rewrite")
    ctx.invalidate()
    assert_parity(P.local_spgemm(da, da, sr, ctx=ctx, method="direct"), want2, sr.id, "after invalidate")
