"""Column batching (batched.hpp:14-170) on the GPU: concatenated batch outputs
equal the unbatched product for b in {1, 2, 4, 8} (test_distkernels.cpp:222-250),
budget plans match the compiled reference's plan_batches_by_budget exactly,
and the reference's error contract (BudgetError, ShapeError) holds."""
import numpy as np
import pytest

import oracle
from tests.helpers import assert_parity, to_device, with_values

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import batched as BT  # noqa: E402


@pytest.mark.parametrize("nb", [1, 2, 4, 8])
def test_batches_concatenate_to_product(port, nb):
    a = with_values(port, port.gen_rmat(11), oracle.MIN_PLUS_I32)
    want = port.spgemm(oracle.MIN_PLUS_I32, a, a)
    da = to_device(a)
    parts = BT.batched_spgemm(da, da, BT.plan_batches_by_count(da.ncols, nb), P.MinPlusI32)
    rows = np.concatenate([p.rowids.cpu().numpy() for p in parts])
    vals = np.concatenate([p.vals.cpu().numpy() for p in parts])
    counts = np.concatenate([np.diff(p.colptr.cpu().numpy()) for p in parts])
    assert np.array_equal(rows, want.rowids) and np.array_equal(vals, want.vals)
    assert np.array_equal(counts, np.diff(want.colptr))


def test_consumer_called_in_order(port):
    a = with_values(port, port.gen_rmat(10), oracle.OR_AND_U8)
    da = to_device(a)
    seen = []
    BT.batched_spgemm(da, da, BT.plan_batches_by_count(da.ncols, 3), P.OrAnd,
                      consumer=lambda r, s, e, c: seen.append((r, s, e, c.ncols)))
    assert [x[0] for x in seen] == [0, 1, 2] and seen[-1][2] == da.ncols
    assert all(x[3] == x[2] - x[1] for x in seen)


@pytest.mark.parametrize("budget", [4096, 65536, 1 << 20])
def test_budget_plan_matches_reference(port, ref, budget):
    a = port.gen_rmat(10)
    a = a.with_vals(np.ones(a.nnz))
    da = to_device(a.with_vals(np.ones(a.nnz, np.uint8)))
    try:
        want_ranges, want_est = ref.plan_batches(a, a, budget, p=1)
    except RuntimeError as e:  # -7: the reference raised BudgetError
        assert "-7" in str(e)
        with pytest.raises(P.errors.BudgetError):
            BT.plan_batches_by_budget(da, da, budget)
        return
    plan = BT.plan_batches_by_budget(da, da, budget)
    assert plan.col_ranges == want_ranges
    assert plan.est_entries == list(want_est)


def test_budget_errors(port):
    a = to_device(port.gen_rmat(9).with_vals(None))
    with pytest.raises(P.errors.BudgetError):
        BT.plan_batches_by_budget(a, a, 0)
    with pytest.raises(P.errors.BudgetError):
        BT.plan_batches_by_budget(a, a, 16)  # a single column needs more
    plan = BT.BatchPlan([(0, 10), (12, a.ncols)], [0, 0])
    av = P.fill_values(a, P.OrAnd, 0)
    with pytest.raises(P.errors.ShapeError):
        BT.batched_spgemm(av, av, plan, P.OrAnd)
    with pytest.raises(P.errors.ShapeError):
        BT.batched_spgemm(av, av, BT.BatchPlan(), P.OrAnd)
