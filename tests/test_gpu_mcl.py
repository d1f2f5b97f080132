"""GPU parity of the Markov-clustering step (algorithms.cpp:267-293 mcl_step,
SURVEY.md 8f rank 3) against the UNMODIFIED reference compiled in place:
expansion through the direct SpGEMM, inflation, pruning and column
renormalisation; pattern exact, values within 1e-12 (fp64; CUDA's pow and a
different summation order), the reference's StochasticityError on
non-stochastic input, ShapeError on non-square input."""
import numpy as np
import pytest

import oracle
from tests.helpers import assert_parity, to_device

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_14402_b200 as P  # noqa: E402


def stochastic_rmat(port, scale, seed=1):
    """R-MAT pattern plus self loops (no empty column), values 1/deg(col)."""
    a = port.gen_rmat(scale, 8, seed)
    n = a.ncols
    rows, cols = [], []
    for j in range(n):
        r = set(a.rowids[a.colptr[j]:a.colptr[j + 1]].tolist())
        r.add(j)
        rows += sorted(r)
        cols += [j] * len(r)
    m = oracle.from_triples(n, n, rows, cols, np.ones(len(rows)))
    deg = np.diff(m.colptr)
    return m.with_vals(np.repeat(1.0 / deg, deg))


@pytest.mark.parametrize("scale", [8, 11])
@pytest.mark.parametrize("inflation,prune", [(2.0, 1e-4), (1.5, 1e-3), (3.0, 0.0), (1.0, 1e-3)])
def test_mcl_step_matches_reference(ref, port, scale, inflation, prune):
    a = stochastic_rmat(port, scale)
    want = ref.mcl_step(a, inflation, prune)
    got = P.mcl_step(to_device(a), inflation, prune)
    assert_parity(got, want, oracle.PLUS_TIMES_F64, f"mcl s{scale} e={inflation} thr={prune}")


def test_mcl_step_f32_columns_stochastic(port):
    """C4's fp32 expansion step: output columns sum to 1 (fp32 rounding)."""
    a = stochastic_rmat(port, 11)
    a32 = a.with_vals(a.vals.astype(np.float32))
    got = P.mcl_step(to_device(a32), 2.0, 1e-4, sr=P.PlusTimesF32).to_host()
    sums = np.add.reduceat(got.vals.astype(np.float64), got.colptr[:-1])
    assert np.allclose(sums, 1.0, atol=1e-5)


def test_mcl_step_errors(port):
    a = stochastic_rmat(port, 8)
    with pytest.raises(P.errors.StochasticityError):
        P.mcl_step(to_device(a.with_vals(a.vals * 1.5)))
    rect = oracle.from_triples(4, 3, [0, 1, 2], [0, 1, 2], np.ones(3))
    with pytest.raises(P.errors.ShapeError):
        P.mcl_step(to_device(rect))
