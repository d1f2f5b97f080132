"""CPU tests of the benchmark's host-side planning: column batches under a
byte budget (batched.hpp:122-148 semantics) and the flops-balanced column
blocks of the multi-GPU 1D split."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def test_plan_batches_respects_budget():
    rng = np.random.default_rng(3)
    counts = rng.integers(0, 100, size=1000)
    batches = bench.plan_batches(counts, 4, 4000)
    assert batches[0][0] == 0 and batches[-1][1] == 1000
    for (s, e), (s2, _e2) in zip(batches, batches[1:]):
        assert e == s2
    for s, e in batches:
        assert counts[s:e].sum() * 4 <= 4000


def test_plan_batches_rejects_oversized_column():
    with pytest.raises(RuntimeError):
        bench.plan_batches(np.array([1, 2000, 3]), 4, 4000)


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_flops_balanced_blocks(parts):
    rng = np.random.default_rng(parts)
    fl = rng.integers(0, 1000, size=5000) ** 2
    b = bench.flops_balanced_blocks(fl, parts)
    assert b[0] == 0 and b[-1] == len(fl) and len(b) == parts + 1
    assert all(x <= y for x, y in zip(b, b[1:]))
    share = [fl[s:e].sum() for s, e in zip(b, b[1:])]
    assert max(share) <= fl.sum() / parts + fl.max()
