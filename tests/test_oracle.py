"""CPU tests of the oracle (no GPU): the C restatement (oracle/oracle.c) is
pinned against (1) the reference's own golden vectors and (2) the unmodified
reference compiled in place (oracle/_ref/libslapref.so) plus the committed
fixtures in tests/golden/ that were generated from it
(tests/golden/make_golden.py)."""
import hashlib
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
ALL_SR = [oracle.PLUS_TIMES_F64, oracle.PLUS_TIMES_F32, oracle.PLUS_TIMES_I64, oracle.MIN_PLUS_I32,
          oracle.MIN_PLUS_F64, oracle.OR_AND_U8]
KIND = {0: 2, 1: 1, 2: 5, 3: 3, 4: 5, 5: 0}


def same(a, b):
    return (np.array_equal(a.colptr, b.colptr) and np.array_equal(a.rowids, b.rowids)
            and (a.vals is None or a.vals.tobytes() == b.vals.tobytes()))


# ------------------------------------------------- reference golden vectors


def test_worked_example(port):
    # test_localkernels.cpp:126-131
    a = oracle.from_triples(2, 2, [0, 1, 1], [0, 0, 1], np.array([1, 2, 3], np.int64))
    b = oracle.from_triples(2, 2, [0, 1], [1, 0], np.array([4, 5], np.int64))
    c = port.spgemm(oracle.PLUS_TIMES_I64, a, b)
    cols = np.repeat(np.arange(2), np.diff(c.colptr))
    assert c.rowids.tolist() == [1, 0, 1] and cols.tolist() == [0, 1, 1] and c.vals.tolist() == [15, 4, 8]
    # test_localkernels.cpp:69-73 estimate_flops [1,2] / 3 and :102 symbolic [1,2]
    tot, per = port.estimate_flops(a, b)
    assert tot == 3 and per.tolist() == [1, 2]
    assert port.symbolic_nnz(a, b)[1].tolist() == [1, 2]


def test_min_plus_two_cycle(port):
    m = oracle.from_triples(2, 2, [0, 1], [1, 0], np.array([1.0, 2.0]))
    c = port.spgemm(oracle.MIN_PLUS_F64, m, m)
    assert c.rowids.tolist() == [0, 1] and c.vals.tolist() == [3.0, 3.0] and c.colptr.tolist() == [0, 1, 2]


def test_disjoint_patterns_give_zero(port):
    # test_localkernels.cpp:104-114
    a = oracle.from_triples(3, 3, [0], [0], np.array([1], np.int64))
    b = oracle.from_triples(3, 3, [1], [1], np.array([1], np.int64))
    assert port.symbolic_nnz(a, b)[1].tolist() == [0, 0, 0]


def test_rng_matches_reference_constants(port):
    # rng.hpp:34-41 splitmix64 finalizer known answers
    assert port.mix(0) == 0
    z = 0x9E3779B97F4A7C15
    assert port.mix(z) == 0xE220A8397B1DCDAF


# --------------------------------------------- against the compiled reference


@pytest.mark.parametrize("scale,ef", [(6, 4), (8, 16), (10, 16), (12, 8)])
def test_gen_rmat_matches_reference(port, ref, scale, ef):
    assert same(port.gen_rmat(scale, ef, 1), ref.gen_rmat(scale, ef, 1))


@pytest.mark.parametrize("sr", ALL_SR)
def test_spgemm_matches_reference_bitwise(port, ref, sr):
    """The restated fold (ascending k) is bit-identical to every reference
    algorithm, fp64 included (SURVEY.md finding 0.4)."""
    a = port.gen_rmat(9)
    a = a.with_vals(port.fill_values(sr, KIND[sr], a))
    want = port.spgemm(sr, a, a)
    for alg in (oracle.HEAP, oracle.HASH, oracle.HYBRID):
        for dcsc in (False, True):
            got = ref.local_spgemm(sr, a, a, alg=alg, threads=2, b_dcsc=dcsc)
            assert same(got, want), (alg, dcsc)


@pytest.mark.parametrize("sr", ALL_SR)
def test_random_small_matches_reference(port, ref, sr):
    """acceptance.cpp:58-97 style random pairs (dims 2..64, density 1-30%)."""
    rng = np.random.default_rng(1000 + sr)
    kind = {0: "u10", 1: "u10", 2: "small_int", 3: "small_int", 4: "small_int", 5: "one"}[sr]
    for _ in range(10):
        m, n, k = (int(x) for x in rng.integers(2, 65, 3))
        d = 0.01 + 0.29 * float(rng.random())
        s = int(rng.integers(1, 1 << 30))
        a = oracle.random_triples(s, m, n, d, kind, oracle.DTYPES[sr])
        b = oracle.random_triples(s + 1, n, k, d, kind, oracle.DTYPES[sr])
        want = ref.local_spgemm(sr, a, b, alg=oracle.HYBRID, threads=1)
        assert same(port.spgemm(sr, a, b), want)
        dense = port.spgemm(sr, a, b)
        assert dense.nnz == port.symbolic_nnz(a, b)[0]


def test_flops_and_symbolic_match_reference(port, ref):
    a = port.gen_rmat(11)
    tot, per = port.estimate_flops(a, a)
    rtot, rper = ref.estimate_flops(a, a)
    assert tot == rtot and np.array_equal(per, rper)
    assert np.array_equal(port.symbolic_nnz(a, a)[1], ref.symbolic_nnz(a, a, threads=2)[1])


@pytest.mark.parametrize("sr", ALL_SR)
def test_merge_matches_reference(port, ref, sr):
    parts = []
    for s in range(3):
        m = port.gen_rmat(8, 4, 20 + s)
        parts.append(m.with_vals(port.fill_values(sr, 2 if sr in (0, 1) else KIND[sr], m)))
    assert same(port.merge(sr, parts), ref.merge(sr, parts))


def test_column_slices_preserve_columns(port):
    """Column j of C depends only on B(:,j): slicing is exact."""
    a = port.gen_rmat(10)
    a = a.with_vals(port.fill_values(oracle.PLUS_TIMES_F64, 2, a))
    full = port.spgemm(oracle.PLUS_TIMES_F64, a, a)
    part = port.spgemm(oracle.PLUS_TIMES_F64, a, a, 100, 300)
    lo, hi = full.colptr[100], full.colptr[300]
    assert np.array_equal(part.rowids, full.rowids[lo:hi])
    assert part.vals.tobytes() == full.vals[lo:hi].tobytes()


def test_reference_timed_call(ref, port):
    a = port.gen_rmat(10)
    a = a.with_vals(port.fill_values(oracle.MIN_PLUS_I32, 3, a))
    secs, nnz, fl = ref.time_local_spgemm(oracle.MIN_PLUS_I32, a, a, 0, 64, 2)
    want = port.spgemm(oracle.MIN_PLUS_I32, a, a, 0, 64)
    assert secs > 0 and nnz == want.nnz and fl == port.estimate_flops(a, a)[1][:64].sum()


# ------------------------------------------------------- committed fixtures


def _load(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"missing fixture {name}")
    return np.load(p)


def _csc(z, prefix, n, vals=True):
    return oracle.Csc(n, n, z[prefix + "_colptr"], z[prefix + "_rowids"], z[prefix + "_vals"] if vals else None)


@pytest.mark.parametrize("sr", ALL_SR)
def test_fixture_rmat8_square(port, sr):
    z = _load(f"rmat8_square_sr{sr}.npz")
    n = int(z["n"])
    a = _csc(z, "a", n)
    assert same(port.spgemm(sr, a, a), _csc(z, "c", n))


def test_fixture_gen_rmat_digests(port):
    z = _load("gen_rmat_digests.npz")
    for scale, nnz, digest in zip(z["scales"], z["nnz"], z["digests"]):
        m = port.gen_rmat(int(scale))
        h = hashlib.sha256(m.colptr.tobytes() + m.rowids.tobytes()).hexdigest()
        assert m.nnz == int(nnz) and h == str(digest), scale


def test_fixture_summa_2x2_fp64(port):
    """The reference's summa2d_spgemm on a 2x2 grid folds stage partials in
    stage order (summa.hpp:145-156); restating it block by block with the
    oracle reproduces it bit-for-bit."""
    from tests import sim

    z = _load("summa_p4_rmat7_f64.npz")
    n = int(z["n"])
    a = _csc(z, "a", n)
    want = _csc(z, "c", n)
    got = sim.simulate_summa2d(port, oracle.PLUS_TIMES_F64, a, a, q=2)
    assert same(got, want)


def test_fixture_ca3d_2x2x2_i64(port):
    from tests import sim

    z = _load("ca3d_p8_c2_rmat7_i64.npz")
    n = int(z["n"])
    a = _csc(z, "a", n)
    want = _csc(z, "c", n)
    got = sim.simulate_ca3d(port, oracle.PLUS_TIMES_I64, a, a, c=2, q=2)
    assert same(got, want)
