"""Generates the committed fixtures in tests/golden/ from the UNMODIFIED
reference compiled in place (oracle/_ref/libslapref.so, built by
oracle/Makefile from /root/reference/proj/core).  Run in the build
container:  python tests/golden/make_golden.py

Fixtures:
  rmat8_square_sr{S}.npz     A = gen_rmat(8,16,1) with the SURVEY value
                             recipe of semiring S; C = slap::local_spgemm(A, A)
  gen_rmat_digests.npz       nnz and sha256(colptr|rowids) of gen_rmat(s,16,1)
                             for s in 8, 10, 12, 14 (reference generator)
  summa_p4_rmat7_f64.npz     slap::summa2d_spgemm on a 2x2 grid (fp64, values
                             U[0,10)): stage-order fold differs bitwise from
                             the local product
  ca3d_p8_c2_rmat7_i64.npz   slap::ca3d_spgemm on a 2x2x2 grid (i64)
  cb2b_rmat6_f64.npz         A = gen_rmat(6,16,1), values U[0,10) (f64)
  cb2b_rmat6_p1.cb2b         slap::write_binary of A distributed on 1x1
  cb2b_rmat6_p4.cb2b         ... on 2x2 (records rank by rank, each rank's
                             column-major block order)
(`python tests/golden/make_golden.py cb2b` regenerates only the CB2B files.)
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

KIND = {0: 2, 1: 1, 2: 5, 3: 3, 4: 5, 5: 0}


def save(name, **kw):
    np.savez_compressed(os.path.join(HERE, name), **kw)


def main():
    R = oracle.ref()
    P = oracle.port()  # only for the value recipes (pinned by tests)
    a = R.gen_rmat(8, 16, 1)
    for sr in range(6):
        av = a.with_vals(P.fill_values(sr, KIND[sr], a))
        c = R.local_spgemm(sr, av, av, alg=oracle.HYBRID, threads=2)
        save(f"rmat8_square_sr{sr}.npz", n=a.nrows, a_colptr=av.colptr, a_rowids=av.rowids, a_vals=av.vals,
             c_colptr=c.colptr, c_rowids=c.rowids, c_vals=c.vals)
    scales, nnz, digests = [], [], []
    for s in (8, 10, 12, 14):
        m = R.gen_rmat(s, 16, 1)
        scales.append(s)
        nnz.append(m.nnz)
        digests.append(hashlib.sha256(m.colptr.tobytes() + m.rowids.tobytes()).hexdigest())
    save("gen_rmat_digests.npz", scales=np.array(scales), nnz=np.array(nnz), digests=np.array(digests))
    a7 = R.gen_rmat(7, 16, 1)
    av = a7.with_vals(P.fill_values(oracle.PLUS_TIMES_F64, 2, a7))
    c, stages, bcasts = R.summa2d(oracle.PLUS_TIMES_F64, av, av, p=4)
    assert stages == 2 and bcasts == 4, (stages, bcasts)
    save("summa_p4_rmat7_f64.npz", n=a7.nrows, a_colptr=av.colptr, a_rowids=av.rowids, a_vals=av.vals,
         c_colptr=c.colptr, c_rowids=c.rowids, c_vals=c.vals)
    ai = a7.with_vals(P.fill_values(oracle.PLUS_TIMES_I64, 5, a7))
    c3 = R.ca3d(oracle.PLUS_TIMES_I64, ai, ai, p=8, pr=2, pc=4, layers=2)
    save("ca3d_p8_c2_rmat7_i64.npz", n=a7.nrows, a_colptr=ai.colptr, a_rowids=ai.rowids, a_vals=ai.vals,
         c_colptr=c3.colptr, c_rowids=c3.rowids, c_vals=c3.vals)
    cb2b()
    print("fixtures written to", HERE)


def cb2b():
    R = oracle.ref()
    P = oracle.port()
    a6 = R.gen_rmat(6, 16, 1)
    av = a6.with_vals(P.fill_values(oracle.PLUS_TIMES_F64, 2, a6))
    save("cb2b_rmat6_f64.npz", n=a6.nrows, a_colptr=av.colptr, a_rowids=av.rowids, a_vals=av.vals)
    R.write_binary(av, os.path.join(HERE, "cb2b_rmat6_p1.cb2b"), p=1, pr=1, pc=1)
    R.write_binary(av, os.path.join(HERE, "cb2b_rmat6_p4.cb2b"), p=4, pr=2, pc=2)


if __name__ == "__main__":
    cb2b() if sys.argv[1:] == ["cb2b"] else main()
