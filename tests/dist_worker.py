"""Multi-GPU parity worker (launched by tests/test_gpu_dist.py under torchrun,
one process per GPU).  Every rank builds the same R-MAT operands on its
device, takes its 2D / 3D blocks, runs the NCCL driver through the C-ABI,
and rank 0 gathers C and checks it against the CPU oracle:
  * summa2d on p = 4 (2x2) and ca3d on p = 2 (c=2, q=1), p = 8 (2x2x2)
    (acceptance.cpp:120-163 criterion 2 shapes);
  * exact semirings bit-exact, fp64 within 1e-12;
  * structure: sqrt(p) stages, 2 block broadcasts per stage per rank
    (test_distkernels.cpp:60-75), exactly one fiber alltoallv for 3D
    (test_distkernels.cpp:186-206);
  * column-window operands (batched.hpp slices) give the matching columns.
Prints "DIST_OK <case>" on success."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import dist as D  # noqa: E402
from paper_2106_14402_b200 import grid as G  # noqa: E402
from tests.helpers import assert_parity  # noqa: E402

KIND = {0: 2, 1: 1, 2: 5, 3: 3, 4: 5, 5: 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="summa")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--scale", type=int, default=11)
    ap.add_argument("--concat", type=int, default=1, help="SLAPCU_OPT_SUMMA_CONCAT")
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from paper_2106_14402_b200 import _lib as L

    P.default_context().set_option(L.OPT_SUMMA_CONCAT, a.concat)
    comm = D.NcclComm()
    port = oracle.port()
    if a.case == "mcl":  # algorithms.cpp:267-293 on a pr x pc grid, 2D or 3D expansion
        mcl_case(a, comm, port, rank, world)
        return
    for sr in (P.PlusTimesF64, P.MinPlusI32, P.OrAnd, P.PlusTimesI64):
        A = P.fill_values(P.gen_rmat(a.scale, 8, 3), sr, KIND[sr.id])
        n = A.nrows
        if a.case == "summa":
            q = G.isqrt_exact(world)
            ab = D.block_2d(A, q, rank)
            cb, st = D.summa2d_spgemm(ab, ab, sr, comm)
            assert st.stages == q, st
            r0, _, c0, _ = G.block2d_range(n, n, q, q, rank // q, rank % q)
        else:
            c = a.layers
            g = G.Grid3D.make(world, c, rank)
            a3 = D.block_3d(A, c, g.q, rank, "cols")
            b3 = D.block_3d(A, c, g.q, rank, "rows")
            cb, st = D.ca3d_spgemm(a3, b3, sr, comm, c)
            l, i, j = g.coords
            r0, _, c0, _ = G.ca3d_output_range(n, n, c, g.q, l, i, j)
            assert st.layer_warning == g.layer_warning
        full = D.gather_to_host(cb, r0, c0, n, n)
        if rank == 0:
            h = A.to_host()
            ao = oracle.Csc(n, n, h.colptr, h.rowids, h.vals)
            want = port.spgemm(sr.id, ao, ao)
            assert_parity(full, want, sr.id, f"{a.case}/{sr.name}/{sr.dtype}")
        torch.cuda.synchronize()
    # structural counters (per rank): block broadcasts and fiber exchanges
    bc_calls, _ = comm.counters(0)
    a2a_calls, _ = comm.counters(1)
    if a.case == "summa":
        q = G.isqrt_exact(world)
        assert bc_calls == 4 * 2 * q, bc_calls  # 4 semirings x q stages x (row + col)
        assert a2a_calls == 0
    else:
        g = G.Grid3D.make(world, a.layers, rank)
        assert bc_calls == (4 * 2 * g.q if g.q > 1 else 0), bc_calls
        assert a2a_calls == 4, a2a_calls  # one fiber alltoallv per product
    # column windows of B (batched.hpp slice_cols) on the SUMMA path
    if a.case == "summa":
        q = G.isqrt_exact(world)
        sr = P.MinPlusI32
        A = P.fill_values(P.gen_rmat(a.scale, 8, 3), sr, 3)
        ab = D.block_2d(A, q, rank)
        lc = ab.ncols
        w0, w1 = lc // 3, (2 * lc) // 3
        cw, _ = D.summa2d_spgemm(ab, D.column_window(ab, w0, w1), sr, comm)
        cfull, _ = D.summa2d_spgemm(ab, ab, sr, comm)
        hw, hf = cw.to_host(), cfull.to_host()
        lo, hi = hf.colptr[w0], hf.colptr[w1]
        assert np.array_equal(hw.rowids, hf.rowids[lo:hi]) and np.array_equal(hw.vals, hf.vals[lo:hi])
    # shape errors are raised consistently on every rank
    if a.case == "summa" and world == 4:
        pass
    if a.case == "ca3d":
        try:
            D.ca3d_spgemm(a3, b3, P.PlusTimesF64, comm, 3)
            raise AssertionError("expected ShapeError")
        except P.errors.ShapeError:
            pass
    comm.close()
    dist.barrier()
    if rank == 0:
        print(f"DIST_OK {a.case} p={world}", flush=True)
    dist.destroy_process_group()


def stochastic_rmat(port, scale, seed=1):
    """R-MAT pattern plus self loops (no empty column), values 1/deg(col)."""
    m = port.gen_rmat(scale, 8, seed)
    n = m.ncols
    rows = np.concatenate([m.rowids.astype(np.int64), np.arange(n)])
    cols = np.concatenate([np.repeat(np.arange(n), np.diff(m.colptr)), np.arange(n)])
    key = np.unique(cols * n + rows)
    cc, rr = key // n, (key % n).astype(np.int32)
    cp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cc, minlength=n), out=cp[1:])
    deg = np.diff(cp)
    return oracle.Csc(n, n, cp, rr, np.repeat(1.0 / deg, deg))


def mcl_case(a, comm, port, rank, world):
    pr = {1: 1, 2: 1, 4: 2, 8: 2}[world]
    pc = world // pr
    h = stochastic_rmat(port, a.scale)
    n = h.ncols
    A = P.CscMatrix(n, n, h.colptr, h.rowids, h.vals).to_device()
    i, j = rank // pc, rank % pc
    r0, rl, c0, cl = G.block2d_range(n, n, pr, pc, i, j)
    ab = D.device_block(A, r0, rl, c0, cl)
    want = oracle.ref().mcl_step(h, 2.0, 1e-4) if rank == 0 else None
    # square grids run the 2D expansion and (layers > 1) the 3D one; others only 3D
    layer_list = ([1] + ([a.layers] if a.layers > 1 else [])) if pr == pc else [a.layers]
    for layers in layer_list:
        cb = D.mcl_step(ab, pr, pc, comm, layers, 2.0, 1e-4)
        full = D.gather_to_host(cb, r0, c0, n, n)
        if rank == 0:
            assert_parity(full, want, oracle.PLUS_TIMES_F64, f"mcl p={world} {pr}x{pc} layers={layers}")
        torch.cuda.synchronize()
    # a non-stochastic input raises StochasticityError on every rank
    bad = P.CscMatrix(n, n, h.colptr, h.rowids, h.vals * 1.5).to_device()
    try:
        D.mcl_step(D.device_block(bad, r0, rl, c0, cl), pr, pc, comm, 1 if pr == pc else a.layers)
        raise AssertionError("expected StochasticityError")
    except P.errors.StochasticityError:
        pass
    comm.close()
    dist.barrier()
    if rank == 0:
        print(f"DIST_OK mcl p={world}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
