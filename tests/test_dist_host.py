"""Multi-process host logic on CPU (gloo): the grid geometry, block
distribution and gather used by the NCCL drivers, exercised the way the
drivers use them -- one process per rank, blocks cut with
paper_2106_14402_b200.grid, the 3D fiber exchange and the SUMMA stage
exchange done with gloo collectives, local products from the CPU oracle, and
the gathered C compared with the oracle's global product.  (The device path
of the same drivers is covered by tests/test_gpu_dist.py on >= 2 GPUs.)"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2106_14402_b200 import grid as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _blk(m, r0, rl, c0, cl):
    cp, rw, vv = G.extract_block(m.colptr, m.rowids, m.vals, r0, rl, c0, cl)
    return oracle.Csc(rl, cl, cp, rw, vv)


def _worker(rank, world, port, case, q_or_c, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = oracle.port()
    sr = oracle.PLUS_TIMES_I64
    a = P.gen_rmat(8, 8, 5)
    a = a.with_vals(P.fill_values(sr, 5, a))
    n = a.nrows
    if case == "summa":
        q = q_or_c
        g = G.Grid2D.square_of(world, rank)
        i, j = g.myrow, g.mycol
        ro, co = G.block_offsets(n, q), G.block_offsets(n, q)
        mine_a = _blk(a, ro[i], ro[i + 1] - ro[i], co[j], co[j + 1] - co[j])
        blocks = [None] * world
        dist.all_gather_object(blocks, mine_a)  # stands in for the stage broadcasts
        parts = []
        for s in range(q):
            ablk = blocks[g.rank_of(i, s)]
            bblk = blocks[g.rank_of(s, j)]
            parts.append(P.spgemm(sr, ablk, bblk))
        cb = P.merge(sr, parts)
        r0, c0 = ro[i], co[j]
    else:
        c = q_or_c
        g = G.Grid3D.make(world, c, rank)
        l, i, j = g.coords
        a3 = _blk(a, *G.regular_3d_range(n, n, c, g.q, "cols", l, i, j))
        b3 = _blk(a, *G.regular_3d_range(n, n, c, g.q, "rows", l, i, j))
        assert g.q == 1  # one stage per layer here
        cint = P.spgemm(sr, a3, b3)
        poff = G.block_offsets(cint.ncols, c)
        pieces = [_blk(cint, 0, cint.nrows, poff[k], poff[k + 1] - poff[k]) for k in range(c)]
        allp = [None] * world
        dist.all_gather_object(allp, pieces)  # stands in for the fiber alltoallv
        recv = [allp[g.rank_of(src, i, j)][l] for src in range(c)]
        cb = P.merge(sr, recv)
        r0, _, c0, _ = G.ca3d_output_range(n, n, c, g.q, l, i, j)
    parts = [None] * world if rank == 0 else None
    dist.gather_object((r0, c0, cb.colptr, cb.rowids, cb.vals), parts, dst=0)
    if rank == 0:
        cp, rw, vv = G.assemble(n, n, parts)
        want = P.spgemm(sr, a, a)
        out["ok"] = bool(np.array_equal(cp, want.colptr) and np.array_equal(rw, want.rowids)
                         and np.array_equal(vv, want.vals))
    dist.destroy_process_group()


def _run(world, case, arg):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, arg, out), nprocs=world, join=True)
    return out.get("ok", False)


def test_ca3d_geometry_two_ranks():
    assert _run(2, "ca3d", 2)


def test_summa_geometry_four_ranks():
    assert _run(4, "summa", 2)


def test_grid_shapes():
    assert G.block_offsets(10, 3) == [0, 3, 6, 10]
    assert G.block_of([0, 3, 6, 10], 6) == 2
    g = G.Grid3D.make(8, 2, 5)
    assert (g.q, g.coords) == (2, (1, 0, 1)) and g.rank_of(1, 0, 1) == 5
    with pytest.raises(Exception):
        G.Grid3D.make(8, 3, 0)
    with pytest.raises(Exception):
        G.Grid3D.make(6, 2, 0)  # p/c = 3 not square
    assert G.Grid3D.make(8, 2, 0).layer_warning is False  # c=2 <= cbrt(8)
    assert G.Grid3D.make(4, 4, 0).layer_warning is True


def test_plan_batches_by_count_matches_reference_rule():
    # batched.hpp:25-37: remainder one per range from the front
    from paper_2106_14402_b200 import batched as BT

    p = BT.plan_batches_by_count(10, 4)
    assert p.col_ranges == [(0, 3), (3, 6), (6, 8), (8, 10)]
    with pytest.raises(Exception):
        BT.plan_batches_by_count(10, 0)
    q = BT.plan_from_counts([1, 2, 3, 4], 16 * 5)
    assert q.col_ranges == [(0, 2), (2, 3), (3, 4)] and q.est_entries == [3, 3, 4]
