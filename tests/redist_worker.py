"""Device redistribution parity worker (launched by tests/test_gpu_redist.py
under torchrun, one process per GPU; p = 1 works on a single GPU).

Every rank builds the same inputs, runs the NCCL redistribution through the
C-ABI (slapcu_distribute_triples / slapcu_redistribute) and checks ITS OWN
resulting block bit-exactly against the oracle restatement (oracle.redistribute,
pinned to the compiled reference by tests/test_redistribute_host.py):
  * distribute_triples of per-rank triple sets with duplicates, keep-first and
    semiring-add combines, all six semirings (dist_matrix.hpp:89-119);
  * redistribute_3d of R-MAT 2D blocks for split cols / rows and every valid
    layer count, and redistribute_2d back to the identical 2D blocks
    (dist_matrix3d.hpp:117-261);
  * the reference's 3D pipeline end to end (acceptance.cpp:140-160):
    redistribute_3d(A, cols), redistribute_3d(B, rows), ca3d_spgemm,
    redistribute_2d(C3) against the oracle product's 2D block;
  * CB2B read_binary / write_binary (binary_io.cpp): reading the reference-
    written fixture gives the routed blocks, writing them back reproduces the
    reference's bytes, an s+2 R-MAT round-trips, a bad magic is a FormatError;
  * an out-of-range triple on one rank fails with IndexError on EVERY rank,
    and ranks passing different layouts all fail with ShapeError.
Prints "REDIST_OK p=<p>" on success."""
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

SRS = (P.PlusTimesF64, P.PlusTimesF32, P.PlusTimesI64, P.MinPlusI32, P.MinPlusF64, P.OrAnd)
KIND = {0: 2, 1: 1, 2: 5, 3: 3, 4: 2, 5: 0}


def grid_2d(p):
    if G.is_perfect_square(p):
        q = G.isqrt_exact(p)
        return q, q
    return 1, p


def layer_counts(p):
    return [c for c in range(1, p + 1) if p % c == 0 and G.is_perfect_square(p // c)]


def same_block(got, want, what):
    blk, rs, cs = got
    wrs, wcs, wm = want
    assert (rs, cs) == (wrs, wcs), f"{what}: offsets {(rs, cs)} vs {(wrs, wcs)}"
    h = blk.to_host()
    assert (h.nrows, h.ncols) == (wm.nrows, wm.ncols), f"{what}: shape"
    assert np.array_equal(h.colptr, wm.colptr), f"{what}: colptr"
    assert np.array_equal(h.rowids, wm.rowids), f"{what}: rowids"
    assert np.asarray(h.vals).tobytes() == np.asarray(wm.vals).tobytes(), f"{what}: values"


def host_triples(m: oracle.Csc, rs=0, cs=0):
    cnt = np.diff(m.colptr)
    cols = np.repeat(np.arange(m.ncols, dtype=np.int64), cnt) + cs
    return np.asarray(m.rowids, np.int64) + rs, cols, m.vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=10)
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    p = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    comm = D.NcclComm()
    dev = torch.device("cuda", torch.cuda.current_device())
    pr, pc = grid_2d(p)
    t2 = G.tiling_2d

    # ---- distribute_triples with duplicates, both combines, all semirings
    rng = np.random.default_rng(11)
    m, n, cnt = 97, 83, 4000
    rows = rng.integers(0, m, cnt)
    cols = rng.integers(0, n, cnt)
    rows[:1500], cols[:1500] = rows[1500:3000], cols[1500:3000]
    src = rng.integers(0, p, cnt)
    for sr in SRS:
        dt = oracle.DTYPES[sr.id]
        if sr.id == oracle.OR_AND_U8:
            vals = rng.integers(0, 2, cnt).astype(dt)
        elif np.issubdtype(dt, np.integer):
            vals = rng.integers(-100, 100, cnt).astype(dt)
        else:
            vals = rng.standard_normal(cnt).astype(dt)
        parts = [(rows[src == r], cols[src == r], vals[src == r]) for r in range(p)]
        tl = t2(m, n, pr, pc)
        for combine in ("first", "add"):
            want = oracle.redistribute(sr.id, tl.row_cuts, tl.col_cuts, tl.owner, m, n, parts, combine)[rank]
            mr, mc, mv = parts[rank]
            got = D.distribute_triples(torch.from_numpy(mr).to(dev), torch.from_numpy(mc).to(dev),
                                       torch.from_numpy(np.ascontiguousarray(mv)).to(dev), m, n, sr, comm, pr, pc,
                                       combine=combine)
            same_block(got, want, f"distribute_triples {sr.name}/{sr.dtype} {combine}")

    # ---- redistribute_3d / redistribute_2d on R-MAT blocks
    for sr in (P.PlusTimesF64, P.MinPlusI32, P.OrAnd):
        A = P.fill_values(P.gen_rmat(a.scale, 8, 5), sr, KIND[sr.id])
        h = A.to_host()
        N = A.nrows
        ao = oracle.Csc(N, N, h.colptr, h.rowids, h.vals)
        r0, rl, c0, cl = G.block2d_range(N, N, pr, pc, rank // pc, rank % pc)
        a2 = D.device_block(A, r0, rl, c0, cl)
        # oracle 2D blocks (every rank) for the expected 3D routing
        blocks2 = []
        for r in range(p):
            br0, brl, bc0, bcl = G.block2d_range(N, N, pr, pc, r // pc, r % pc)
            cp, rw, vv = G.extract_block(ao.colptr, ao.rowids, ao.vals, br0, brl, bc0, bcl)
            blocks2.append((br0, bc0, oracle.Csc(brl, bcl, cp, rw, vv)))
        for layers in layer_counts(p):
            q = G.Grid3D.make(p, layers, rank).q
            for split in ("cols", "rows"):
                t3 = G.tiling_3d(N, N, layers, q, split)
                want3 = oracle.redistribute(sr.id, t3.row_cuts, t3.col_cuts, t3.owner, N, N,
                                            [host_triples(b, rs, cs) for rs, cs, b in blocks2])[rank]
                got3 = D.redistribute_3d(a2, N, N, sr, comm, layers, split, pr, pc)
                what = f"redistribute_3d {sr.name} c={layers} {split}"
                same_block(got3, want3, what)
                back = D.redistribute_2d(got3[0], got3[1], got3[2], N, N, sr, comm, pr, pc)
                same_block(back, blocks2[rank], what + " -> 2d")

    # ---- the reference's 3D pipeline end to end
    port = oracle.port()
    for sr in (P.PlusTimesF64, P.OrAnd):
        A = P.fill_values(P.gen_rmat(a.scale, 8, 3), sr, KIND[sr.id])
        h = A.to_host()
        N = A.nrows
        ao = oracle.Csc(N, N, h.colptr, h.rowids, h.vals)
        want_c = port.spgemm(sr.id, ao, ao)
        r0, rl, c0, cl = G.block2d_range(N, N, pr, pc, rank // pc, rank % pc)
        a2 = D.device_block(A, r0, rl, c0, cl)
        for layers in layer_counts(p):
            g = G.Grid3D.make(p, layers, rank)
            a3, _, _ = D.redistribute_3d(a2, N, N, sr, comm, layers, "cols", pr, pc)
            b3, _, _ = D.redistribute_3d(a2, N, N, sr, comm, layers, "rows", pr, pc)
            c3, _ = D.ca3d_spgemm(a3, b3, sr, comm, layers)
            l, i, j = g.coords
            cr0, _, cc0, _ = G.ca3d_output_range(N, N, layers, g.q, l, i, j)
            c2, rs, cs = D.redistribute_2d(c3, cr0, cc0, N, N, sr, comm, pr, pc)
            assert (rs, cs) == (r0, c0)
            cp, rw, vv = G.extract_block(want_c.colptr, want_c.rowids, want_c.vals, r0, rl, c0, cl)
            assert_parity(c2, oracle.Csc(rl, cl, cp, rw, vv), sr.id, f"3D pipeline {sr.name} c={layers}")

    # ---- CB2B binary I/O (binary_io.cpp) against the reference-written fixtures
    gold = os.path.join(ROOT, "tests", "golden")
    path4 = os.path.join(gold, "cb2b_rmat6_p4.cb2b")
    m6, n6, rec = oracle.read_cb2b(path4)
    nnz6 = len(rec)
    parts = [(rec["row"][nnz6 * r // p:nnz6 * (r + 1) // p], rec["col"][nnz6 * r // p:nnz6 * (r + 1) // p],
              rec["val"][nnz6 * r // p:nnz6 * (r + 1) // p]) for r in range(p)]
    tl = G.tiling_2d(m6, n6, pr, pc)
    want = oracle.redistribute(oracle.PLUS_TIMES_F64, tl.row_cuts, tl.col_cuts, tl.owner, m6, n6, parts)[rank]
    blk, rs, cs, mm, nn = D.read_binary(path4, comm, pr, pc)
    assert (mm, nn) == (m6, n6)
    same_block((blk, rs, cs), want, "read_binary")
    # write the blocks back: bytes identical to the reference's write_binary rule
    obj = [f"/tmp/slapcu_cb2b_{os.getpid()}.cb2b" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out_path = obj[0]
    D.write_binary(blk, rs, cs, m6, n6, comm, out_path)
    dist.barrier()
    if rank == 0:
        z = np.load(os.path.join(gold, "cb2b_rmat6_f64.npz"))
        a6 = oracle.Csc(int(z["n"]), int(z["n"]), z["a_colptr"], z["a_rowids"], z["a_vals"])
        rows_w, cols_w, vals_w = [], [], []
        for r in range(p):
            r0, rl, c0, cl = G.block2d_range(m6, n6, pr, pc, r // pc, r % pc)
            cp, rw, vv = G.extract_block(a6.colptr, a6.rowids, a6.vals, r0, rl, c0, cl)
            cols_w.append(np.repeat(np.arange(cl, dtype=np.int64), np.diff(cp)) + c0)
            rows_w.append(rw.astype(np.int64) + r0)
            vals_w.append(vv)
        want_path = out_path + ".want"
        oracle.write_cb2b(want_path, m6, n6, np.concatenate(rows_w), np.concatenate(cols_w), np.concatenate(vals_w))
        got_b = open(out_path, "rb").read()
        assert got_b == open(want_path, "rb").read(), "write_binary bytes differ from the reference rule"
        if (pr, pc) in ((1, 1), (2, 2)):
            assert got_b == open(os.path.join(gold, f"cb2b_rmat6_p{p}.cb2b"), "rb").read()
        os.remove(want_path)
    dist.barrier()
    # round trip at scale
    A = P.fill_values(P.gen_rmat(a.scale + 2, 16, 7), P.PlusTimesF64, 2)
    N = A.nrows
    r0, rl, c0, cl = G.block2d_range(N, N, pr, pc, rank // pc, rank % pc)
    a2 = D.device_block(A, r0, rl, c0, cl)
    D.write_binary(a2, r0, c0, N, N, comm, out_path)
    assert D.binary_header(out_path) == (N, N, A.nnz)
    back, brs, bcs, _, _ = D.read_binary(out_path, comm, pr, pc)
    assert (brs, bcs) == (r0, c0)
    assert torch.equal(back.colptr, a2.colptr) and torch.equal(back.rowids, a2.rowids)
    assert torch.equal(back.vals, a2.vals)
    dist.barrier()
    if rank == 0:
        with open(out_path, "r+b") as f:
            f.write(b"XXXX")
    dist.barrier()
    try:
        D.read_binary(out_path, comm, pr, pc)
        raise AssertionError("expected FormatError")
    except P.errors.FormatError:
        pass
    dist.barrier()
    if rank == 0:
        os.remove(out_path)

    # ---- errors are raised on every rank
    bad_r = torch.tensor([0, 5 if rank != p - 1 else 10**6], dtype=torch.int64, device=dev)
    bad_c = torch.tensor([0, 1], dtype=torch.int64, device=dev)
    bad_v = torch.ones(2, dtype=torch.float64, device=dev)
    try:
        D.distribute_triples(bad_r, bad_c, bad_v, 100, 100, P.PlusTimesF64, comm, pr, pc)
        raise AssertionError("expected IndexError")
    except P.errors.IndexError_:
        pass
    if p > 1:
        tl = G.tiling_2d(100, 100, pr, pc)
        if rank == 0:  # a valid but different layout on one rank
            tl = G.Tiling(tl.row_cuts, tl.col_cuts, tuple(reversed(tl.owner)))
        try:
            D.distribute_triples(bad_r[:1], bad_c[:1], bad_v[:1], 100, 100, P.PlusTimesF64, comm, target=tl)
            raise AssertionError("expected ShapeError")
        except P.errors.ShapeError:
            pass
    c_in, _ = comm.counters(1)
    assert c_in > 0
    comm.close()
    dist.barrier()
    if rank == 0:
        print(f"REDIST_OK p={p}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
