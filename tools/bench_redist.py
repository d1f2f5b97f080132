"""Device redistribution throughput under torchrun, one
process per GPU: R-MAT s<scale> (ef 16, PlusTimes f64 values) on the
sqrt(p) x sqrt(p) 2D layout (1 x p when p is not square) is redistributed to
the c x q x q 3D layout split by columns (redistribute_3d,
dist_matrix3d.hpp:117-170) and back (redistribute_2d, :250-261), timed with
CUDA events per step, max over ranks, median step reported (mean and max
beside it).  Also times distribute_triples of the
whole matrix held as COO on rank 0 (the reference's test pattern,
dist_matrix.hpp:89-119).  Rank 0 prints one JSON line per operation:
entries/s over all ranks and the bytes moved per entry.

    torchrun --nproc-per-node 4 tools/bench_redist.py --scale 20 --layers 4
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import dist as D  # noqa: E402
from paper_2106_14402_b200 import grid as G  # noqa: E402


STEPS = []


def timed(fn, steps, warmup, comm):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record()
    for k in range(steps):
        fn()
        ev[k + 1].record()
    torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    if os.environ.get("REDIST_VERBOSE"):
        print(f"rank {dist.get_rank()} per-step ms: {[round(x, 2) for x in per]}", file=sys.stderr, flush=True)
    # per-step max over ranks, then the median step (isolated slow steps --
    # allocator / host hiccups -- are reported as ms_max, not averaged in)
    t = torch.tensor(per, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    STEPS.append({"ms_mean": round(float(t.mean()), 3), "ms_max": round(float(t.max()), 3)})
    return float(t.median())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--layers", type=int, default=0, help="0: largest valid c")
    ap.add_argument("--steps", type=int, default=9)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--ref-scale", type=int, default=18, help="reference CB2B timing scale (p=1 only; 0 = off)")
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    p = int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    comm = D.NcclComm()
    sr = P.PlusTimesF64
    if G.is_perfect_square(p):
        pr = pc = G.isqrt_exact(p)
    else:
        pr, pc = 1, p
    layers = a.layers or max(c for c in range(1, p + 1) if p % c == 0 and G.is_perfect_square(p // c))
    A = P.fill_values(P.gen_rmat(a.scale, 16, 1), sr, 2)
    N = A.nrows
    nnz = A.nnz
    r0, rl, c0, cl = G.block2d_range(N, N, pr, pc, rank // pc, rank % pc)
    a2 = D.device_block(A, r0, rl, c0, cl)
    holder = {}

    def to3d():
        holder["a3"] = D.redistribute_3d(a2, N, N, sr, comm, layers, "cols", pr, pc)

    ms3 = timed(to3d, a.steps, a.warmup, comm)
    a3, rs3, cs3 = holder["a3"]

    def to2d():
        holder["b2"] = D.redistribute_2d(a3, rs3, cs3, N, N, sr, comm, pr, pc)

    ms2 = timed(to2d, a.steps, a.warmup, comm)
    b2 = holder["b2"][0]
    assert torch.equal(b2.colptr, a2.colptr) and torch.equal(b2.rowids, a2.rowids) and torch.equal(b2.vals, a2.vals)
    # distribute_triples: the whole matrix as COO on rank 0
    if rank == 0:
        cnt = A.colptr[1:] - A.colptr[:-1]
        cols = torch.repeat_interleave(torch.arange(N, device=A.rowids.device), cnt)
        rows = A.rowids.to(torch.int64)
        vals = A.vals
    else:
        dev = A.rowids.device
        rows = cols = torch.zeros(0, dtype=torch.int64, device=dev)
        vals = torch.zeros(0, dtype=torch.float64, device=dev)

    def dtrip():
        holder["d"] = D.distribute_triples(rows, cols, vals, N, N, sr, comm, pr, pc)

    msd = timed(dtrip, a.steps, a.warmup, comm)
    d = holder["d"][0]
    assert torch.equal(d.colptr, a2.colptr) and torch.equal(d.rowids, a2.rowids) and torch.equal(d.vals, a2.vals)
    # CB2B write_binary / read_binary through /tmp (binary_io.cpp)
    obj = [f"/tmp/bench_redist_{os.getpid()}.cb2b" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    path = obj[0]

    def wr():
        D.write_binary(a2, r0, c0, N, N, comm, path)

    msw = timed(wr, a.steps, a.warmup, comm)

    def rd():
        holder["r"] = D.read_binary(path, comm, pr, pc)

    msr = timed(rd, a.steps, a.warmup, comm)
    rb = holder["r"][0]
    assert torch.equal(rb.colptr, a2.colptr) and torch.equal(rb.rowids, a2.rowids) and torch.equal(rb.vals, a2.vals)
    ref_line = None
    if rank == 0 and p == 1 and a.ref_scale > 0:
        import time

        import oracle

        if oracle.ref_available():
            R = oracle.ref()
            Ar = P.fill_values(P.gen_rmat(a.ref_scale, 16, 1), sr, 2).to_host()
            ao = oracle.Csc(Ar.nrows, Ar.ncols, Ar.colptr, Ar.rowids, Ar.vals)
            rp = path + ".ref"
            t0 = time.perf_counter()
            R.write_binary(ao, rp)
            t1 = time.perf_counter()
            R.read_binary(rp)
            t2 = time.perf_counter()
            os.remove(rp)
            ref_line = {"scale": a.ref_scale, "nnz": ao.nnz, "write_s": round(t1 - t0, 3), "read_s": round(t2 - t1, 3),
                        "write_entries_per_s": ao.nnz / (t1 - t0), "read_entries_per_s": ao.nnz / (t2 - t1),
                        "kind": "reference", "cores": 1}
    dist.barrier()
    if rank == 0:
        os.remove(path)
        base = {"unit": "entries/s", "n_gpus": p, "scale": a.scale, "nnz": nnz, "pr": pr, "pc": pc,
                "layers": layers, "steps": a.steps, "warmup": a.warmup, "semiring": "plus_times f64",
                "wire_bytes_per_entry": 16, "parity": "round trip bit-exact"}
        for op, ms in (("redistribute_3d (2D -> 3D split cols)", ms3), ("redistribute_2d (3D -> 2D)", ms2),
                       ("distribute_triples (COO on rank 0 -> 2D)", msd),
                       ("write_binary (CB2B, /tmp)", msw), ("read_binary (CB2B, /tmp -> 2D)", msr)):
            line = dict(base, op=op, ms=round(ms, 3), value=nnz / (ms * 1e-3), **STEPS.pop(0))
            if op.startswith(("write_binary", "read_binary")):
                line["file_gb_per_s"] = round(nnz * 24 / (ms * 1e-3) / 1e9, 3)
                if ref_line:
                    line["cpu_baseline"] = ref_line
            print(json.dumps(line), flush=True)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
