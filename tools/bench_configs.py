"""Secondary workloads of BASELINE.json (configs C1, C2, C4, C5) through the
public API on one B200, each with a parity spot check against the compiled
reference on a column slice and the reference's own CPU time on the same
slice.  (bench.py measures the headline C3.)  One JSON line per config.

    python tools/bench_configs.py [--configs C1,C2,C4,C5] [--steps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: parity + CPU baseline only)
import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import batched as BT  # noqa: E402


def workload(name, ctx):
    if name == "C1":  # R-MAT s14 ef16, A*A, PlusTimes f64, U[0,10) values
        a = P.fill_values(P.gen_rmat(14, 16, 1, ctx=ctx), P.PlusTimesF64, 2, ctx=ctx)
        return "C1: R-MAT s14 ef16 A*A plus_times f64 (U[0,10) values)", a, a, P.PlusTimesF64
    if name == "C2":  # ER n=2^20, 8n draws, PlusTimes f64 U[0,1)
        a = P.gen_er(1 << 20, 8 << 20, 1, ctx=ctx)
        return "C2: Erdos-Renyi n=2^20 d=8 A*A plus_times f64", a, a, P.PlusTimesF64
    if name == "C4":  # MCL expansion: R-MAT s18 column-stochastic fp32
        a = P.fill_values(P.gen_rmat(18, 16, 1, ctx=ctx), P.PlusTimesF32, 4, ctx=ctx)
        return "C4: MCL expansion, column-stochastic R-MAT s18 A*A plus_times f32", a, a, P.PlusTimesF32
    if name == "C5":  # tall-skinny: A = R-MAT s22 ef8, B = 2^22 x 2^10 one nonzero per row
        a = P.fill_values(P.gen_rmat(22, 8, 1, ctx=ctx), P.PlusTimesF64, 1, ctx=ctx)
        b = P.gen_one_per_row(1 << 22, 1 << 10, 2, ctx=ctx)
        return "C5: tall-skinny R-MAT s22 ef8 x (2^22 x 2^10, 1 nz/row) plus_times f64", a, b, P.PlusTimesF64
    raise ValueError(name)


def stochastic_with_loops(A, sr):
    """A's pattern plus the diagonal (isolated vertices would leave empty,
    zero-sum columns, which mcl_step rejects), values 1/deg(col)."""
    h = A.to_host()
    n = h.ncols
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(h.colptr))
    key = np.unique(np.concatenate([cols * n + h.rowids.astype(np.int64), np.arange(n, dtype=np.int64) * (n + 1)]))
    c, r = key // n, (key % n).astype(np.int32)
    cp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(c, minlength=n), out=cp[1:])
    deg = np.diff(cp)
    vals = np.repeat(1.0 / deg, deg).astype(sr.np_dtype)
    return P.CscMatrix(n, n, cp, r, vals).to_device()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C4,C5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-cols", type=int, default=256)
    ap.add_argument("--method", default="direct", choices=["direct", "fused", "two_pass"])
    ap.add_argument("--value-hash", type=int, default=None, help="value pass hash kernel for small items (0 off)")
    ap.add_argument("--value-interleave", type=int, default=None, help="value pass gathers interleaved: 0 off, 1 4-byte values, 2 all")
    ap.add_argument("--opt", action="append", default=[],
                    help="NAME=VALUE library option (e.g. DETERMINISTIC=1, DIRECT_ESC=1, DIRECT_WORDS=1)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    ctx = P.Context(0, stream)
    if args.value_hash is not None:
        from paper_2106_14402_b200 import _lib as L
        ctx.set_option(L.OPT_DIRECT_VALUE_HASH, args.value_hash)
    if args.value_interleave is not None:
        from paper_2106_14402_b200 import _lib as L
        ctx.set_option(L.OPT_DIRECT_VALUE_INTERLEAVE, args.value_interleave)
    from paper_2106_14402_b200 import _lib as L
    for kv in args.opt:
        k, v = kv.split("=")
        ctx.set_option(getattr(L, "OPT_" + k), int(v))
    from bench import measured_peak_gbs
    peak, peak_kind = measured_peak_gbs()
    threads = os.cpu_count() or 1
    for name in args.configs.split(","):
        desc, A, B, sr = workload(name, ctx)
        flops, _ = P.estimate_flops(A, B, ctx=ctx)
        C = P.local_spgemm(A, B, sr, ctx=ctx, method=args.method)
        nnz = C.nnz
        del C
        for _ in range(args.warmup):
            P.local_spgemm(A, B, sr, ctx=ctx, method=args.method)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            P.local_spgemm(A, B, sr, ctx=ctx, method=args.method)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        # parity + CPU reference on a column slice of B
        w = min(args.cpu_cols, B.ncols)
        c0 = 0
        ha, hb = A.to_host(), B.to_host()
        oa = oracle.Csc(ha.nrows, ha.ncols, ha.colptr, ha.rowids, ha.vals)
        ob = oracle.Csc(hb.nrows, hb.ncols, hb.colptr, hb.rowids, hb.vals)
        gpu_slice = P.local_spgemm(A, BT.column_window(B, c0, c0 + w), sr, ctx=ctx, method=args.method).to_host()
        secs, ref_nnz, ref_fl = oracle.ref().time_local_spgemm(sr.id, oa, ob, c0, c0 + w, threads)
        want = oracle.port().spgemm(sr.id, oa, ob, c0, c0 + w)
        same_pattern = bool(np.array_equal(gpu_slice.colptr, want.colptr) and
                            np.array_equal(gpu_slice.rowids, want.rowids))
        tol = 1e-12 if sr.dtype == "f64" else 1e-5
        gv, wv = gpu_slice.vals.astype(np.float64), want.vals.astype(np.float64)
        close = bool(np.all(np.abs(gv - wv) <= tol * np.maximum(1.0, np.maximum(np.abs(gv), np.abs(wv)))))
        bitwise = bool(same_pattern and gpu_slice.vals.tobytes() == np.asarray(want.vals).tobytes())
        extra = {}
        if name == "C4":  # the whole Markov-clustering step around the expansion (algorithms.cpp:267-293)
            A = stochastic_with_loops(A, sr)  # mcl_step needs every column to sum to 1
            P.mcl_step(A, 2.0, 1e-4, sr=sr, ctx=ctx)
            torch.cuda.synchronize()
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(stream)
            for _ in range(args.steps):
                P.mcl_step(A, 2.0, 1e-4, sr=sr, ctx=ctx)
            m1.record(stream)
            torch.cuda.synchronize()
            extra["mcl_step_ms"] = round(m0.elapsed_time(m1) / args.steps, 3)
            extra["mcl_step_input"] = "A + I (no empty column), values 1/deg(col), inflation 2, prune 1e-4"
        vs = np.dtype(sr.np_dtype).itemsize
        step_bytes = sum(nz * (4 + vs) + (nc + 1) * 8 for nz, nc in ((A.nnz, A.ncols), (B.nnz, B.ncols), (nnz, B.ncols)))
        print(json.dumps({
            "config": name, "workload": desc, "gflops": round(2 * flops / (ms / 1e3) / 1e9, 3),
            "ms_per_product": round(ms, 3), "multiplies": int(flops), "nnz_C": int(nnz),
            "step_bytes_alg": int(step_bytes), "step_frac_hbm": round(step_bytes / (ms / 1e3) / 1e9 / peak, 5),
            "peak_gbs": peak, "peak_source": peak_kind, "options": args.opt,
            "cpu_reference": {"gflops": round(2 * ref_fl / secs / 1e9, 4), "threads": threads,
                              "sample": f"columns [{c0},{c0 + w}) of B, {ref_fl} multiplies in {secs:.3f} s"},
            "parity_slice": {"pattern_exact": same_pattern, f"values_rel_{tol}": close, "values_bitwise": bitwise},
            **extra,
        }), flush=True)
        del A, B
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
