#!/usr/bin/env python3
"""Benchmark: semiring SpGEMM GFLOPS on R-MAT scale-20 A*A (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  A "step" is one full product C = A*A of the
configured workload through the library (symbolic + numeric for every column
batch; batches exist because C does not fit one GPU's HBM at scale 20).

* value      -- GFLOPS = 2 * multiplies / device time of the step (inputs
                resident in HBM; max over ranks for N > 1).
* e2e        -- the same metric through the public API with HOST buffers:
                H2D of A from pinned memory and D2H of every output batch
                inside the timed region.
* roofline   -- the dominant kernel's algorithmic bytes / its event-timed
                duration, against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline -- the unmodified reference (oracle/_ref/libslapref.so,
                slap::local_spgemm) on a bounded column sample of the same
                product, all host threads.

`--impl reference` runs only the reference CPU arm (rank 0) on that sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpGEMM GFLOPS (R-MAT s20 A·A) at 1/2/4/8 B200; %HBM roofline; vs CPU ref"
UNIT = "GFLOPS"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--semiring", default="or_and", choices=["or_and", "min_plus_i32"])
    ap.add_argument("--budget-gb", type=float, default=0.0, help="output bytes per column batch (0 = auto)")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-cols", type=int, default=256, help="columns per CPU-baseline slice")
    ap.add_argument("--profile", type=int, default=1)
    return ap.parse_args()


# ------------------------------------------------------------------ helpers


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def bytes_alg(nnz_a, ncols_a, nnz_b, ncols_b, nnz_c, ncols_c, vs):
    """sum over A, B, C of nnz*(4+sizeof(VT)) + (ncols+1)*8."""
    return sum(nz * (4 + vs) + (nc + 1) * 8 for nz, nc in ((nnz_a, ncols_a), (nnz_b, ncols_b), (nnz_c, ncols_c)))


def plan_batches(counts: np.ndarray, entry_bytes: int, budget: int):
    """batched.hpp:122-148 plan_batches_by_budget semantics on exact counts."""
    ranges, start, cur = [], 0, 0
    for j, cnt in enumerate(counts.tolist()):
        cost = cnt * entry_bytes
        if cost > budget:
            raise RuntimeError(f"column {j} alone needs {cost} bytes, budget {budget}")
        if cur + cost > budget:
            ranges.append((start, j))
            start, cur = j, 0
        cur += cost
    ranges.append((start, len(counts)))
    return ranges


def cpu_sample_offsets(n, w):
    # the survey's four slices (probe8: 0, n/4+12345, n/2+777, n-4096), width w
    return [0, min(n // 4 + 12345, n - w), min(n // 2 + 777, n - w), n - w]


def run_cpu_reference(sr_id, host_a, cols, threads):
    """Times the unmodified reference local_spgemm on the column sample."""
    import oracle

    R = oracle.ref()
    A = oracle.Csc(host_a.nrows, host_a.ncols, host_a.colptr, host_a.rowids, host_a.vals)
    secs = flops = 0.0
    for c0 in cpu_sample_offsets(A.ncols, cols):
        s, _nnz, f = R.time_local_spgemm(sr_id, A, A, c0, c0 + cols, threads)
        secs += s
        flops += f
    return 2.0 * flops / secs / 1e9, secs, flops


# ---------------------------------------------------------------- our arm


def run_ours(args):
    import torch

    import paper_2106_14402_b200 as P
    from paper_2106_14402_b200 import _lib as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        return run_ours_dist(args, world, rank)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    ctx = P.Context(0, stream)
    lib = ctx.lib
    sr = P.OrAnd if args.semiring == "or_and" else P.MinPlusI32
    kind = 0 if sr is P.OrAnd else 3
    vs = 1 if sr is P.OrAnd else 4

    A = P.fill_values(P.gen_rmat(args.scale, args.edge_factor, 1, ctx=ctx), sr, kind, ctx=ctx)
    n = A.ncols
    total_flops, flops_per = P.estimate_flops(A, A, ctx=ctx)
    # exact counts (validation + roofline byte accounting only; not used by the step)
    counts = P.symbolic_nnz(A, A, ctx=ctx).cpu().numpy()
    nnz_c = int(counts.sum())
    # Column batches sized by the staging bound sum_j min(flops_j, n) -- known
    # before any product is formed -- so every batch runs the single-pass
    # begin/finish with no symbolic pre-pass (batched.hpp:122-170 semantics,
    # with the flops bound in place of the symbolic count).
    bound = np.minimum(flops_per.cpu().numpy(), A.nrows)
    free, _tot = torch.cuda.mem_get_info()
    stage_entry = 4 + (0 if sr is P.OrAnd else vs)
    budget = int(args.budget_gb * 2**30) if args.budget_gb > 0 else int(min(0.30 * free, 40 * 2**30))
    batches = plan_batches(bound, stage_entry, budget)
    max_cap = max(int(bound[s:e].sum()) for s, e in batches)
    max_cols = max(e - s for s, e in batches)
    out_cp = torch.empty(max_cols + 1, dtype=torch.int64, device=dev)
    out_rw = torch.empty(max(max_cap, 1), dtype=torch.int32, device=dev)
    out_v = torch.empty(max(max_cap, 1), dtype=sr.torch_dtype, device=dev)
    av = A.view()
    import ctypes as C

    def window(c0, c1):
        return L.CscView(A.nrows, c1 - c0, A.nnz, A.colptr.data_ptr() + 8 * c0, A.rowids.data_ptr(),
                         A.vals.data_ptr())

    wins = [window(s, e) for s, e in batches]

    def step(collect=None):
        for bi, w in enumerate(wins):
            nz = C.c_int64()
            ctx.check(lib.slapcu_spgemm_begin(ctx.h, C.byref(av), C.byref(w), sr.id, P.SpGemmAlg.hybrid, 0,
                                              out_cp.data_ptr(), C.byref(nz)), "begin")
            ctx.check(lib.slapcu_spgemm_finish(ctx.h, C.byref(av), C.byref(w), sr.id, out_rw.data_ptr(),
                                               out_v.data_ptr()), "finish")
            if collect is not None:
                collect(bi, int(nz.value))

    # parity spot check of the benchmarked configuration (column checksums of
    # the first batch vs. the symbolic counts) happens in tests; here we only
    # verify totals
    got = []
    step(lambda bi, nz: got.append(nz))
    assert sum(got) == nnz_c, (sum(got), nnz_c)

    ctx.set_option(L.OPT_PROFILE, int(args.profile))
    for _ in range(args.warmup - 1):
        step()
    torch.cuda.synchronize()
    ctx.reset_stats()
    launches0 = ctx.launches
    clocks = ClockSampler(0)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = (ctx.launches - launches0) // args.steps
    kstats = ctx.kernel_stats()
    ctx.set_option(L.OPT_PROFILE, 0)
    value = 2.0 * total_flops / (ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel class
    peak, peak_kind = measured_peak_gbs()
    per_step = {k: (nl / args.steps, t / args.steps) for k, (nl, t) in kstats.items() if nl}
    dom = max(per_step, key=lambda k: per_step[k][1])
    # heavy columns of the fused path: flops > max(256, min(n/128, 4096))
    lmax = max(256, min(A.nrows // 128, 4096))
    fl = flops_per.cpu().numpy()
    heavy = fl > lmax
    colnnz_b = np.diff(A.colptr.cpu().numpy())
    dom_bytes = 0
    for s, e in batches:
        h = heavy[s:e] if dom in ("sym_heavy", "num_heavy") else ~heavy[s:e]
        nh = int(h.sum())
        if nh == 0:
            continue
        c_ent = int(counts[s:e][h].sum())
        b_ent = int(colnnz_b[s:e][h].sum())
        if dom == "sym_heavy":  # k_fused_heavy: B cols + A (pattern) in, staged rows out
            dom_bytes += c_ent * 4 + b_ent * 4 + (nh + 1) * 8 + A.nnz * 4 + (n + 1) * 8
        elif dom == "num_heavy":  # k_values_heavy: C rows in, values out, B and A with values
            dom_bytes += c_ent * (4 + vs) + b_ent * (4 + vs) + (nh + 1) * 8 + A.nnz * (4 + vs) + (n + 1) * 8
        elif dom == "sym_light":  # k_fused_light: staged rows+values out
            dom_bytes += c_ent * (4 + vs) + b_ent * (4 + vs) + (nh + 1) * 8
        else:  # copies: read staged, write C
            dom_bytes += 2 * c_ent * (4 + vs) + (nh + 1) * 8
    dom_ms = per_step[dom][1]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    step_bytes = bytes_alg(A.nnz, n, A.nnz, n, nnz_c, n, vs)
    roofline = {
        "bound": "hbm",
        "kernel": {"sym_heavy": "k_fused_heavy", "sym_light": "k_fused_light", "num_heavy": "k_values_heavy",
                   "num_light": "k_copy_light+k_copy_heavy"}.get(dom, dom),
        "achieved": round(achieved, 2),
        "peak": peak,
        "unit": "GB/s",
        "frac": round(achieved / peak, 5),
        "traffic": None,
        "peak_source": peak_kind,
        "dominant_share_of_step": round(dom_ms / ms, 4),
        "launches_per_step": per_step[dom][0],
        "algorithmic_bytes_per_step": dom_bytes,
        "step_bytes_alg": step_bytes,
        "step_achieved_gbs": round(step_bytes / (ms / 1e3) / 1e9, 2),
        "step_frac": round(step_bytes / (ms / 1e3) / 1e9 / peak, 5),
        "class_ms_per_step": {k: round(v[1], 3) for k, v in per_step.items()},
    }

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e_single(args, A, sr, batches, counts, total_flops, ctx, stream)

    # ---- CPU baseline (reference, bounded sample)
    cpu = None
    if not args.no_cpu:
        try:
            host = A.to_host()
            threads = os.cpu_count() or 1
            gf, secs, fl = run_cpu_reference(sr.id, host, args.cpu_cols, threads)
            cpu = {"value": round(gf, 4), "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"slap::local_spgemm(A, A(:, J)) hybrid, 4 slices x {args.cpu_cols} cols at offsets "
                             f"{cpu_sample_offsets(n, args.cpu_cols)}; {int(fl)} multiplies in {secs:.2f} s"}
        except Exception as ex:  # the reference .so is optional on the box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": sr.dtype,
        "data": "synthetic",
        "config": {
            "workload": f"C3: R-MAT scale {args.scale} ef {args.edge_factor} seed 1, C = A*A, {sr.name} {sr.dtype}",
            "semiring": f"{sr.name}_{sr.dtype}",
            "n": n, "nnz_A": A.nnz, "multiplies": total_flops, "nnz_C": nnz_c,
            "column_batches": len(batches),
            "batch_budget_bytes": budget,
            "parallelism": "single GPU",
            "l2": "inputs/outputs larger than L2 (A 157 MB, C >> 126 MB); no flush",
        },
        "gpu_launches": int(launches),
        "clocks": clk,
        "roofline": roofline,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_e2e_single(args, A, sr, batches, counts, total_flops, ctx, stream):
    """Host-buffer end-to-end: H2D of A (pinned) + per-batch SpGEMM + D2H of
    every batch's C (chunked into a pinned ring) inside the timed region."""
    import ctypes as C

    import torch

    import paper_2106_14402_b200 as P
    from paper_2106_14402_b200 import _lib as L

    vs = 1 if sr is P.OrAnd else 4
    h_cp = A.colptr.cpu().pin_memory()
    h_rw = A.rowids.cpu().pin_memory()
    h_v = A.vals.cpu().pin_memory()
    d_cp = torch.empty_like(A.colptr)
    d_rw = torch.empty_like(A.rowids)
    d_v = torch.empty_like(A.vals)
    max_nnz = max(int(counts[s:e].sum()) for s, e in batches)
    max_cols = max(e - s for s, e in batches)
    o_cp = torch.empty(max_cols + 1, dtype=torch.int64, device=A.colptr.device)
    o_rw = torch.empty(max(max_nnz, 1), dtype=torch.int32, device=A.colptr.device)
    o_v = torch.empty(max(max_nnz, 1), dtype=sr.torch_dtype, device=A.colptr.device)
    chunk = 1 << 28  # elements per D2H chunk
    h_out_rw = torch.empty(chunk, dtype=torch.int32).pin_memory()
    h_out_v = torch.empty(chunk, dtype=sr.torch_dtype).pin_memory()
    h_out_cp = torch.empty(max_cols + 1, dtype=torch.int64).pin_memory()
    lib = ctx.lib
    h2d = A.colptr.numel() * 8 + A.nnz * (4 + vs)
    d2h = 0

    def one():
        nonlocal d2h
        d2h = 0
        d_cp.copy_(h_cp, non_blocking=True)
        d_rw.copy_(h_rw, non_blocking=True)
        d_v.copy_(h_v, non_blocking=True)
        av = L.CscView(A.nrows, A.ncols, A.nnz, d_cp.data_ptr(), d_rw.data_ptr(), d_v.data_ptr())
        for s, e in batches:
            w = L.CscView(A.nrows, e - s, A.nnz, d_cp.data_ptr() + 8 * s, d_rw.data_ptr(), d_v.data_ptr())
            nz = C.c_int64()
            ctx.check(lib.slapcu_spgemm_begin(ctx.h, C.byref(av), C.byref(w), sr.id, P.SpGemmAlg.hybrid, 0,
                                              o_cp.data_ptr(), C.byref(nz)), "begin")
            ctx.check(lib.slapcu_spgemm_finish(ctx.h, C.byref(av), C.byref(w), sr.id, o_rw.data_ptr(),
                                               o_v.data_ptr()), "finish")
            nzv = int(nz.value)
            h_out_cp[: e - s + 1].copy_(o_cp[: e - s + 1], non_blocking=True)
            d2h += (e - s + 1) * 8
            for o in range(0, nzv, chunk):
                m = min(chunk, nzv - o)
                h_out_rw[:m].copy_(o_rw[o:o + m], non_blocking=True)
                h_out_v[:m].copy_(o_v[o:o + m], non_blocking=True)
                d2h += m * (4 + vs)
        torch.cuda.current_stream().synchronize()

    one()  # warm-up
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(max(args.e2e_steps, 1)):
        one()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / max(args.e2e_steps, 1)
    wall = (time.perf_counter() - t0) / max(args.e2e_steps, 1)
    return {"value": round(2.0 * total_flops / (ms / 1e3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3), "wall_ms_per_step": round(wall * 1e3, 3),
            "steps": max(args.e2e_steps, 1)}


def run_ours_dist(args, world, rank):
    raise SystemExit("multi-GPU bench: see bench_dist (not yet enabled)")


# ----------------------------------------------------------- reference arm


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    sr_id = oracle.OR_AND_U8 if args.semiring == "or_and" else oracle.MIN_PLUS_I32
    kind = 0 if sr_id == oracle.OR_AND_U8 else 3
    Pp = oracle.port()
    a = Pp.gen_rmat(args.scale, args.edge_factor, 1)
    a = a.with_vals(Pp.fill_values(sr_id, kind, a))
    threads = os.cpu_count() or 1
    vals = []
    for it in range(args.warmup + args.steps):
        gf, secs, fl = run_cpu_reference(sr_id, a, args.cpu_cols, threads)
        if it >= args.warmup:
            vals.append((gf, secs, fl))
    gf = statistics.mean(v[0] for v in vals)
    secs = statistics.mean(v[1] for v in vals)
    fl = vals[0][2]
    sample = (f"slap::local_spgemm(A, A(:, J)) hybrid, 4 slices x {args.cpu_cols} cols at offsets "
              f"{cpu_sample_offsets(a.ncols, args.cpu_cols)}; {int(fl)} multiplies per step")
    line = {
        "metric": METRIC, "value": round(gf, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(secs * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8" if sr_id == oracle.OR_AND_U8 else "i32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"C3: R-MAT scale {args.scale} ef {args.edge_factor} seed 1, C = A*A (column sample)",
                   "semiring": args.semiring, "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": round(gf, 4), "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(gf, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
