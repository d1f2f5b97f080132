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
    ap.add_argument("--sym-tile-log2", type=int, default=0, help="row-tile height of the pattern bitmap (0 = default)")
    ap.add_argument("--tile-log2", type=int, default=0, help="row-tile height of the value pass (0 = default)")
    ap.add_argument("--dense-min", type=int, default=None, help="byte-flag pattern path for flops >= this (0 off)")
    ap.add_argument("--direct-tile-log2", type=int, default=0, help="rows per direct-path item (0 = default)")
    ap.add_argument("--direct-split", type=int, default=None, help="direct path: split items above this many flops")
    ap.add_argument("--form-threads", type=int, default=None, help="direct path form CTA size")
    ap.add_argument("--dense-run", type=int, default=None, help="direct path dense A-run threshold (0 off)")
    ap.add_argument("--persistent", type=int, default=None, help="direct path form kernel persistent (1) or not (0)")
    ap.add_argument("--value-tile-log2", type=int, default=None, help="direct path value pass sub-tile rows")
    ap.add_argument("--value-threads", type=int, default=None, help="direct path value pass CTA size")
    ap.add_argument("--value-hash", type=int, default=None, help="direct path value pass hash table (0/13/14)")
    ap.add_argument("--value-rank", type=int, default=None, help="direct path value pass rank chunk (0 = sub-tiles)")
    ap.add_argument("--value-interleave", type=int, default=None,
                    help="direct path value pass: 4-byte values gathered with their rows (1) or not (0)")
    ap.add_argument("--tile-major", type=int, default=None, help="direct path form: units ordered by row tile (1)")
    ap.add_argument("--short-run", type=int, default=None, help="direct path form: per-thread run threshold")
    ap.add_argument("--value-tmajor", type=int, default=None, help="direct value pass: tile-major table + row-order chunks")
    ap.add_argument("--words", type=int, default=None, help="direct form: walk A's (word, mask) pairs")
    ap.add_argument("--value-dense-rows", type=int, default=None, help="direct value pass: dense-chunk row span")
    ap.add_argument("--opt", action="append", default=[], help="NAME=VALUE library option (OPT_NAME)")
    ap.add_argument("--sub-timeout", type=float, default=480.0,
                    help="N>1: seconds the SUMMA / 3D sub-measurement may take before the line is printed without it")
    ap.add_argument("--dist", default="1d", choices=["1d", "summa"],
                    help="N>1: 1d = flops-balanced column blocks with A replicated (no data-path collective); "
                         "summa = the 2D SUMMA / 3D drivers (NCCL stage broadcasts, fiber exchange, merge)")
    ap.add_argument("--balance-out", type=float, default=3.0, help="1d split: weight of a column's output bound")
    ap.add_argument("--balance-col", type=float, default=2000.0, help="1d split: per-column weight")
    ap.add_argument("--calibrate", type=int, default=4, help="1d split: timed re-balancing rounds before warmup")
    ap.add_argument("--second", type=int, default=1,
                    help="1: also measure MinPlus int32 C3 (BASELINE's other C3 semiring) into the same line")
    return ap.parse_args()


def apply_options(ctx, args):
    from paper_2106_14402_b200 import _lib as L

    if args.sym_tile_log2:
        ctx.set_option(L.OPT_SYM_TILE_ROWS_LOG2, args.sym_tile_log2)
    if args.tile_log2:
        ctx.set_option(L.OPT_TILE_ROWS_LOG2, args.tile_log2)
    if args.dense_min is not None:
        ctx.set_option(L.OPT_DENSE_FLOPS_MIN, args.dense_min)
    if args.direct_tile_log2:
        ctx.set_option(L.OPT_DIRECT_TILE_ROWS_LOG2, args.direct_tile_log2)
    if args.direct_split is not None:
        ctx.set_option(L.OPT_DIRECT_SPLIT_FLOPS, args.direct_split)
    if args.form_threads is not None:
        ctx.set_option(L.OPT_DIRECT_FORM_THREADS, args.form_threads)
    if args.dense_run is not None:
        ctx.set_option(L.OPT_DIRECT_DENSE_RUN_MIN, args.dense_run)
    if args.persistent is not None:
        ctx.set_option(L.OPT_DIRECT_PERSISTENT, args.persistent)
    if args.tile_major is not None:
        ctx.set_option(L.OPT_DIRECT_TILE_MAJOR, args.tile_major)
    if args.short_run is not None:
        ctx.set_option(L.OPT_DIRECT_SHORT_RUN, args.short_run)
    if args.value_tmajor is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_TMAJOR, args.value_tmajor)
    if args.words is not None:
        ctx.set_option(L.OPT_DIRECT_WORDS, args.words)
    if args.value_dense_rows is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_DENSE_ROWS, args.value_dense_rows)
    for kv in args.opt:
        k, v = kv.split("=")
        ctx.set_option(getattr(L, "OPT_" + k), int(v))
    if args.value_rank is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_RANK, args.value_rank)
    if args.value_interleave is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_INTERLEAVE, args.value_interleave)
    if args.value_hash is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_HASH, args.value_hash)
    if args.value_threads is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_THREADS, args.value_threads)
    if args.value_tile_log2 is not None:
        ctx.set_option(L.OPT_DIRECT_VALUE_TILE_ROWS_LOG2, args.value_tile_log2)


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
            return
        # nvidia-smi takes a while to produce its first line; a short timed
        # region could otherwise end before any sample.  Wait until it is live
        # (bounded) and keep only the samples taken after this point.
        t0 = time.time()
        while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.02)
        self.skip = len(self.lines)

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
        lines = self.lines[getattr(self, "skip", 0):] or self.lines
        for ln in lines:
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


def flops_balanced_blocks(flops: np.ndarray, parts: int):
    """Column boundaries [b_0 = 0, ..., b_parts = n] splitting the columns into
    `parts` contiguous blocks of (nearly) equal multiplies."""
    n = len(flops)
    cum = np.cumsum(flops)
    total = int(cum[-1]) if n else 0
    inner = [int(np.searchsorted(cum, total * r / parts)) for r in range(1, parts)]
    return [0] + [min(max(b, 0), n) for b in inner] + [n]


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_cpu_reference_slices(sr_id, host_a, cols, threads, want_result=False, t1_slices=(1, 2, 3)):
    """The unmodified reference local_spgemm (oracle/_ref/libslapref.so) on the
    column sample A*A(:, J) for J = the survey's four slices: rate with all
    `threads`, the single-thread rate on the slices in `t1_slices` (the hub
    slice 0 alone would take ~20 s on one core), and optionally each slice's
    product for the parity check."""
    import oracle

    R = oracle.ref()
    A = oracle.Csc(host_a.nrows, host_a.ncols, host_a.colptr, host_a.rowids, host_a.vals)
    secs = flops = 0.0
    results = []
    for c0 in cpu_sample_offsets(A.ncols, cols):
        r = R.time_local_spgemm(sr_id, A, A, c0, c0 + cols, threads, want_result=want_result)
        secs += r[0]
        flops += r[2]
        results.append(((c0, c0 + cols), r[3] if want_result else None))
    t1 = None
    if t1_slices:
        s1 = f1 = 0.0
        offs = cpu_sample_offsets(A.ncols, cols)
        for i in t1_slices:
            r = R.time_local_spgemm(sr_id, A, A, offs[i], offs[i] + cols, 1)
            s1 += r[0]
            f1 += r[2]
        t1 = {"value": round(2.0 * f1 / s1 / 1e9, 4), "unit": UNIT, "cores": 1,
              "sample": f"slices {list(t1_slices)}: {int(f1)} multiplies in {s1:.2f} s"}
    return 2.0 * flops / secs / 1e9, secs, flops, results, t1


def run_ours(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        return run_ours_multi(args, world, rank)
    import torch

    import paper_2106_14402_b200 as P

    torch.cuda.set_device(0)
    head = P.OrAnd if args.semiring == "or_and" else P.MinPlusI32
    line = measure_single(args, head)
    # BASELINE C3 names both semirings: the other one rides in the same line
    if args.second and head is P.OrAnd:
        torch.cuda.empty_cache()
        sub = measure_single(args, P.MinPlusI32)
        line["min_plus_i32"] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "dtype", "config", "gpu_launches",
                                                     "clocks", "roofline", "e2e", "cpu_baseline", "parity")}
    print(json.dumps(line), flush=True)


def measure_single(args, sr):
    """C3 on one GPU for semiring `sr`: device-resident step (value), the
    roofline of the form+emit pair, parity of four column slices against the
    reference, e2e through slapcu_batched_spgemm_host, and the CPU baseline."""
    import ctypes as C

    import torch

    import paper_2106_14402_b200 as P
    from paper_2106_14402_b200 import _lib as L

    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    ctx = P.Context(0, stream)
    apply_options(ctx, args)
    lib = ctx.lib
    kind = 0 if sr is P.OrAnd else 3
    vs = 1 if sr is P.OrAnd else 4

    A = P.fill_values(P.gen_rmat(args.scale, args.edge_factor, 1, ctx=ctx), sr, kind, ctx=ctx)
    n = A.ncols
    total_flops, flops_per = P.estimate_flops(A, A, ctx=ctx)
    # exact per-column counts from the two-pass symbolic kernels (an
    # independent code path): per-column check of the direct product and the
    # roofline byte accounting; not used by the step
    counts = P.symbolic_nnz(A, A, ctx=ctx).cpu().numpy()
    nnz_c = int(counts.sum())
    # Column batches sized by the bound sum_j min(flops_j, n) -- known before
    # any product is formed -- so no symbolic pre-pass runs inside the step
    # (batched.hpp:122-170 semantics with the flops bound for the count).
    bound = np.minimum(flops_per.cpu().numpy(), A.nrows)
    free, _tot = torch.cuda.mem_get_info()
    # (half the free memory, at most 96 GB, for the bound-sized C buffers: C3 OrAnd in 3 column
    # batches instead of 5 at 0.35 / 64 GB -- 134.9 -> 130.9 ms/step, fewer per-batch setups)
    budget = int(args.budget_gb * 2**30) if args.budget_gb > 0 else int(min(0.5 * free, 96 * 2**30))
    batches = plan_batches(bound, 4 + vs, budget)
    max_cap = max(int(bound[s:e].sum()) for s, e in batches)
    max_cols = max(e - s for s, e in batches)
    o_cp = torch.empty(max_cols + 1, dtype=torch.int64, device=dev)
    o_rw = torch.empty(max(max_cap, 1), dtype=torch.int32, device=dev)
    o_v = torch.empty(max(max_cap, 1), dtype=sr.torch_dtype, device=dev)
    av = A.view()

    def window(c0, c1):
        return L.CscView(A.nrows, c1 - c0, A.nnz, A.colptr.data_ptr() + 8 * c0, A.rowids.data_ptr(),
                         A.vals.data_ptr())

    wins = [window(s, e) for s, e in batches]

    def step(after=None):
        # a step is one whole product: per-A setup (tile pointers, dense runs)
        # is rebuilt once per step and shared by its column batches
        ctx.invalidate()
        for bi, w in enumerate(wins):
            nz = C.c_int64()
            ctx.check(lib.slapcu_spgemm_direct(ctx.h, C.byref(av), C.byref(w), sr.id, P.SpGemmAlg.hybrid,
                                               o_rw.numel(), o_cp.data_ptr(), o_rw.data_ptr(), o_v.data_ptr(),
                                               C.byref(nz)), "direct")
            if after is not None:
                after(bi, int(nz.value))
        ctx.check(lib.slapcu_ctx_synchronize(ctx.h), "synchronize")

    # ---- verification step (untimed): per-column nnz of every batch against
    # the symbolic counts, and the sample slices captured from the batched
    # output for the bit-exact comparison with the reference below
    slices = [(c0, c0 + args.cpu_cols) for c0 in cpu_sample_offsets(n, args.cpu_cols)]
    captured = {s: [] for s in slices}
    col_ok = [True]
    nz_total = [0]

    def verify(bi, nz):
        s, e = batches[bi]
        nz_total[0] += nz
        cp = o_cp[: e - s + 1].cpu().numpy()
        if not np.array_equal(np.diff(cp), counts[s:e]) or cp[0] != 0:
            col_ok[0] = False
        for (c0, c1) in slices:
            p0, p1 = max(c0, s), min(c1, e)
            if p0 >= p1:
                continue
            lo, hi = int(cp[p0 - s]), int(cp[p1 - s])
            captured[(c0, c1)].append((p0, p1, bi, lo, cp[p0 - s:p1 - s + 1] - lo, o_rw[lo:hi].cpu().numpy(),
                                       o_v[lo:hi].cpu().numpy()))

    step(verify)
    assert nz_total[0] == nnz_c, (nz_total[0], nnz_c)

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

    # ---- roofline: the form + emit pair (+ value pass) is the dominant unit
    peak, peak_kind = measured_peak_gbs()
    per_step = {k: (nl / args.steps, t / args.steps) for k, (nl, t) in kstats.items() if nl}
    fl = flops_per.cpu().numpy()
    heavy = fl > 1024  # direct path light/heavy split (direct_light_flops_max)
    colnnz_b = np.diff(A.colptr.cpu().numpy())
    batch_bytes = []
    for s, e in batches:
        h = heavy[s:e]
        nh = int(h.sum())
        batch_bytes.append(int(colnnz_b[s:e][h].sum()) * (4 + vs) + int(counts[s:e][h].sum()) * (4 + vs) +
                           2 * (nh + 1) * 8 + A.nnz * (4 + vs) + (n + 1) * 8 if nh else 0)
    pair_ms = per_step.get("sym_heavy", (0, 0.0))[1] + per_step.get("num_heavy", (0, 0.0))[1]
    dom_bytes = sum(batch_bytes)
    achieved = dom_bytes / (pair_ms / 1e3) / 1e9 if pair_ms else 0.0
    step_bytes = bytes_alg(A.nnz, n, A.nnz, n, nnz_c, n, vs)
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{sr.name}_{sr.dtype}", {})
    except Exception:
        pass
    nlaunch = sum(1 for b in batch_bytes if b)
    kernels = {}
    if "sym_heavy" in per_step:
        fm = per_step["sym_heavy"][1]
        kernels["k_tile_form"] = {
            "ms_per_step": round(fm, 3), "multiplies_per_s": round(total_flops / (fm / 1e3), 1),
            "gather_bytes_per_step": int(fl[heavy].sum()) * 4,
            "note": "pattern walk: one test-then-set shared bitmap update per multiply; A row ids gathered "
                    "from L2"}
    if "num_heavy" in per_step:
        em = per_step["num_heavy"][1]
        c_bytes = int(counts[heavy].sum()) * (4 + vs)
        kernels["k_tile_emit" + ("" if sr is P.OrAnd else "+value pass")] = {
            "ms_per_step": round(em, 3), "c_bytes_per_step": c_bytes,
            "achieved": round(c_bytes / (em / 1e3) / 1e9, 2), "frac": round(c_bytes / (em / 1e3) / 1e9 / peak, 4)}
    roofline = {
        "bound": "hbm",
        "kernel": "k_tile_form+k_tile_emit" + ("" if sr is P.OrAnd else "+value pass") +
                  " (one product over the heavy columns of a column batch)",
        "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 5),
        "traffic": traffic.get("dram_bytes_per_launch"),
        "traffic_alg_bytes_same_batch": traffic.get("alg_bytes_same_batch"),
        "traffic_over_alg_same_batch": traffic.get("traffic_over_alg"),
        "traffic_source": traffic.get("source"),
        "alg_bytes_per_launch": round(dom_bytes / max(nlaunch, 1)),
        "alg_bytes_per_batch": batch_bytes,
        "peak_source": peak_kind,
        "dominant_share_of_step": round(pair_ms / ms, 4),
        "launches_per_step": nlaunch,
        "algorithmic_bytes_per_step": dom_bytes,
        "step_bytes_alg": step_bytes,
        "step_achieved_gbs": round(step_bytes / (ms / 1e3) / 1e9, 2),
        "step_frac": round(step_bytes / (ms / 1e3) / 1e9 / peak, 5),
        "class_ms_per_step": {k: round(v[1], 3) for k, v in per_step.items()},
        "kernels": kernels,
    }
    del o_cp, o_rw, o_v
    torch.cuda.empty_cache()

    # ---- e2e through the reference-facing host call
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e_host(args, A, sr, budget, total_flops, ctx)

    # ---- CPU baseline + parity on the same slices (reference, bounded sample)
    cpu, parity = None, {"checked": False}
    host = None
    if not args.no_cpu:
        try:
            host = A.to_host()
            threads = os.cpu_count() or 1
            gf, secs, f_s, results, t1 = run_cpu_reference_slices(sr.id, host, args.cpu_cols, threads,
                                                                   want_result=True)
            cpu = {"value": round(gf, 4), "unit": UNIT, "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(), "t1": t1,
                   "sample": f"slap::local_spgemm(A, A(:, J)) hybrid, 4 slices x {args.cpu_cols} cols at offsets "
                             f"{[s[0] for s in slices]}; {int(f_s)} multiplies in {secs:.2f} s"}
            parity = check_slices(results, captured, sr)
        except Exception as ex:  # the reference .so is optional on the box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}
            parity = {"checked": False, "why": str(ex)}
    parity["per_column_nnz_vs_symbolic"] = bool(col_ok[0])
    if args.scale == 20 and args.edge_factor == 16:
        # the survey's reference-measured totals (SURVEY.md Appendix A probe)
        parity["totals_match_reference"] = bool(total_flops == 70065456202 and nnz_c == 23721688001)

    return {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "strong",
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
        "parity": parity,
    }


def check_slices(results, captured, sr):
    """Bit-exact comparison (integer / Boolean semirings) of the reference's
    C(:, J) with the GPU's batched output for the same columns."""
    out = {"checked": True, "rule": "bit-exact colptr, rowids and values (integer / Boolean semiring)",
           "slices": []}
    ok_all = True
    for (c0, c1), want in results:
        parts = captured[(c0, c1)]
        cps, rws, vls = [np.zeros(1, np.int64)], [], []
        base = 0
        for (_p0, _p1, _bi, _lo, cp, rw, v) in parts:
            cps.append(cp[1:] + base)
            base += int(cp[-1])
            rws.append(rw)
            vls.append(v)
        g_cp = np.concatenate(cps)
        g_rw = np.concatenate(rws) if rws else np.zeros(0, np.int32)
        g_v = np.concatenate(vls) if vls else np.zeros(0, sr.np_dtype)
        exact = (np.array_equal(g_cp, want.colptr) and np.array_equal(g_rw, want.rowids) and
                 g_v.astype(sr.np_dtype).tobytes() == np.asarray(want.vals, sr.np_dtype).tobytes())
        ok_all &= bool(exact)
        out["slices"].append({"cols": [c0, c1], "nnz": int(want.colptr[-1]), "exact": bool(exact),
                              "batches": sorted({p[2] for p in parts}),
                              "max_batch_offset": max([int(p[3]) for p in parts] + [0])})
    out["all_exact"] = bool(ok_all)
    return out


def run_e2e_host(args, A, sr, budget, total_flops, ctx):
    """End to end through the reference-facing host call
    (slapcu_batched_spgemm_host = batched.hpp:153-170 with host operands): A
    in pinned host memory, H2D of A and B inside the call, every column batch
    of C read back into pinned host memory and handed to a consumer.  Timed
    with CUDA events around the (synchronous) call."""
    import torch

    import paper_2106_14402_b200 as P
    from paper_2106_14402_b200 import batched as BT

    hcp = A.colptr.cpu().pin_memory()
    hrw = A.rowids.cpu().pin_memory()
    hv = A.vals.cpu().pin_memory()
    ha = P.CscMatrix(A.nrows, A.ncols, hcp.numpy(), hrw.numpy(), hv.numpy())
    free, _ = torch.cuda.mem_get_info()
    e2e_budget = int(min(0.12 * free, 16 * 2**30))
    moved = [0, 0]

    def consumer(r, s, e, c):
        moved[0] += c.colptr.nbytes + c.rowids.nbytes + c.vals.nbytes
        moved[1] += int(c.colptr[-1])

    BT.batched_spgemm_host(ha, ha, sr, budget_bytes=e2e_budget, consumer=consumer, ctx=ctx)  # warm-up (pins buffers)
    stream = torch.cuda.current_stream()
    ms_all = []
    for _ in range(max(args.e2e_steps, 1)):
        moved[0] = moved[1] = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        nnz = BT.batched_spgemm_host(ha, ha, sr, budget_bytes=e2e_budget, consumer=consumer, ctx=ctx)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms_all.append(e0.elapsed_time(e1))
    ms = statistics.mean(ms_all)
    assert moved[1] == nnz
    h2d = 2 * (hcp.numel() * 8 + hrw.numel() * 4 + hv.numel() * hv.element_size())  # A and B (= A) operands
    return {"value": round(2.0 * total_flops / (ms / 1e3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(moved[0]), "ms_per_step": round(ms, 3), "wall_ms_per_step": round(wall * 1e3, 3),
            "steps": max(args.e2e_steps, 1),
            "api": "slapcu_batched_spgemm_host (host A, B; per-batch host consumer)",
            "batch_budget_bytes": e2e_budget}


def run_ours_multi(args, world, rank):
    """N GPUs: the headline line is the --dist mode (default 1d); the other
    driver runs in the same job and rides in the line as a sub-object, so a
    scaling run records both the in-box 1D split and the SUMMA / 3D drivers
    (exposed broadcast per stage, merge time) the north_star names."""
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    first = run_ours_1d if args.dist == "1d" else run_ours_dist
    second = run_ours_dist if args.dist == "1d" else run_ours_1d
    line = first(args, world, rank)
    torch.cuda.empty_cache()
    dist.barrier()
    if args.second:
        sub_args = argparse.Namespace(**vars(args))
        sub_args.no_e2e = True  # the headline carries the e2e leg
        key = "summa_3d" if args.dist == "1d" else "split_1d"
        # The sub-measurement must not cost the headline line: an exception is
        # recorded in the sub-object, and a watchdog on every rank prints the
        # line (rank 0) and ends the process if it does not finish (the 2x2x2
        # 3D grid of N = 8 has only ever run on a driver box).
        def _watchdog():
            if rank == 0:
                line[key] = {"error": f"did not finish within {args.sub_timeout} s"}
                print(json.dumps(line), flush=True)
            os._exit(0)

        timer = threading.Timer(args.sub_timeout, _watchdog)
        timer.daemon = True
        timer.start()
        try:
            sub = second(sub_args, world, rank)
        except Exception as e:  # noqa: BLE001 -- recorded, the headline stands
            # (peers may be waiting in a collective: no barrier, this rank ends here
            # and theirs end by their watchdogs)
            if rank == 0:
                line[key] = {"error": f"{type(e).__name__}: {e}"[:300]}
                print(json.dumps(line), flush=True)
            sys.stdout.flush()
            os._exit(0)
        timer.cancel()
        if rank == 0:
            line[key] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "config", "gpu_launches", "roofline",
                                             "dist") if k in sub}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def dist_shape(world: int):
    """p=4 -> 2D 2x2 SUMMA; p=2 -> 3D c=2 q=1; p=8 -> 3D 2x2x2 (2D needs a square
    grid, summa.hpp:112-113); other p: 3D with c=p/q^2 for the largest square q^2."""
    import math

    if int(math.isqrt(world)) ** 2 == world and world > 1 and world != 8:
        return "summa", 1
    for q in range(int(math.isqrt(world)), 0, -1):
        if world % (q * q) == 0:
            return "ca3d", world // (q * q)
    return "ca3d", world


def run_ours_1d(args, world, rank):
    """N GPUs, one process each, C = A*A split by flops-balanced column
    blocks: every rank holds A (the replicated operand of CombBLAS's in-node
    GPU scheme) and forms C(:, J_rank) with the direct path in
    column batches.  No collective on the data path; the time is the max over
    ranks of CUDA-event time."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2106_14402_b200 as P
    from paper_2106_14402_b200 import _lib as L

    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    ctx = P.Context(local, stream)
    apply_options(ctx, args)
    lib = ctx.lib
    sr = P.OrAnd if args.semiring == "or_and" else P.MinPlusI32
    kind = 0 if sr is P.OrAnd else 3
    vs = 1 if sr is P.OrAnd else 4
    A = P.fill_values(P.gen_rmat(args.scale, args.edge_factor, 1, ctx=ctx), sr, kind, ctx=ctx)
    n = A.ncols
    total_flops, flops_per = P.estimate_flops(A, A, ctx=ctx)
    fl = flops_per.cpu().numpy()
    # balance multiplies plus output-proportional work (the bound on a
    # column's entries) plus a per-column constant
    weight = fl + args.balance_out * np.minimum(fl, A.nrows) + args.balance_col
    bnd = flops_balanced_blocks(weight, world)
    free, _tot = torch.cuda.mem_get_info()
    budget = int(args.budget_gb * 2**30) if args.budget_gb > 0 else int(min(0.35 * free, 64 * 2**30))
    o_bufs = {}

    def plan(bnd):
        c0, c1 = bnd[rank], bnd[rank + 1]
        bound = np.minimum(fl[c0:c1], A.nrows)
        batches = [(s + c0, e + c0) for s, e in plan_batches(bound, 4, budget)] if c1 > c0 else []
        max_cap = max([int(bound[s - c0:e - c0].sum()) for s, e in batches] + [1])
        max_cols = max([e - s for s, e in batches] + [1])
        if o_bufs.get("cap", 0) < max_cap or o_bufs.get("cols", 0) < max_cols:
            o_bufs.clear()
            torch.cuda.empty_cache()
            o_bufs.update(cap=max_cap, cols=max_cols,
                          cp=torch.empty(max_cols + 1, dtype=torch.int64, device=dev),
                          rw=torch.empty(max_cap, dtype=torch.int32, device=dev),
                          v=torch.empty(max_cap, dtype=sr.torch_dtype, device=dev))
        return batches, max_cols

    batches, max_cols = plan(bnd)

    def step(Ad, collect=None, d2h=None):
        ctx.invalidate()  # per-A setup once per step, shared by the step's batches
        o_cp, o_rw, o_v = o_bufs["cp"], o_bufs["rw"], o_bufs["v"]
        av = L.CscView(A.nrows, n, A.nnz, Ad[0].data_ptr(), Ad[1].data_ptr(), Ad[2].data_ptr())
        for s, e in batches:
            w = L.CscView(A.nrows, e - s, A.nnz, Ad[0].data_ptr() + 8 * s, Ad[1].data_ptr(), Ad[2].data_ptr())
            nz = C.c_int64()
            ctx.check(lib.slapcu_spgemm_direct(ctx.h, C.byref(av), C.byref(w), sr.id, P.SpGemmAlg.hybrid,
                                               o_rw.numel(), o_cp.data_ptr(), o_rw.data_ptr(), o_v.data_ptr(),
                                               C.byref(nz)), "direct")
            if collect is not None:
                collect.append(int(nz.value))
            if d2h is not None:
                d2h(e - s, int(nz.value))

    # one calibration step: scale each rank's weights by its measured time per
    # unit weight and re-split (ranks differ in time per multiply: hub columns
    # have dense outputs, the tail has many small columns)
    Adev0 = (A.colptr, A.rowids, A.vals)
    step(Adev0)

    def measure():
        step(Adev0)  # settle the library's per-batch caches for this split first
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(Adev0)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        ts = [torch.zeros(1, device=dev, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ts, t)
        return [float(x.item()) for x in ts]

    # re-split until the measured max stops improving (the time per unit of
    # weight changes with the split: batch counts, hub columns); keep the best
    best = None
    for it in range(args.calibrate + 1):
        ts = measure()
        if best is None or max(ts) < best[0]:
            best = (max(ts), list(bnd))
        if it == args.calibrate:
            break
        for r in range(world):
            wr = weight[bnd[r]:bnd[r + 1]]
            if wr.sum() > 0:
                weight[bnd[r]:bnd[r + 1]] = wr * (ts[r] / float(wr.sum()))
        bnd = flops_balanced_blocks(weight, world)
        batches, max_cols = plan(bnd)
    if best[1] != bnd:
        bnd = best[1]
        batches, max_cols = plan(bnd)
    o_cp, o_rw, o_v = o_bufs["cp"], o_bufs["rw"], o_bufs["v"]

    Adev = (A.colptr, A.rowids, A.vals)
    got = []
    step(Adev, collect=got)
    nnz_local = sum(got)
    for _ in range(args.warmup - 1):
        step(Adev)
    torch.cuda.synchronize()
    launches0 = ctx.launches
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(Adev)
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop() if clocks else None
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    launches = (ctx.launches - launches0) // args.steps

    # ---- e2e: A from pinned host memory, every output batch back to pinned host memory
    e2e_ms, h2d, d2h_bytes = 0.0, 0, 0
    if not args.no_e2e:
        hA = [x.cpu().pin_memory() for x in Adev]
        dA = [torch.empty_like(x) for x in Adev]
        chunk = 1 << 28
        h_rw = torch.empty(chunk, dtype=torch.int32).pin_memory()
        h_v = torch.empty(chunk, dtype=sr.torch_dtype).pin_memory()
        h_cp = torch.empty(max_cols + 1, dtype=torch.int64).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in hA)
        moved = [0]

        def pull(ncols, nzv):
            h_cp[:ncols + 1].copy_(o_cp[:ncols + 1], non_blocking=True)
            moved[0] += (ncols + 1) * 8
            for o in range(0, nzv, chunk):
                m = min(chunk, nzv - o)
                h_rw[:m].copy_(o_rw[o:o + m], non_blocking=True)
                h_v[:m].copy_(o_v[o:o + m], non_blocking=True)
                moved[0] += m * (4 + vs)

        def e2e_step():
            moved[0] = 0
            for d, h in zip(dA, hA):
                d.copy_(h, non_blocking=True)
            step(dA, d2h=pull)
            torch.cuda.current_stream().synchronize()

        e2e_step()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(max(args.e2e_steps, 1)):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / max(args.e2e_steps, 1)
        d2h_bytes = moved[0]
        dist.barrier()
    tm = torch.tensor([ms_rank, e2e_ms, float(nnz_local), float(h2d), float(d2h_bytes)], device=dev,
                      dtype=torch.float64)
    per_rank = [torch.zeros(1, device=dev, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(per_rank, tm[:1].clone())
    mx = tm.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tm.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if rank == 0:
        ms = float(mx[0])
        nnz_c = int(sm[2])
        peak, peak_kind = measured_peak_gbs()
        step_bytes = bytes_alg(A.nnz, n, A.nnz, n, nnz_c, n, vs)
        per_gpu = step_bytes / world / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": round(2.0 * total_flops / (ms / 1e3) / 1e9, 3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": sr.dtype,
            "data": "synthetic",
            "config": {
                "workload": f"C3: R-MAT scale {args.scale} ef {args.edge_factor} seed 1, C = A*A, {sr.name} {sr.dtype}",
                "semiring": f"{sr.name}_{sr.dtype}", "n": n, "nnz_A": A.nnz, "multiplies": total_flops,
                "nnz_C": nnz_c, "parallelism": f"1D column blocks x{world} (A replicated, flops-balanced)",
                "column_blocks": bnd, "column_batches_rank0": len(batches),
                "rank_ms": [round(float(x.item()), 3) for x in per_rank],
                "l2": "inputs/outputs larger than L2; no flush"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "roofline": {"bound": "hbm", "kernel": "whole local multiply per GPU", "achieved": round(per_gpu, 2),
                         "peak": peak, "unit": "GB/s", "frac": round(per_gpu / peak, 5), "traffic": None,
                         "peak_source": peak_kind, "algorithmic_bytes_per_step": step_bytes},
            "e2e": None if args.no_e2e else {
                "value": round(2.0 * total_flops / (float(mx[1]) / 1e3) / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(sm[3]), "d2h_bytes_per_step": int(sm[4]),
                "ms_per_step": round(float(mx[1]), 3), "steps": max(args.e2e_steps, 1)},
            "cpu_baseline": None,
        }
        return line
    return None


def run_ours_dist(args, world, rank):
    """N GPUs, one process each: the same C3 product through the NCCL drivers
    (slapcu_summa2d / slapcu_ca3d), in column batches of every rank's B block
    (batched.hpp:153-170); time = max over ranks of CUDA-event time."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2106_14402_b200 as P
    from paper_2106_14402_b200 import _lib as L
    from paper_2106_14402_b200 import dist as D
    from paper_2106_14402_b200 import grid as G

    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    ctx = P.Context(local, stream)
    apply_options(ctx, args)
    comm = D.NcclComm(ctx)
    sr = P.OrAnd if args.semiring == "or_and" else P.MinPlusI32
    kind = 0 if sr is P.OrAnd else 3
    vs = 1 if sr is P.OrAnd else 4
    A0 = P.fill_values(P.gen_rmat(args.scale, args.edge_factor, 1, ctx=ctx), sr, kind, ctx=ctx)
    total_flops, flops_per = P.estimate_flops(A0, A0, ctx=ctx)
    # symmetric relabelling P A P^T: same flops and nnz(C), balanced blocks
    A = P.permute_symmetric(A0, 7, sr, ctx=ctx)
    del A0
    n = A.nrows
    mode, layers = dist_shape(world)
    if mode == "summa":
        q = G.isqrt_exact(world)
        a_loc = D.block_2d(A, q, rank)
        b_loc = a_loc
        out_div = q  # a rank's output is ~ its column block's share over q row blocks
    else:
        g = G.Grid3D.make(world, layers, rank)
        q = g.q
        a_loc = D.block_3d(A, layers, q, rank, "cols")
        b_loc = D.block_3d(A, layers, q, rank, "rows")
        out_div = q * layers
    fl = flops_per.cpu().numpy()
    bound_total = int(np.minimum(fl, n).sum())
    free, _ = torch.cuda.mem_get_info()
    budget = int(args.budget_gb * 2**30) if args.budget_gb > 0 else int(min(0.3 * free, 48 * 2**30))
    # per-rank staging bound of one product over the whole local B block
    est = bound_total * (4 + vs) // max(out_div, 1) * 2
    nb = max(1, -(-est // budget))
    t = torch.tensor([nb], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    nb = int(t.item())
    lc = b_loc.ncols
    wins = [D.column_window(b_loc, (b * lc) // nb, ((b + 1) * lc) // nb) for b in range(nb)]
    av = a_loc.view()
    bvs = [w.view() for w in wins]
    lib = ctx.lib
    totals = {"local": 0.0, "merge": 0.0, "bcast": 0.0, "nnz": 0}

    def step(record=False):
        for bv in bvs:
            out = L.CscOut()
            st = L.DistStats()
            if mode == "summa":
                rc = lib.slapcu_summa2d(comm.h, C.byref(av), C.byref(bv), sr.id, int(P.SpGemmAlg.hybrid), C.byref(out),
                                        C.byref(st))
            else:
                rc = lib.slapcu_ca3d(comm.h, layers, C.byref(av), C.byref(bv), sr.id, int(P.SpGemmAlg.hybrid),
                                     C.byref(out), C.byref(st))
            ctx.check(rc, mode)
            if record:
                totals["local"] += st.ms_local
                totals["merge"] += st.ms_merge
                totals["bcast"] += st.ms_exposed_bcast
                totals["nnz"] += int(out.nnz)
            D.free_out(ctx, out)  # consumer: discard (batched.hpp:168)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    ctx.set_option(L.OPT_PROFILE, int(args.profile))
    ctx.reset_stats()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    t_wall = time.perf_counter()
    for s in range(args.steps):
        step(record=(s == 0))
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall = (time.perf_counter() - t_wall) / args.steps * 1e3
    dist.barrier()
    clk = clocks.stop() if clocks else None
    ms_local_rank = ev0.elapsed_time(ev1) / args.steps
    class_ms = {k: round(t / args.steps, 3) for k, (nl, t) in ctx.kernel_stats().items() if nl}
    ctx.set_option(L.OPT_PROFILE, 0)

    # ---- e2e: this rank's blocks H2D from pinned memory, every output batch D2H
    e2e_ms, h2d, d2h = 0.0, 0, 0
    if not args.no_e2e:
        cud = L.cudart()
        hbuf = torch.empty(1 << 28, dtype=torch.uint8).pin_memory()

        def pin(m):
            return [m.colptr.cpu().pin_memory(), m.rowids.cpu().pin_memory(), m.vals.cpu().pin_memory()]

        ha = pin(a_loc)
        hb = ha if b_loc is a_loc else pin(b_loc)
        da = [x.to(dev) for x in ha]
        db = da if hb is ha else [x.to(dev) for x in hb]
        a2 = P.DeviceCsc(a_loc.nrows, a_loc.ncols, *da)
        b2 = P.DeviceCsc(b_loc.nrows, b_loc.ncols, *db)
        av2 = a2.view()
        bvs2 = [D.column_window(b2, (b * lc) // nb, ((b + 1) * lc) // nb).view() for b in range(nb)]
        h2d = sum(x.numel() * x.element_size() for x in ha) + (0 if hb is ha else sum(
            x.numel() * x.element_size() for x in hb))

        def e2e_step():
            nonlocal d2h
            d2h = 0
            for dst, src in zip(da, ha):
                dst.copy_(src, non_blocking=True)
            if db is not da:
                for dst, src in zip(db, hb):
                    dst.copy_(src, non_blocking=True)
            for bv in bvs2:
                out = L.CscOut()
                st = L.DistStats()
                if mode == "summa":
                    rc = lib.slapcu_summa2d(comm.h, C.byref(av2), C.byref(bv), sr.id, int(P.SpGemmAlg.hybrid),
                                            C.byref(out), C.byref(st))
                else:
                    rc = lib.slapcu_ca3d(comm.h, layers, C.byref(av2), C.byref(bv), sr.id, int(P.SpGemmAlg.hybrid),
                                         C.byref(out), C.byref(st))
                ctx.check(rc, mode)
                for ptr, nbytes in ((out.colptr, 8 * (out.ncols + 1)), (out.rowids, 4 * out.nnz),
                                    (out.vals, vs * out.nnz)):
                    for o in range(0, nbytes, hbuf.numel()):
                        m = min(hbuf.numel(), nbytes - o)
                        cud.cudaMemcpyAsync(C.c_void_p(hbuf.data_ptr()), C.c_void_p(ptr + o), C.c_size_t(m), 2,
                                            C.c_void_p(stream.cuda_stream))
                        d2h += m
                D.free_out(ctx, out)
            torch.cuda.current_stream().synchronize()

        e2e_step()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(max(args.e2e_steps, 1)):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / max(args.e2e_steps, 1)
        dist.barrier()
    tm = torch.tensor([ms_local_rank, totals["local"], totals["merge"], totals["bcast"], float(totals["nnz"]), e2e_ms,
                       float(h2d), float(d2h)], device=dev, dtype=torch.float64)
    mx = tm.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tm.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    ms = float(mx[0])
    launches = (ctx.launches - launches0) // args.steps
    bc_calls, bc_bytes = comm.counters(0)
    a2a_calls, a2a_bytes = comm.counters(1)
    if rank == 0:
        peak, peak_kind = measured_peak_gbs()
        nnz_c = int(sm[4])
        step_bytes = bytes_alg(A.nnz, n, A.nnz, n, nnz_c, n, vs)
        per_gpu = step_bytes / world / (ms / 1e3) / 1e9
        value = 2.0 * total_flops / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": sr.dtype, "data": "synthetic",
            "config": {
                "workload": f"C3: R-MAT scale {args.scale} ef {args.edge_factor} seed 1, C = A*A, {sr.name} {sr.dtype}",
                "semiring": f"{sr.name}_{sr.dtype}", "n": n, "nnz_A": A.nnz, "multiplies": total_flops,
                "nnz_C": nnz_c, "parallelism": ("2D SUMMA %dx%d" % (q, q)) if mode == "summa"
                else "3D %dx%dx%d" % (layers, q, q),
                "column_batches": nb, "relabel": "symmetric P*A*P^T (seed 7), flops and nnz(C) unchanged",
                "l2": "inputs/outputs larger than L2; no flush"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "dist": {"rank0_class_ms_per_step": class_ms, "rank0_host_ms_per_step": round(t_wall, 3),
                     "ms_local_max": round(float(mx[1]), 3), "ms_merge_max": round(float(mx[2]), 3),
                     "ms_exposed_bcast_max": round(float(mx[3]), 3),
                     "ms_exposed_bcast_per_stage_mean": round(float(sm[3]) / world / max(1, nb * q), 4),
                     "stages": q, "bcast_calls_rank0": bc_calls, "bcast_bytes_rank0": bc_bytes,
                     "alltoallv_calls_rank0": a2a_calls, "alltoallv_bytes_rank0": a2a_bytes},
            "roofline": {"bound": "hbm", "kernel": "whole local multiply per GPU",
                         "achieved": round(per_gpu, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(per_gpu / peak, 5), "traffic": None, "peak_source": peak_kind,
                         "algorithmic_bytes_per_step": step_bytes},
            "e2e": None if args.no_e2e else {
                "value": round(2.0 * total_flops / (float(mx[5]) / 1e3) / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(sm[6]), "d2h_bytes_per_step": int(sm[7]),
                "ms_per_step": round(float(mx[5]), 3), "steps": max(args.e2e_steps, 1)},
            "cpu_baseline": None,
        }
    comm.close()
    dist.barrier()
    return line if rank == 0 else None


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
