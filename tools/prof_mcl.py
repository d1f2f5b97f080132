"""Phase breakdown of mcl_step (C4: R-MAT s18 + I, column-stochastic f32) on
one GPU: the expansion alone (direct product of the same A) vs the whole step,
with per-kernel-class device times (OPT_PROFILE)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402
from bench_configs import stochastic_with_loops  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
    sr = P.PlusTimesF32
    ctx = P.Context(0)
    A = P.fill_values(P.gen_rmat(scale, 16, 1, ctx=ctx), sr, 4, ctx=ctx)
    A = stochastic_with_loops(A, sr)
    stream = torch.cuda.current_stream()
    out = {"scale": scale, "nnz_A": A.nnz}

    def run(name, fn, steps=3):
        fn()
        torch.cuda.synchronize()
        ctx.set_option(L.OPT_PROFILE, 1)
        ctx.reset_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        out[name + "_ms"] = round(e0.elapsed_time(e1) / steps, 3)
        out[name + "_classes"] = {k: round(v[1] / steps, 3) for k, v in ctx.kernel_stats().items() if v[0]}
        ctx.set_option(L.OPT_PROFILE, 0)
        return r

    c = run("expansion", lambda: P.local_spgemm(A, A, sr, ctx=ctx, method="direct"))
    out["nnz_expansion"] = c.nnz
    del c
    m = run("mcl_step", lambda: P.mcl_step(A, 2.0, 1e-4, sr=sr, ctx=ctx))
    out["nnz_mcl"] = m.nnz
    print(json.dumps(out))


if __name__ == "__main__":
    main()
