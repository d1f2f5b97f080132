"""Same-process A/B of the ESC policy on C2 / C5 (auto vs forced vs off)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402

ctx = P.Context(0)
cfgs = {
    "C5": (lambda: P.fill_values(P.gen_rmat(22, 8, 1, ctx=ctx), P.PlusTimesF64, 1, ctx=ctx),
           lambda: P.gen_one_per_row(1 << 22, 1 << 10, 2, ctx=ctx)),
    "C2": (lambda: P.gen_er(1 << 20, 8 << 20, 1, ctx=ctx), None),
}
for name, (ga, gb) in cfgs.items():
    A = ga()
    B = gb() if gb else A
    for mode in (-1, 1, 0, -1):
        ctx.set_option(L.OPT_DIRECT_ESC, mode)
        for _ in range(3):
            P.local_spgemm(A, B, P.PlusTimesF64, ctx=ctx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.local_spgemm(A, B, P.PlusTimesF64, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        print(name, "esc", mode, round(e0.elapsed_time(e1) / 5, 3), "ms", flush=True)
