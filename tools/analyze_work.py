"""Work distribution of A*A for an R-MAT matrix: columns, multiplies and
output entries per log2(flops) bucket and per log2(nnz) bucket, plus the
A-column-length profile of the multiplies.  Used to size the GPU work classes
(DESIGN.md).  Runs on the GPU box: python tools/analyze_work.py --scale 20"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2106_14402_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    a = ap.parse_args()
    A = P.gen_rmat(a.scale, a.ef, 1)
    tot, flops = P.estimate_flops(A, A)
    cnt = P.symbolic_nnz(A, A).cpu().numpy()
    flops = flops.cpu().numpy()
    deg = np.diff(A.colptr.cpu().numpy())
    out = {"scale": a.scale, "nnz_A": A.nnz, "flops": int(tot), "nnz_C": int(cnt.sum())}
    rows = []
    fb = np.floor(np.log2(np.maximum(flops, 1))).astype(int)
    for b in range(fb.max() + 1):
        m = fb == b
        if m.any():
            rows.append({"log2_flops": b, "cols": int(m.sum()), "flops": int(flops[m].sum()),
                         "nnz": int(cnt[m].sum())})
    out["by_flops"] = rows
    rows = []
    nb = np.floor(np.log2(np.maximum(cnt, 1))).astype(int)
    for b in range(nb.max() + 1):
        m = nb == b
        if m.any():
            rows.append({"log2_nnz": b, "cols": int(m.sum()), "flops": int(flops[m].sum()), "nnz": int(cnt[m].sum())})
    out["by_nnz"] = rows
    # multiplies grouped by the length of the A column that produces them:
    # every B entry (k, j) contributes deg(k) products
    rw = A.rowids.cpu().numpy()
    contrib = deg[rw].astype(np.int64)  # per B entry
    lb = np.floor(np.log2(np.maximum(contrib, 1))).astype(int)
    rows = []
    for b in range(lb.max() + 1):
        m = lb == b
        if m.any():
            rows.append({"log2_acol_len": b, "b_entries": int(m.sum()), "flops": int(contrib[m].sum())})
    out["by_acol_len"] = rows
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
