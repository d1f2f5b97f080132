"""Debug: value-walk counters of one MinPlus C3 column batch (variant build
with -DSLAPCU_VCOUNT; SLAPCU_LIB points at it)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_14402_b200 as P  # noqa: E402
from paper_2106_14402_b200 import _lib as L  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ctx = P.Context(0)
A = P.fill_values(P.gen_rmat(scale, 16, 1, ctx=ctx), P.MinPlusI32, 3, ctx=ctx)
_, fl = P.estimate_flops(A, A, ctx=ctx)
bound = torch.clamp(fl, max=A.nrows).cpu().numpy()
c1 = int(np.searchsorted(np.cumsum(bound), bound.sum() / 4))
cap = int(bound[:c1].sum())
cp = torch.empty(c1 + 1, dtype=torch.int64, device="cuda")
rw = torch.empty(cap, dtype=torch.int32, device="cuda")
vv = torch.empty(cap, dtype=torch.int32, device="cuda")
w = L.CscView(A.nrows, c1, A.nnz, A.colptr.data_ptr(), A.rowids.data_ptr(), A.vals.data_ptr())
av = A.view()
lib = ctx.lib
dbg = lib.slapcu_debug_vcount
out = (C.c_ulonglong * 12)()
dbg(out, 1)
nz = C.c_int64()
ctx.check(lib.slapcu_spgemm_direct(ctx.h, C.byref(av), C.byref(w), P.MinPlusI32.id, 2, cap, cp.data_ptr(),
                                   rw.data_ptr(), vv.data_ptr(), C.byref(nz)), "direct")
dbg(out, 0)
print(f"columns [0,{c1}) nnz {nz.value} flops {int(fl[:c1].sum())}: entry visits {out[0]:.3e} nonempty runs {out[1]:.3e} "
      f"products {out[2]:.3e} batches(512) {out[3]:.3e}; rank-chunk products {out[4]:.3e} dense-chunk {out[5]:.3e}; "
      f"runs <=2 {out[8]:.3e} 3..31 {out[9]:.3e} >=32 {out[10]:.3e}")
