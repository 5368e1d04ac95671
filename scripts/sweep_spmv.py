"""Tuning sweep of the SpMV launch parameters (env overrides read by tvr_create)."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = harness.preset(cfg)
x = torch.from_numpy(harness.random_x(w.N)).cuda()
r = torch.empty(w.A.n_rows, device="cuda")
wt = torch.empty(w.N, device="cuda")
bytesA = 8 * w.A.nnz + 8 * (w.A.n_rows + 1) + 4 * w.N + 8 * w.A.n_rows
bytesT = 8 * w.A.nnz + 8 * (w.N + 1) + 4 * w.A.n_rows + 4 * w.N
grid = json.loads(os.environ.get("SWEEP", '{"TVR_LPR_A":[8,16,32],"TVR_LPR_AT":[8,16,32],"TVR_SPMV_BLOCK":[256,512]}'))
keys = list(grid)
for vals in itertools.product(*[grid[k] for k in keys]):
    for k, v in zip(keys, vals):
        os.environ[k] = str(v)
    P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                      stream=torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        P.residual(x, r)
        P.apply_AT(r, wt)
    P.profile(True)
    for _ in range(30):
        P.residual(x, r)
        P.apply_AT(r, wt)
    st = P.kernel_stats()
    a = st["spmv_A"]["ms"] / st["spmv_A"]["launches"]
    t = st["spmv_AT"]["ms"] / st["spmv_AT"]["launches"]
    print(json.dumps(dict(zip(keys, vals)) | dict(A_ms=round(a, 4), A_gbs=round(bytesA / a / 1e6, 1),
                                                   AT_ms=round(t, 4), AT_gbs=round(bytesT / t / 1e6, 1),
                                                   staged=[P.info.slab_staged_A, P.info.slab_staged_AT])), flush=True)
    P.close()
