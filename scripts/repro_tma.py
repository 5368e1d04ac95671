"""Small repro for TMA SpMV configurations (used under compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import harness
from paper_1105_4002_b200 import tvreg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
w = harness.separable_workload("r", (n, n, 8), 24, int(1.41 * n) | 1, 4)
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
print("info", P.info.slab_staged_A, P.info.slab_staged_AT, flush=True)
x = torch.from_numpy(harness.random_x(w.N)).cuda()
r = torch.empty(w.A.n_rows, device="cuda")
print("fid", P.residual(x, r), flush=True)
wt = torch.empty(w.N, device="cuda")
P.apply_AT(r, wt)
torch.cuda.synchronize()
print("ok", float(wt.sum()))
