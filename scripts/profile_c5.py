"""Driver for ncu on c5 (non-separable, int32 global gathers): a few gradient evaluations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

w = harness.preset("c5")
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
x = torch.from_numpy(harness.random_x(w.N)).cuda()
g = torch.empty(w.N, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    P.objective_grad(x, g)
torch.cuda.synchronize()
print("ok")
