"""Driver for ncu: a few tvr_objective_grad_host calls (pinned buffers, chunked pipeline) on c2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

w = harness.preset("c2")
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
x = harness.random_x(w.N)
xh = torch.from_numpy(x.copy()).pin_memory()
gh = torch.empty(w.N, dtype=torch.float32).pin_memory()
for _ in range(3):
    P.objective_grad_host(xh.numpy(), gh.numpy())
xd = torch.from_numpy(x).cuda()
gd = torch.empty_like(xd)
P.objective_grad(xd, gd)
torch.cuda.synchronize()
print("ok")
