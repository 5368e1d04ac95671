"""Short driver for ncu: build one workload, run a few gradient evaluations through the C ABI."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import harness
from paper_1105_4002_b200 import tvreg

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--sliced", action="store_true", help="slice-shared operator (tvr_create_sliced)")
a = ap.parse_args()
w = harness.sliced_preset(a.config) if a.sliced else harness.preset(a.config)
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  sliced=a.sliced)
N = int(np.prod(w.grid))
x = torch.from_numpy(harness.random_x(N)).cuda()
g = torch.empty(N, device="cuda")
for _ in range(a.steps):
    f, _ = P.objective_grad(x, g)
torch.cuda.synchronize()
print("f", f, "staged", P.info.slab_staged_A, P.info.slab_staged_AT)
