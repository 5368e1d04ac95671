"""Unprofiled time of a gradient evaluation (no per-kernel events between the launches, so
programmatic dependent launches overlap as in the bench's value region): scripts/step_time.py
<config> <steps> [reps]; also checks f and g against the first evaluation (determinism)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = harness.preset(cfg)
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=torch.cuda.current_stream().cuda_stream)
x = torch.from_numpy(harness.random_x(w.N)).cuda()
g = torch.empty(w.N, device="cuda")
f0, _ = P.objective_grad(x, g)
g0 = g.clone()
for _ in range(5):
    P.objective_grad(x, g)
out = []
same = True
for _ in range(reps):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        f, _ = P.objective_grad(x, g)
    e1.record()
    torch.cuda.synchronize()
    same = same and f == f0 and torch.equal(g, g0)
    out.append(round(1e3 * steps / e0.elapsed_time(e1), 1))
print(json.dumps(dict(config=cfg, env={k: v for k, v in os.environ.items() if k.startswith("TVR_")},
                      evals_per_s=out, bitwise_repeatable=same)))
