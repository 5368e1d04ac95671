"""e2e (tvr_objective_grad_host, pinned host x in / g out) at the driver's --steps 20 against long
runs: per-call wall times, so that a slow first call or a clock ramp shows up."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import harness
from paper_1105_4002_b200 import tvreg

w = harness.preset("c2")
stream = torch.cuda.current_stream()
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=stream.cuda_stream)
x_h = harness.random_x(w.N)
x = torch.from_numpy(x_h).cuda()
g = torch.empty(w.N, device="cuda")
for _ in range(5):
    P.objective_grad(x, g)
xh = torch.from_numpy(x_h.copy()).pin_memory()
gh = torch.empty(w.N, dtype=torch.float32).pin_memory()
out = {}
for rep, steps in enumerate([20, 20, 20, 200, 20]):
    if rep == 0:
        for _ in range(2):
            P.objective_grad_host(xh.numpy(), gh.numpy())
    torch.cuda.synchronize()
    ts = []
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(steps):
        a = time.perf_counter()
        P.objective_grad_host(xh.numpy(), gh.numpy())
        ts.append(time.perf_counter() - a)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ts = np.array(ts) * 1e6
    out[f"rep{rep}_{steps}"] = dict(evals_per_s=steps / wall, ev_ms=e0.elapsed_time(e1),
                                    wall_ms=wall * 1e3, us_first5=ts[:5].round(1).tolist(),
                                    us_median=float(np.median(ts)), us_max=float(ts.max()))
    print(json.dumps({f"rep{rep}_{steps}": out[f"rep{rep}_{steps}"]}), flush=True)
# device-resident for comparison
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    P.objective_grad(x, g)
torch.cuda.synchronize()
print(json.dumps(dict(device_20=20 / (time.perf_counter() - t0))))
