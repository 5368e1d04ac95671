"""Time-to-eps of the solvers under host and device control:
python scripts/solver_ab.py [configs...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

for cfg in (sys.argv[1:] or ["c1", "c2"]):
    w = harness.preset(cfg)
    P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                      stream=torch.cuda.current_stream().cuda_stream)
    for solver in ("gpbb", "upn", "gp"):
        for mode in ("host", "device", "host", "device"):
            P.set_control(mode)
            x = torch.zeros(w.N, device="cuda")
            r = getattr(P, f"solve_{solver}")(x, max_iters=2000 if solver == "gp" else 20000, eps=1e-6)
            print(f"{cfg:6s} {solver:4s} {mode:6s} iters {r.iters:5d} {r.seconds * 1e3:9.2f} ms "
                  f"{1e3 * r.seconds / max(1, r.iters):7.4f} ms/it f {r.f:.12g}", flush=True)
    P.close()
