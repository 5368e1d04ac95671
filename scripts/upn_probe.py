"""UPN / GPBB solve timings at c2 with host and device control, and the per-kernel split of a
host-controlled UPN solve (A/B of solver-state changes with TVR_LIB_PATH)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = harness.preset(cfg)
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=torch.cuda.current_stream().cuda_stream)
out = {"lib": os.path.basename(tvreg.LIB_PATH)}
for solver in ("upn", "gpbb"):
    for mode in ("device", "host"):
        P.set_control(mode)
        x = torch.zeros(w.N, device="cuda")
        getattr(P, f"solve_{solver}")(x, max_iters=50, eps=1e-6)  # warm
        x = torch.zeros(w.N, device="cuda")
        r = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6)
        out[f"{solver}_{mode}"] = dict(iters=r.iters, seconds=round(r.seconds, 4),
                                       ms_per_iter=round(1e3 * r.seconds / r.iters, 4), n_f=r.n_f)
P.set_control("host")
P.profile(True)
x = torch.zeros(w.N, device="cuda")
r = P.solve_upn(x, max_iters=20000, eps=1e-6)
st = P.kernel_stats()
out["upn_host_kernels_us_per_iter"] = {k: round(1e3 * v["ms"] / r.iters, 1) for k, v in st.items() if v["launches"]}
out["upn_host_launches_per_iter"] = {k: round(v["launches"] / r.iters, 2) for k, v in st.items() if v["launches"]}
print(json.dumps(out), flush=True)
