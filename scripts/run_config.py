"""Time a few gradient evaluations of a preset (c2/c3/c5) through the C ABI and print per-kernel
CUDA-event stats and the create-time breakdown (for large-workload checks on the GPU box)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import harness
from paper_1105_4002_b200 import tvreg

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t0 = time.time()
w = harness.preset(cfg)
t1 = time.time()
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
t2 = time.time()
x = torch.from_numpy(harness.random_x(w.N)).cuda()
g = torch.empty(w.N, device="cuda")
for _ in range(3):
    P.objective_grad(x, g)
P.profile(True)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(steps):
    f, _ = P.objective_grad(x, g)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
st = P.kernel_stats()
out = dict(config=cfg, nnz=w.A.nnz, m=w.A.n_rows, N=w.N, gen_s=t1 - t0, create_s=t2 - t1, ms_per_eval=ms,
           evals_per_s=1e3 / ms, staged=[P.info.slab_staged_A, P.info.slab_staged_AT],
           device_gb=P.info.device_bytes / 1e9, f=f)
for k, v in st.items():
    if v["launches"]:
        out[k] = dict(ms=v["ms"] / v["launches"], gbs=v["bytes"] / v["launches"] / (v["ms"] / v["launches"]) / 1e6)
print(json.dumps(out), flush=True)
