"""c5 (BJ configs[4], 256^3 tilted rays) A / A^T pass times and gradient evaluations per second
on one GPU, with the gather-layout statistics (A/B: TVR_SELL32_LAYOUTS=0).
usage: python scripts/c5_time.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t0 = time.time()
w = harness.preset("c5")
t1 = time.time()
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=torch.cuda.current_stream().cuda_stream)
t2 = time.time()
x = torch.from_numpy(harness.random_x(w.N)).cuda()
g = torch.empty(w.N, device="cuda")
for _ in range(3):
    P.objective_grad(x, g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    P.objective_grad(x, g)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
P.profile(True)
for _ in range(steps):
    P.objective_grad(x, g)
torch.cuda.synchronize()
st = P.kernel_stats()
print(json.dumps(dict(layouts=os.environ.get("TVR_SELL32_LAYOUTS", "1"), gen_s=t1 - t0, create_s=t2 - t1,
                      evals_per_s=1e3 / ms, ms=ms,
                      layout_blocks=list(P.get_info().gather_layout_blocks),
                      kernels={k: round(v["ms"] / v["launches"], 4) for k, v in st.items() if v["launches"]})))
