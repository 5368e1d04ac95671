import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch, harness
from paper_1105_4002_b200 import tvreg
w = harness.preset("c2")
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi, stream=torch.cuda.current_stream().cuda_stream)
x = harness.random_x(w.N)
xh = torch.from_numpy(x.copy()).pin_memory(); gh = torch.empty(w.N, dtype=torch.float32).pin_memory()
for _ in range(5): P.objective_grad_host(xh.numpy(), gh.numpy())
os.environ["TVR_E2E_TRACE"] = "1"
for _ in range(3):
    t = time.perf_counter(); P.objective_grad_host(xh.numpy(), gh.numpy()); print("wall", round((time.perf_counter() - t) * 1e6), flush=True)
