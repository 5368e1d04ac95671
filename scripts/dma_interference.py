"""Does a concurrent PCIe copy slow the SpMV passes?  Times tvr_objective_grad on c2 alone and
while another stream keeps H2D / D2H copies of pinned buffers running."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

w = harness.preset("c2")
st = torch.cuda.current_stream()
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=st.cuda_stream)
x = torch.from_numpy(harness.random_x(w.N)).cuda()
g = torch.empty_like(x)
hb = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
db = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
cs = torch.cuda.Stream()


def run(n=100, mode=None):
    torch.cuda.synchronize()
    if mode:
        with torch.cuda.stream(cs):
            for _ in range(40):
                if mode in ("h2d", "both"):
                    db.copy_(hb, non_blocking=True)
                if mode in ("d2h", "both"):
                    hb.copy_(db, non_blocking=True)
    P.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        P.objective_grad(x, g)
    e1.record(st)
    torch.cuda.synchronize()
    ks = P.kernel_stats()
    P.profile(False)
    return e0.elapsed_time(e1) / n * 1e3, {k: round(v["ms"] / v["launches"] * 1e3, 1) for k, v in ks.items() if v["launches"]}


for _ in range(3):
    P.objective_grad(x, g)
for mode in (None, "h2d", "d2h", "both", None):
    print(mode, run(30, mode))
