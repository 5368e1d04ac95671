"""e2e probe: tvr_objective_grad_host on c2 with pinned buffers (the bench's e2e) against the
device-resident evaluation and raw PCIe copy rates of the same 8 MB vectors."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import harness
from paper_1105_4002_b200 import tvreg

w = harness.preset(sys.argv[1] if len(sys.argv) > 1 else "c2")
st = torch.cuda.current_stream()
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=st.cuda_stream)
x = harness.random_x(w.N)
xd = torch.from_numpy(x).cuda()
gd = torch.empty_like(xd)
xh = torch.from_numpy(x.copy()).pin_memory()
gh = torch.empty(w.N, dtype=torch.float32).pin_memory()


def timed(fn, n=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


dev_us = timed(lambda: P.objective_grad(xd, gd))
e2e_us = timed(lambda: P.objective_grad_host(xh.numpy(), gh.numpy()))
h2d = timed(lambda: xd.copy_(xh, non_blocking=True))
d2h = timed(lambda: gh.copy_(gd, non_blocking=True))
s2 = torch.cuda.Stream()


def both():
    xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        gh.copy_(gd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


bi = timed(both)
print(f"{os.environ.get('TAG', '')} device {dev_us:.0f} us  e2e {e2e_us:.0f} us ({1e6 / e2e_us:.0f}/s)  "
      f"h2d {h2d:.0f} us  d2h {d2h:.0f} us  both {bi:.0f} us")
