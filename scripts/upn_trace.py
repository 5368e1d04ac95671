"""UPN gradient-map trajectory on one preset (where the extended-precision evaluation switches on,
and what it costs): per-50-iteration samples of ||G||/||G_1(x_0)|| and the solve time.
usage: python scripts/upn_trace.py [config]   (TVR_EXT_EVAL=0: hi evaluation throughout)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = harness.preset(cfg)
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                  stream=torch.cuda.current_stream().cuda_stream)
x = torch.zeros(w.N, device="cuda")
r = P.solve_upn(x, max_iters=20000, eps=1e-6, hist_cap=20000)
h = r.history
print(json.dumps(dict(config=cfg, ext_eval=os.environ.get("TVR_EXT_EVAL", "1"), iters=r.iters,
                      n_f=r.n_f, n_grad=r.n_grad, seconds=r.seconds, f=r.f,
                      trace=[(e["iter"], e["gmap_rel"]) for e in h if e["iter"] % 50 == 0])))
