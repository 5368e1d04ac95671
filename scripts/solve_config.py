"""Time-to-eps of GPBB / UPN on one preset through the C ABI (BJ configs[2]: c3 GPBB full solve).
usage: python scripts/solve_config.py [--config c3] [--eps 1e-6] [--max-iters 5000] [--out PATH]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--max-iters", type=int, default=5000)
    ap.add_argument("--solvers", default="gpbb,upn")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    t0 = time.time()
    w = harness.preset(a.config)
    gen_s = time.time() - t0
    P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                      stream=torch.cuda.current_stream().cuda_stream)
    out = dict(config=a.config, grid=list(w.grid), nnz=int(w.A.nnz), eps=a.eps, gen_s=gen_s, runs=[])
    for solver in a.solvers.split(","):
        x = torch.zeros(w.N, device="cuda")
        r = getattr(P, f"solve_{solver}")(x, max_iters=a.max_iters, eps=a.eps)
        rec = dict(solver=solver, converged=r.converged, iters=r.iters, n_f=r.n_f, n_grad=r.n_grad,
                   seconds=r.seconds, ms_per_iter=1e3 * r.seconds / max(1, r.iters), f=r.f,
                   gmap_rel=r.gmap_rel, solve_hbm_gbs=r.bytes / r.seconds / 1e9)
        out["runs"].append(rec)
        print(json.dumps(rec), flush=True)
    P.close()
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
