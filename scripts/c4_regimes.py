"""BJ c4 (BASELINE.json configs[3]): the 256^3 problem with the box 0 <= x <= 1, UPN against GPBB
at two strong-convexity regimes (tau in {1e-2, 1e-5}) and alpha in {0.003, 0.03}, on one GPU
(the 8-GPU z-slab runs are not available to this build).  Reports iterations, time-to-eps and the
solve's algorithmic HBM GB/s.

usage: python scripts/c4_regimes.py [--eps 1e-5] [--max-iters 3000] [--grid 256] [--out PATH]
"""
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
    ap.add_argument("--eps", type=float, default=1e-5)
    ap.add_argument("--max-iters", type=int, default=3000)
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    t0 = time.time()
    over = {} if a.grid == 256 else dict(grid=(a.grid,) * 3, views=max(12, 90 * a.grid // 256),
                                          bins=int(363 * a.grid / 256) | 1)
    w = harness.preset("c4", **over)
    gen_s = time.time() - t0
    out = dict(workload=f"c4 {w.grid[0]}^3, box [0,1], REL eps {a.eps:g}", gen_s=gen_s,
               nnz=int(w.A.nnz), runs=[])
    for tau in (1e-2, 1e-5):
        for alpha in (0.003, 0.03):
            P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, alpha, tau, 0.0, 1.0,
                              stream=torch.cuda.current_stream().cuda_stream)
            for solver in ("upn", "gpbb"):
                x = torch.zeros(w.N, device="cuda")
                try:
                    r = getattr(P, f"solve_{solver}")(x, max_iters=a.max_iters, eps=a.eps)
                    rec = dict(tau=tau, alpha=alpha, solver=solver, converged=r.converged,
                               iters=r.iters, n_f=r.n_f, seconds=r.seconds, f=r.f,
                               gmap_rel=r.gmap_rel, solve_hbm_gbs=r.bytes / r.seconds / 1e9)
                except tvreg.TVRError as e:
                    rec = dict(tau=tau, alpha=alpha, solver=solver, error=str(e))
                out["runs"].append(rec)
                print(json.dumps(rec), flush=True)
            P.close()
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
