"""BJ c4 (BASELINE.json configs[3]) study: the 256^3 box-constrained problem (0 <= x <= 1) solved by
UPN and GPBB at (tau, alpha) in {1e-2, 1e-5} x {0.003, 0.03} to 20,000 iterations (SURVEY §8(d) c4
row), with the gradient-map history sampled so that iterations and time to each eps in
{1e-4, 1e-5, 1e-6} can be read off, plus hi = +inf controls that isolate the box.

usage: python scripts/c4_study.py [--grid 256] [--max-iters 20000] [--eps 1e-6] [--controls]
                                  [--only upn|gpbb] [--out PATH]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import harness
from paper_1105_4002_b200 import tvreg

MARKS = (1e-3, 1e-4, 1e-5, 1e-6, 1e-7)


def crossings(hist, seconds, iters):
    """First iteration (and the proportional time) at which gmap_rel <= each mark."""
    out = {}
    for m in MARKS:
        it = next((h["iter"] for h in hist if h["gmap_rel"] <= m), None)
        out[f"{m:g}"] = None if it is None else dict(iter=it, seconds=seconds * it / max(iters, 1))
    return out


def run(P, w, solver, max_iters, eps, hist_cap):
    x = torch.zeros(w.N, device="cuda")
    try:
        r = getattr(P, f"solve_{solver}")(x, max_iters=max_iters, eps=eps, hist_cap=hist_cap)
    except tvreg.TVRError as e:
        return dict(solver=solver, error=str(e))
    hist = r.history
    samp = [dict(iter=h["iter"], f=h["f"], gmap_rel=h["gmap_rel"], L=h["L"], mu=h["mu"],
                 step=h["step"]) for h in hist if h["iter"] % 250 == 0 or h is hist[-1]]
    best = min((h["gmap_rel"] for h in hist), default=math.nan)
    return dict(solver=solver, converged=r.converged, iters=r.iters, n_f=r.n_f, n_grad=r.n_grad,
                seconds=r.seconds, ms_per_iter=1e3 * r.seconds / max(r.iters, 1), f=r.f,
                gmap_rel=r.gmap_rel, best_gmap_rel=best, solve_hbm_gbs=r.bytes / r.seconds / 1e9,
                crossings=crossings(hist, r.seconds, r.iters), history=samp)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--max-iters", type=int, default=20000)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--controls", action="store_true", help="also hi=+inf runs (alpha=0.003)")
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    t0 = time.time()
    over = {} if a.grid == 256 else dict(grid=(a.grid,) * 3, views=max(12, 90 * a.grid // 256),
                                          bins=int(363 * a.grid / 256) | 1)
    w = harness.preset("c4", **over)
    out = dict(workload=f"c4 {w.grid[0]}^3, box [0,1], REL eps {a.eps:g}, max_iters {a.max_iters}",
               gen_s=time.time() - t0, nnz=int(w.A.nnz), runs=[])
    solvers = [a.only] if a.only else ["upn", "gpbb"]
    cases = [(tau, alpha, 1.0) for tau in (1e-2, 1e-5) for alpha in (0.003, 0.03)]
    if a.controls:
        cases += [(tau, 0.003, math.inf) for tau in (1e-2, 1e-5)]
    for tau, alpha, hi in cases:
        P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, alpha, tau, 0.0, hi,
                          stream=torch.cuda.current_stream().cuda_stream)
        for solver in solvers:
            rec = dict(tau=tau, alpha=alpha, hi=hi if math.isfinite(hi) else "inf")
            rec.update(run(P, w, solver, a.max_iters, a.eps, a.max_iters + 2))
            out["runs"].append(rec)
            short = {k: v for k, v in rec.items() if k != "history"}
            print(json.dumps(short), flush=True)
            if a.out:
                json.dump(out, open(a.out, "w"), indent=1)
        P.close()


if __name__ == "__main__":
    main()
