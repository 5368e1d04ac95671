"""Per-CTA durations of the sliced-ELL passes (TVR_SELL_PROF=1 diagnostic): are the slow CTAs the
same ones launch after launch (work-model error / SM position), or noise?
scripts/sell_prof.py <config> <launches>  -- parses the library's SELLPROF stderr lines."""
import json
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import harness
    from paper_1105_4002_b200 import tvreg
    cfg, n = sys.argv[2], int(sys.argv[3])
    w = harness.preset(cfg)
    P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
    x = torch.from_numpy(harness.random_x(w.N)).cuda()
    g = torch.empty(w.N, device="cuda")
    for _ in range(n):
        P.objective_grad(x, g)
    sys.exit(0)

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = sys.argv[2] if len(sys.argv) > 2 else "8"
env = dict(os.environ, TVR_SELL_PROF="1", TVR_PDL="0")
r = subprocess.run([sys.executable, __file__, "--child", cfg, n], env=env, capture_output=True, text=True)
runs = {"A": [], "AT": []}
for line in r.stderr.splitlines():
    if not line.startswith("SELLPROF"):
        continue
    head, body = line.split(":", 1)
    kind = head.split()[1]
    span = int(head.split()[-1])
    t = np.array([[int(v) for v in e.split(",")] for e in body.split()])
    runs[kind].append((span, t))
out = {}
for kind, rs in runs.items():
    rs = rs[2:]  # warm-up
    if not rs:
        continue
    med = np.median([s for s, _ in rs])
    rs = [(s, t) for s, t in rs if s < 1.15 * med]  # drop launches hit by a clock ramp / hiccup
    dur = np.array([t[:, 1] - t[:, 0] for _, t in rs], float)  # launches x CTAs
    end = np.array([t[:, 1] for _, t in rs], float)
    start = np.array([t[:, 0] for _, t in rs], float)
    sm = np.array([t[:, 2] for _, t in rs])
    mean = dur.mean(0)
    cc = np.corrcoef(dur)
    out[kind] = dict(
        launches=len(rs), ctas=dur.shape[1],
        span_us=[round(s / 1e3, 1) for s, _ in rs],
        start_max_us=round(start.max(1).mean() / 1e3, 2),
        dur_mean_us=round(dur.mean() / 1e3, 1), dur_min_us=round(dur.min(1).mean() / 1e3, 1),
        dur_max_us=round(dur.max(1).mean() / 1e3, 1),
        end_spread_us=round((end.max(1) - end.min(1)).mean() / 1e3, 1),
        launch_to_launch_corr=round(float((cc.sum() - len(rs)) / (len(rs) * (len(rs) - 1))), 3),
        smid_stable=bool((sm == sm[0]).all()),
        mean_dur_rel_spread=round(float((mean.max() - mean.min()) / mean.mean()), 4),
        slowest_ctas=[int(i) for i in np.argsort(-mean)[:8]],
        fastest_ctas=[int(i) for i in np.argsort(mean)[:8]],
        mean_dur_by_cta_us=[round(v / 1e3, 1) for v in mean],
        sm_of_cta=[int(v) for v in sm[0]],
    )
print(json.dumps(out))
