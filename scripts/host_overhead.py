"""Per-call host overhead of tvr_objective_grad at c2: device time per step with and without
per-kernel event profiling, and host wall time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import harness
from paper_1105_4002_b200 import tvreg
w = harness.preset(sys.argv[1] if len(sys.argv) > 1 else "c2")
st = torch.cuda.current_stream()
P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi, stream=st.cuda_stream)
x = torch.from_numpy(harness.random_x(w.N)).cuda(); g = torch.empty(w.N, device="cuda")
for prof in (False, True, False):
    P.profile(prof)
    for _ in range(5): P.objective_grad(x, g)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record(st)
    for _ in range(200): P.objective_grad(x, g)
    e1.record(st); torch.cuda.synchronize(); t1 = time.perf_counter()
    ks = P.kernel_stats() if prof else {}
    ksum = sum(v["ms"] for v in ks.values()) / 200 if ks else float("nan")
    print(f"prof={prof} device {e0.elapsed_time(e1)/200*1e3:.1f} us/step, host {1e6*(t1-t0)/200:.1f} us/step, kernels {ksum*1e3:.1f} us")
