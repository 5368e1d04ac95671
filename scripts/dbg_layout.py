import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import harness, oracle
from tests._helpers import SmallCSR
from tests.test_gpu_kernels import _row_length_zoo
from paper_1105_4002_b200 import tvreg
cfg = sys.argv[1]
rng = np.random.default_rng(21)
if cfg == "zoo":
    grid = (16, 16, 4); A = _row_length_zoo(16 * 16 * 4, 9)
    x = rng.integers(0, 9, A.n_cols).astype(np.float32); b = rng.integers(0, 9, A.n_rows).astype(np.float32)
else:
    grid = (32, 24, 16); A = harness.siddon_tilted(32, 24, 16, 12, 16, 41, 10.0)
    x = harness.random_x(A.n_cols); b = rng.random(A.n_rows).astype(np.float32)
print("create", flush=True)
P = tvreg.Problem(A.row_ptr, A.col, A.val, b, grid, 0.01, 1e-4, 0.0, np.inf)
print("info", list(P.info.gather_layout_blocks), flush=True)
r = torch.empty(A.n_rows, device="cuda")
fid = P.residual(torch.from_numpy(x).cuda(), r)
torch.cuda.synchronize()
r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
rr = r.cpu().numpy().astype(np.float64)
print("rel", np.linalg.norm(rr - r_ora) / np.linalg.norm(r_ora), flush=True)
