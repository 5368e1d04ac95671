"""Stencil timing (a4): tvr_objective_grad on a volume with a 3-row system matrix, so the TV
kernel (W1 | G instantiation) dominates; per-kernel CUDA-event times from the library's profile.
usage: python scripts/tv_time.py [nx ny nz] [iters]   (TVR_TV_ROW=0: the 32x8 xy-tile kernel)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import harness  # noqa: E402
from paper_1105_4002_b200 import tvreg  # noqa: E402
from tests._helpers import random_csr  # noqa: E402


def main():
    a = sys.argv[1:]
    shapes = [(128, 128, 128), (256, 256, 256)] if len(a) < 3 else [tuple(int(v) for v in a[:3])]
    iters = int(a[3]) if len(a) > 3 else 200
    for grid in shapes:
        N = grid[0] * grid[1] * grid[2]
        A = random_csr(3, N, 1e-6, seed=1)
        P = tvreg.Problem(A.row_ptr, A.col, A.val, np.zeros(3, np.float32), grid, 0.01, 1e-4, 0.0,
                          np.inf)
        x = torch.from_numpy(harness.phantom(*grid, 10)).cuda() + 0.01 * torch.rand(N, device="cuda")
        g = torch.empty(N, device="cuda")
        for _ in range(20):
            P.objective_grad(x, g)
        P.profile(True)
        for _ in range(iters):
            P.objective_grad(x, g)
        torch.cuda.synchronize()
        st = P.kernel_stats()
        P.profile(False)
        tv = st["tv_grad"]
        us = tv["ms"] / tv["launches"] * 1e3
        print(f"{grid} tv_grad {us:.2f} us  {25165824 * N / 2**21 / (us * 1e3):.0f} GB/s  "
              f"(row kernel {'off' if os.environ.get('TVR_TV_ROW') == '0' else 'on'}, "
              f"ZC {os.environ.get('TVR_TV_ZC', 'auto')})", flush=True)
        P.close()


if __name__ == "__main__":
    main()
