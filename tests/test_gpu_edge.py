"""Degenerate inputs through the C ABI (SURVEY §8(c).4 edge cases): an all-empty matrix, a matrix
with no rows, a one-voxel volume, a single slice, and a solve that starts at its minimiser."""
import math

import numpy as np
import pytest

import harness
import oracle
from tests._helpers import SmallCSR, random_csr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tvreg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1105_4002_b200 import tvreg as T
    return T


def _check_fg(T, A, b, grid, alpha=0.05, tau=1e-2, seed=0):
    P = T.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau)
    x = np.random.default_rng(seed).random(A.n_cols).astype(np.float32)
    g = torch.empty(A.n_cols, device="cuda")
    f, _ = P.objective_grad(torch.from_numpy(x).cuda(), g)
    Po = oracle.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau)
    fo, go = Po.fg(x.astype(np.float64))
    assert abs(f - fo) <= 1e-10 * max(1.0, abs(fo))
    gn = np.linalg.norm(go)
    assert np.linalg.norm(g.cpu().numpy() - go) <= 1e-6 * max(gn, 1e-30) + 1e-12
    return P


def test_all_rows_empty(tvreg):
    grid = (3, 2, 2)
    A = SmallCSR(np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32), 12)
    b = np.arange(5, dtype=np.float32)
    P = _check_fg(tvreg, A, b, grid)
    r = torch.empty(5, device="cuda")
    fid = P.residual(torch.zeros(12, device="cuda"), r)
    assert torch.equal(r.cpu(), -torch.from_numpy(b)) and fid == 0.5 * float(b @ b)


def test_no_rows(tvreg):
    grid = (4, 3, 2)
    A = SmallCSR(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32), 24)
    _check_fg(tvreg, A, np.zeros(0, np.float32), grid)


def test_one_voxel_volume(tvreg):
    A = SmallCSR([0, 1, 1, 2], [0, 0], [2.0, 0.5], 1)
    _check_fg(tvreg, A, np.array([1.0, 2.0, 3.0], np.float32), (1, 1, 1))


def test_single_slice_volume(tvreg):
    w = harness.separable_workload("s", (23, 19, 1), 7, 31, 2)
    _check_fg(tvreg, w.A, w.b, w.grid)


def test_ragged_random_volume_shapes(tvreg):
    for grid, seed in (((1, 7, 3), 1), ((7, 1, 3), 2), ((5, 4, 1), 3)):
        N = grid[0] * grid[1] * grid[2]
        A = random_csr(40, N, 0.3, seed=seed, empty_rows=5)
        b = np.random.default_rng(seed).random(40).astype(np.float32)
        _check_fg(tvreg, A, b, grid, seed=seed)


@pytest.mark.parametrize("solver", ["gpbb", "upn", "gp"])
def test_solve_from_the_minimiser(tvreg, solver):
    """b = A x with x constant (TV = 0) and alpha > 0: x is the minimiser over x >= 0, the
    gradient map at x_0 is zero and every solver stops at once with x unchanged."""
    w = harness.separable_workload("m", (12, 10, 4), 6, 17, 2)
    xs = np.full(w.N, 0.5, np.float32)
    b = oracle.matvec(w.A.row_ptr, w.A.col, w.A.val, xs.astype(np.float64)).astype(np.float32)
    P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, b, w.grid, 0.01, 1e-3)
    x = torch.from_numpy(xs.copy()).cuda()
    res = getattr(P, f"solve_{solver}")(x, max_iters=50, eps=1e-6,
                                        stop_mode=tvreg.TVR_STOP_ABS_PER_N)
    assert res.converged
    assert np.allclose(x.cpu().numpy(), xs, atol=1e-6)
