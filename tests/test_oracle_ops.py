"""Pins of the oracle's operators against mathematics, not against itself
(SURVEY.md §8(c).3): exact dyadic adjointness, dense brute force, closed forms,
invariants, finite differences.  CPU only."""
import math
import os

import numpy as np
import pytest

import oracle
from tests._helpers import dense_D, random_csr

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ A, A^T
def test_matvec_rmatvec_match_dense_bruteforce():
    A = random_csr(37, 4 * 4 * 4, 0.2, seed=1, empty_rows=3)
    M = A.dense()
    x = np.random.default_rng(2).standard_normal(64)
    y = np.random.default_rng(3).standard_normal(37)
    assert np.allclose(oracle.matvec(A.row_ptr, A.col, A.val, x), M @ x, rtol=1e-14, atol=1e-14)
    assert np.allclose(oracle.rmatvec(A.row_ptr, A.col, A.val, y, 64), M.T @ y, rtol=1e-14, atol=1e-14)


def test_exact_dyadic_adjointness():
    """Values k/1024 and integer x, y in [0, 8]: every partial sum is exact, so
    <Ax, y> == <x, A^T y> bitwise and A x equals exact integer arithmetic (App. A.4)."""
    A = random_csr(200, 300, 0.1, seed=5, dyadic=True, empty_rows=7)
    rng = np.random.default_rng(6)
    x = rng.integers(0, 9, 300).astype(np.float64)
    y = rng.integers(0, 9, 200).astype(np.float64)
    Ax = oracle.matvec(A.row_ptr, A.col, A.val, x)
    ATy = oracle.rmatvec(A.row_ptr, A.col, A.val, y, 300)
    # exact integer reference in units of 1/1024
    kv = np.rint(A.val.astype(np.float64) * 1024).astype(np.int64)
    for i in range(200):
        s = sum(int(kv[k]) * int(x[A.col[k]]) for k in range(A.row_ptr[i], A.row_ptr[i + 1]))
        assert Ax[i] == s / 1024.0
    assert float(Ax @ y) == float(x @ ATy)


def test_adjointness_random_fp64(c1):
    A = c1.A
    rng = np.random.default_rng(11)
    for _ in range(20):
        x = rng.standard_normal(A.n_cols)
        y = rng.standard_normal(A.n_rows)
        Ax = oracle.matvec(A.row_ptr, A.col, A.val, x)
        ATy = oracle.rmatvec(A.row_ptr, A.col, A.val, y, A.n_cols)
        assert abs(Ax @ y - x @ ATy) <= 1e-12 * np.linalg.norm(Ax) * np.linalg.norm(y)


def test_transpose_is_canonical():
    """Compared with an independent construction (dict of lists, sorted by row) and
    with scipy's CSC conversion (a library routine)."""
    import scipy.sparse as sp
    A = random_csr(120, 90, 0.08, seed=9, empty_rows=5)
    rT, cT, vT = oracle.transpose(A.row_ptr, A.col, A.val, 90)
    buckets = {j: [] for j in range(90)}
    for i in range(A.n_rows):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            buckets[int(A.col[k])].append((i, A.val[k]))
    ptr = [0]
    for j in range(90):
        ptr.append(ptr[-1] + len(buckets[j]))
    assert np.array_equal(rT, np.asarray(ptr, np.int64))
    for j in range(90):
        got = list(zip(cT[rT[j]:rT[j + 1]].tolist(), vT[rT[j]:rT[j + 1]].tolist()))
        exp = sorted((i, float(v)) for i, v in buckets[j])
        assert got == exp
    S = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(120, 90)).tocsc()
    S.sort_indices()
    assert np.array_equal(S.indptr, rT) and np.array_equal(S.indices, cT)
    assert np.array_equal(S.data.view(np.uint32), vT.view(np.uint32))


@pytest.mark.parametrize("j0,j1", [(0, 90), (0, 1), (17, 61), (89, 90), (30, 30)])
def test_transpose_range_is_a_slice_of_the_canonical_transpose(j0, j1):
    """transpose_range (the column-range form used for c5's > 2^31-entry check) against scipy's
    CSC conversion (a library routine): rowT in full, and exactly the entries of rows j0..j1-1."""
    import scipy.sparse as sp
    A = random_csr(120, 90, 0.08, seed=9, empty_rows=5)
    rT, cT, vT = oracle.transpose_range(A.row_ptr, A.col, A.val, 90, j0, j1)
    S = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(120, 90)).tocsc()
    S.sort_indices()
    assert np.array_equal(S.indptr, rT)
    s, e = S.indptr[j0], S.indptr[j1]
    assert np.array_equal(S.indices[s:e], cT)
    assert np.array_equal(S.data[s:e].view(np.uint32), vT.view(np.uint32))


def test_transpose_product_equals_scatter(c1):
    A = c1.A
    rT, cT, vT = oracle.transpose(A.row_ptr, A.col, A.val, A.n_cols)
    y = np.random.default_rng(4).standard_normal(A.n_rows)
    a = oracle.matvec(rT, cT, vT, y)
    b = oracle.rmatvec(A.row_ptr, A.col, A.val, y, A.n_cols)
    assert np.allclose(a, b, rtol=1e-13, atol=1e-13)


# ----------------------------------------------------------------------- TV
def _golden_tv():
    rows = []
    for line in open(os.path.join(GOLDEN, "tv_closed_forms.txt")):
        if line.startswith("#") or not line.strip():
            continue
        rows.append([float(t) for t in line.split()])
    return rows


@pytest.mark.parametrize("row", _golden_tv())
def test_tv_closed_forms(row):
    nx, ny, nz, x0, x1, tau, TV, g0, g1 = row
    grid = (int(nx), int(ny), int(nz))
    val, g = oracle.tv(grid, [x0, x1], tau, want_grad=tau > 0)
    assert val == pytest.approx(TV, abs=1e-15)
    if tau > 0:
        assert g[0] == pytest.approx(g0, abs=1e-15) and g[1] == pytest.approx(g1, abs=1e-15)


def test_tv_constant_volume_is_zero():
    for c in (0.0, 0.7, -3.25):
        val, g = oracle.tv((5, 4, 3), np.full(60, c), 1e-3)
        assert val == 0.0 and np.all(g == 0.0)


def test_tv_matches_dense_D_bruteforce():
    """TV_tau(x) = sum_j h(||D_j x||), grad = D^T (Dx / max(t, tau)) with the
    explicitly assembled 3N x N difference matrix on a 4^3 grid."""
    grid = (4, 4, 4)
    D = dense_D(*grid)
    x = np.random.default_rng(1).standard_normal(64)
    for tau in (0.5, 1e-2):
        Dx = (D @ x).reshape(-1, 3)
        t = np.sqrt((Dx ** 2).sum(1))
        h = np.where(t >= tau, t - tau / 2, t * t / (2 * tau))
        u = Dx / np.maximum(t, tau)[:, None]
        val, g = oracle.tv(grid, x, tau)
        assert val == pytest.approx(h.sum(), rel=1e-14)
        assert np.allclose(g, D.T @ u.ravel(), rtol=1e-13, atol=1e-13)


def test_tv_translation_invariance_and_nonneg():
    x = np.random.default_rng(2).standard_normal(6 * 5 * 4)
    a, _ = oracle.tv((6, 5, 4), x, 1e-2, False)
    b, _ = oracle.tv((6, 5, 4), x + 3.0, 1e-2, False)
    assert a >= 0 and a == pytest.approx(b, rel=1e-12)


@pytest.mark.parametrize("tau", [1e-1, 1e-2, 1e-4])
def test_tv_huber_sandwich(tau):
    """0 <= TV(x) - TV_tau(x) <= N tau / 2 (h_tau(t) in [t - tau/2, t])."""
    grid = (8, 8, 8)
    x = np.random.default_rng(3).random(512)
    tv0, _ = oracle.tv(grid, x, 0.0, False)
    tvt, _ = oracle.tv(grid, x, tau, False)
    assert 0.0 <= tv0 - tvt <= 512 * tau / 2 + 1e-12


@pytest.mark.parametrize("tau", [1e-1, 1e-2, 1e-3])
@pytest.mark.parametrize("grid", [(6, 6, 6), (7, 5, 8)])
def test_tv_gradient_central_differences(tau, grid):
    N = grid[0] * grid[1] * grid[2]
    rng = np.random.default_rng(4)
    x = rng.random(N)
    _, g = oracle.tv(grid, x, tau)
    h = 1e-6
    idx = rng.choice(N, 40, replace=False)
    fd = np.empty(40)
    for n, j in enumerate(idx):
        e = np.zeros(N)
        e[j] = h
        fd[n] = (oracle.tv(grid, x + e, tau, False)[0] - oracle.tv(grid, x - e, tau, False)[0]) / (2 * h)
    assert np.linalg.norm(fd - g[idx]) <= 1e-5 * np.linalg.norm(g[idx])


def test_tv_gradient_lipschitz_bound():
    """||grad TV_tau(x) - grad TV_tau(y)|| <= (12/tau)||x - y||."""
    rng = np.random.default_rng(5)
    tau = 1e-2
    for _ in range(10):
        x = rng.random(216)
        y = x + 1e-3 * rng.standard_normal(216)
        gx = oracle.tv((6, 6, 6), x, tau)[1]
        gy = oracle.tv((6, 6, 6), y, tau)[1]
        assert np.linalg.norm(gx - gy) <= 12.0 / tau * np.linalg.norm(x - y)


# ---------------------------------------------------------------- objective
def _small_problem(alpha=0.05, tau=1e-2, lo=0.0, hi=math.inf, seed=0, grid=(6, 6, 6)):
    N = grid[0] * grid[1] * grid[2]
    A = random_csr(150, N, 0.05, seed=seed)
    b = np.random.default_rng(seed + 1).random(150).astype(np.float32)
    return oracle.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau, lo, hi), A


def test_objective_gradient_central_differences():
    P, _ = _small_problem()
    rng = np.random.default_rng(7)
    x = rng.random(P.N)
    f, g = P.fg(x)
    h = 1e-6
    idx = rng.choice(P.N, 40, replace=False)
    fd = np.array([(P.f(x + h * np.eye(P.N)[j]) - P.f(x - h * np.eye(P.N)[j])) / (2 * h) for j in idx])
    assert np.linalg.norm(fd - g[idx]) <= 1e-5 * np.linalg.norm(g[idx])


def test_objective_alpha_zero_and_dense():
    P, A = _small_problem(alpha=0.0)
    M = A.dense()
    x = np.random.default_rng(8).random(P.N)
    f, g = P.fg(x)
    r = M @ x - P.b.astype(np.float64)
    assert f == pytest.approx(0.5 * r @ r, rel=1e-13)
    assert np.allclose(g, M.T @ r, rtol=1e-12, atol=1e-12)


def test_objective_zero_at_consistent_constant():
    """x = c 1 with b = A (c 1) gives phi = 0 and grad = 0."""
    from tests._helpers import random_csr as rc
    A = rc(80, 125, 0.1, seed=3, dyadic=True)
    c = 2.0
    b = (A.dense() @ np.full(125, c)).astype(np.float32)   # exact: dyadic * 2
    P = oracle.Problem(A.row_ptr, A.col, A.val, b, (5, 5, 5), 0.1, 1e-3)
    f, g = P.fg(np.full(125, c))
    assert f == 0.0 and np.all(g == 0.0)


def test_gradient_map_special_cases():
    P, _ = _small_problem(lo=0.0)
    x = np.full(P.N, 5.0)
    g = P.grad(x)
    nu = 10.0 * max(1.0, np.abs(g).max())
    # projection inactive (x - g/nu stays > 0): G_nu = grad f exactly
    assert np.allclose(P.gradient_map(x, nu, g), g, rtol=1e-12, atol=1e-12)
    # x = lo on a coordinate with grad f > 0: that component of G is 0
    x0 = np.zeros(P.N)
    g0 = P.grad(x0)
    G = P.gradient_map(x0, 1.0, g0)
    assert np.all(G[g0 > 0] == 0.0)
