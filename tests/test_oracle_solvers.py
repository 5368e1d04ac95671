"""Pins of the oracle's solvers (GPBB Alg. 1, BT Alg. 2, mu_k Eq.(9), UPN Alg. 3,
stopping rule Eq.(10)/P:228) against closed forms, invariants and an independent
library optimiser.  CPU only."""
import math

import numpy as np
import pytest

import harness
import oracle
from tests._helpers import dense_D, diag_csr, identity_csr, random_csr


def _prob(A, b, grid, alpha, tau, lo=0.0, hi=math.inf):
    return oracle.Problem(A.row_ptr, A.col, A.val, np.asarray(b, np.float32), grid, alpha, tau, lo, hi)


# ------------------------------------------------------------ special cases
@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_identity_alpha_zero_minimiser_is_projection_of_b(solver):
    """A = I, alpha = 0: argmin_{x in Q} 1/2||x - b||^2 = P_Q(b)."""
    n = 64
    b = np.random.default_rng(1).uniform(-1, 1, n).astype(np.float32)
    P = _prob(identity_csr(n), b, (4, 4, 4), 0.0, 1e-3, lo=0.0, hi=0.5)
    res = getattr(oracle, solver)(P, np.zeros(n), eps=1e-9, max_iters=5000)
    assert res.converged
    assert np.allclose(res.x, np.clip(b.astype(np.float64), 0.0, 0.5), atol=1e-8)


@pytest.mark.parametrize("b,alpha,tau", [((1.0, 2.0), 0.1, 0.01),      # linear branch
                                         ((2.0, 1.0), 0.3, 0.05),
                                         ((1.0, 1.0078125), 0.1, 0.01)])  # quadratic branch
@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_two_voxel_closed_form(b, alpha, tau, solver):
    """A = I on a 2x1x1 grid: with s = x0 + x1, d = x1 - x0, delta = b1 - b0,
    phi = (s - s_b)^2/4 + (d - delta)^2/4 + alpha h_tau(|d|), so s* = b0 + b1 and
    d* = delta - 2 alpha sign(delta) if |delta| >= 2 alpha + tau else delta/(1 + 2 alpha/tau)."""
    b0, b1 = b
    delta = b1 - b0
    if abs(delta) >= 2 * alpha + tau:
        d = delta - 2 * alpha * math.copysign(1.0, delta)
    else:
        d = delta / (1 + 2 * alpha / tau)
    s = b0 + b1
    exp = np.array([(s - d) / 2, (s + d) / 2])
    P = _prob(identity_csr(2), b, (2, 1, 1), alpha, tau, lo=-math.inf)
    res = getattr(oracle, solver)(P, np.zeros(2), eps=1e-10, max_iters=20000)
    assert res.converged
    assert np.allclose(res.x, exp, atol=1e-8)
    if b == (1.0, 2.0):
        assert np.allclose(res.x, [1.1, 1.9], atol=1e-8)   # SURVEY App. A.4 example


# --------------------------------------------------------------------- GPBB
def test_gpbb_bb_step_closed_forms():
    """f = 1/2||x||^2 gives theta_k = 1; Hessian 2I gives theta_k = 1/2."""
    n = 50
    x0 = np.random.default_rng(2).uniform(0.5, 1.5, n)
    P = _prob(identity_csr(n), np.zeros(n), (5, 5, 2), 0.0, 1e-3, lo=-math.inf)
    res = oracle.gpbb(P, x0, eps=1e-9, max_iters=100)
    steps = [h["step"] for h in res.history[1:]]
    assert len(steps) >= 2 and np.allclose(steps, 1.0, rtol=1e-12)
    s2 = np.float32(math.sqrt(2.0))
    P2 = _prob(diag_csr(np.full(n, s2)), np.zeros(n), (5, 5, 2), 0.0, 1e-3, lo=-math.inf)
    res2 = oracle.gpbb(P2, x0, eps=1e-9, max_iters=100)
    steps2 = [h["step"] for h in res2.history[1:]]
    assert len(steps2) >= 2 and np.allclose(steps2, 1.0 / float(s2) ** 2, rtol=1e-12)
    assert abs(steps2[0] - 0.5) < 1e-6


def test_gpbb_armijo_replay_and_counts(c1):
    """Every accepted step satisfies f(x_bar) < f_hat - sigma g^T(x - x_bar)."""
    A = c1.A
    P = _prob(A, c1.b, c1.grid, c1.alpha, 1e-2)
    res = oracle.gpbb(P, np.zeros(c1.N), eps=1e-4, max_iters=3000)
    assert res.converged
    for h in res.history[:-1]:
        assert h["f_next"] < h["armijo_rhs"]
        assert h["trials"] >= 1
        assert h["beta"] == pytest.approx(0.95 ** (2 ** (h["trials"] - 1)), rel=1e-12)
    # f_hat memory is K+1 = 3 accepted values: nonmonotone but bounded by the running max
    fs = [h["f"] for h in res.history]
    for k in range(3, len(fs)):
        assert fs[k] < max(fs[k - 3:k])


# ----------------------------------------------------------------------- BT
@pytest.mark.parametrize("L_bar", [1.0, 0.37, 9.0])
def test_bt_closed_form_on_isotropic_quadratic(L_bar):
    """Hessian L0 I: L~ = L_bar if L_bar >= L0 else L_bar rho^ceil(log_rho(L0/L_bar))."""
    L0, rho, n = 4.0, 1.3, 40
    P = _prob(diag_csr(np.full(n, 2.0)), np.zeros(n), (5, 4, 2), 0.0, 1e-3, lo=-math.inf)
    y = np.random.default_rng(3).standard_normal(n)
    f_y, g_y = P.fg(y)
    x, fx, L, trials = oracle.backtrack(P, y, f_y, g_y, L_bar, rho)
    exp = L_bar if L_bar >= L0 else L_bar * rho ** math.ceil(math.log(L0 / L_bar, rho))
    assert L == pytest.approx(exp, rel=1e-12)
    assert trials == (1 if L_bar >= L0 else math.ceil(math.log(L0 / L_bar, rho)) + 1)


# --------------------------------------------------------------------- mu_k
def test_mu_estimate_exact_and_bracketed():
    """f = 1/2 mu0 ||x||^2 gives M = mu0; eigenvalues in [mu0, L0] bracket M."""
    n = 30
    rng = np.random.default_rng(4)
    P = _prob(diag_csr(np.full(n, 2.0)), np.zeros(n), (5, 3, 2), 0.0, 1e-3, lo=-math.inf)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    fx = P.f(x)
    fy, gy = P.fg(y)
    assert oracle.mu_estimate(1e9, fx, fy, gy, x, y) == pytest.approx(4.0, rel=1e-12)
    assert oracle.mu_estimate(1.5, fx, fy, gy, x, y) == 1.5          # min with mu_{k-1}
    assert oracle.mu_estimate(7.0, fx, fy, gy, y, y) == 7.0          # x = y: keep mu_{k-1}
    d = rng.uniform(1.0, 3.0, n).astype(np.float32)
    P2 = _prob(diag_csr(d), np.zeros(n), (5, 3, 2), 0.0, 1e-3, lo=-math.inf)
    for _ in range(20):
        x, y = rng.standard_normal(n), rng.standard_normal(n)
        fy, gy = P2.fg(y)
        M = oracle.mu_estimate(1e9, P2.f(x), fy, gy, x, y)
        assert d.min() ** 2 * (1 - 1e-9) <= M <= d.max() ** 2 * (1 + 1e-9)


# ---------------------------------------------------------------------- UPN
def test_theta_root_fixed_point_and_range():
    rng = np.random.default_rng(5)
    for _ in range(20000):
        tk = rng.uniform(1e-6, 1.0)
        q = rng.uniform(0.0, 1.0) ** 3
        t = oracle.theta_root(tk, q)
        assert 0.0 < t <= 1.0
        assert abs(t * t - ((1 - t) * tk * tk + q * t)) <= 1e-14 * max(1.0, tk * tk)
    for q in (1e-6, 1e-3, 0.25, 1.0):
        assert oracle.theta_root(math.sqrt(q), q) == pytest.approx(math.sqrt(q), rel=1e-14)


def test_upn_invariants_small_ct():
    """mu_k nonincreasing, L_k nondecreasing, theta in (0, 1]."""
    A = harness.siddon_separable(12, 12, 6, 8, 17)
    xt = harness.phantom(12, 12, 6, 4)
    b = harness.simulate_data(A, xt)
    P = _prob(A, b, (12, 12, 6), 0.01, 1e-3)
    res = oracle.upn(P, np.zeros(P.N), eps=1e-6, max_iters=5000)
    assert res.converged
    mus = [h["mu"] for h in res.history]
    Ls = [h["L"] for h in res.history]
    th = [h["theta"] for h in res.history]
    assert all(a >= b for a, b in zip(mus, mus[1:]))
    assert all(a <= b for a, b in zip(Ls, Ls[1:]))
    assert all(0.0 < t <= 1.0 for t in th)


def test_upn_rate_envelope_on_quadratic():
    """Known mu, L on a 50-dim quadratic with mu/L = 1e-3: the iterates stay under the
    Nesterov envelope (1 - sqrt(mu/L))^k, Eq.(8), and decay log-linearly at
    least that fast."""
    n = 50
    lam = np.geomspace(1e-3, 1.0, n)
    d = np.sqrt(lam).astype(np.float32)
    lam = d.astype(np.float64) ** 2
    b = np.random.default_rng(6).standard_normal(n).astype(np.float32)
    P = _prob(diag_csr(d), b, (5, 5, 2), 0.0, 1e-3, lo=-math.inf)
    q = lam.min() / lam.max()
    res = oracle.upn(P, np.zeros(n), eps=1e-30, max_iters=1500, L_bar=lam.max(), mu_bar=lam.min())
    xs = b.astype(np.float64) / d.astype(np.float64)
    fstar = P.f(xs)
    gaps = np.array([h["f"] for h in res.history]) - fstar
    ks = np.arange(1, len(gaps) + 1)
    env = gaps[0] * (1 - math.sqrt(q)) ** (ks - 1)
    good = gaps > 1e-20
    assert np.all(gaps[good] <= 4.0 * env[good] + 1e-14)
    # fitted log-linear slope over the middle of the run is at least the envelope's
    sel = (ks > 100) & good
    slope = np.polyfit(ks[sel], np.log(gaps[sel]), 1)[0]
    assert slope <= 0.95 * math.log(1 - math.sqrt(q))


# ------------------------------------------------------------ optimality
def _dense_reference_optimum(A, b, grid, alpha, tau):
    """Independent optimiser: scipy L-BFGS-B on the dense assembly of Eq.(1)."""
    from scipy.optimize import minimize
    M = A.dense()
    D = dense_D(*grid)
    bb = np.asarray(b, np.float64)

    def fun(x):
        r = M @ x - bb
        Dx = (D @ x).reshape(-1, 3)
        t = np.sqrt((Dx ** 2).sum(1))
        h = np.where(t >= tau, t - tau / 2, t * t / (2 * tau))
        u = Dx / np.maximum(t, tau)[:, None]
        return 0.5 * r @ r + alpha * h.sum(), M.T @ r + alpha * (D.T @ u.ravel())

    res = minimize(fun, np.zeros(M.shape[1]), jac=True, method="L-BFGS-B",
                   bounds=[(0.0, None)] * M.shape[1],
                   options=dict(maxiter=200000, ftol=1e-16, gtol=1e-13, maxcor=50))
    return res.fun, res.x


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_dense_4cube_reaches_bruteforce_optimum(solver):
    grid = (4, 4, 4)
    A = random_csr(90, 64, 0.15, seed=21)
    b = np.random.default_rng(22).uniform(0, 2, 90).astype(np.float32)
    alpha, tau = 0.05, 1e-2
    fref, _ = _dense_reference_optimum(A, b, grid, alpha, tau)
    P = _prob(A, b, grid, alpha, tau)
    res = getattr(oracle, solver)(P, np.zeros(64), eps=1e-9, max_iters=50000)
    assert res.converged
    assert res.f <= fref * (1 + 1e-6)
    assert abs(res.f - fref) / fref <= 1e-6


def test_kkt_and_discriminative_stop():
    """KKT at the returned x and the stop criterion is discriminative:
    <= eps at exit, > 10 eps fifty iterations earlier."""
    A = harness.siddon_separable(10, 10, 5, 7, 15)
    xt = harness.phantom(10, 10, 5, 3)
    b = harness.simulate_data(A, xt)
    P = _prob(A, b, (10, 10, 5), 0.02, 1e-2)
    eps = 1e-7
    res = oracle.upn(P, np.zeros(P.N), eps=eps, max_iters=20000)
    assert res.converged and res.iters > 60
    g = P.grad(res.x)
    # |g_j| small where lo < x_j; g_j >= -tol where x_j = lo (the active bound)
    tol = 1e-4 * res.gmap_ref
    free = res.x > 1e-12
    assert np.all(np.abs(g[free]) <= tol)
    assert np.all(g[~free] >= -tol)
    gm = [h["gmap"] for h in res.history]
    assert gm[-1] <= eps * res.gmap_ref
    assert gm[-51] > 10 * eps * res.gmap_ref


def test_cross_solver_agreement_c1(c1):
    """GPBB and UPN converge to the same reconstruction on c1 (SURVEY §8(c).3 cross-solver)."""
    A = c1.A
    P = _prob(A, c1.b, c1.grid, c1.alpha, c1.tau)
    r1 = oracle.upn(P, np.zeros(c1.N), eps=1e-6, max_iters=20000)
    r2 = oracle.gpbb(P, np.zeros(c1.N), eps=1e-6, max_iters=20000)
    assert r1.converged and r2.converged
    assert abs(r1.f - r2.f) / r1.f <= 1e-5
    assert np.linalg.norm(r1.x - r2.x) / np.linalg.norm(r1.x) <= 1e-3


def test_gp_converges_and_is_slower_than_upn():
    A = harness.siddon_separable(10, 10, 4, 6, 15)
    b = harness.simulate_data(A, harness.phantom(10, 10, 4, 3))
    P = _prob(A, b, (10, 10, 4), 0.01, 1e-2)
    g = oracle.gp(P, np.zeros(P.N), eps=1e-4, max_iters=20000)
    u = oracle.upn(P, np.zeros(P.N), eps=1e-4, max_iters=20000)
    assert g.converged and u.converged and u.iters < g.iters


# ----------------------------------------------------------------------- GP
def test_gp_exact_step_spec_example():
    """f(x) = 1/2 (x - 1)^2, Q = R_+, x0 = 0, L known = 1 -> x1 = 1 exactly, converged in
    one step (Eq.(6), with BT of Alg. 2 accepting its first trial)."""
    P = _prob(identity_csr(1), [1.0], (1, 1, 1), 0.0, 1e-3)
    res = oracle.gp(P, np.zeros(1), eps=1e-12, max_iters=10, L_bar=1.0)
    assert res.converged and res.iters == 1
    assert res.x[0] == 1.0 and res.f == 0.0
    assert res.history[0]["L"] == 1.0 and res.history[0]["trials"] == 1


def _diag_quadratic(n=40, q=1e-2, seed=31):
    """f(x) = 1/2 ||D x - b||^2 with eigenvalues lam = d^2 in [q, 1] (fp32 d, exact lam)."""

    # one isolated smallest eigenvalue, so the slowest mode dominates after ~100 iterations
    d = np.sqrt(np.concatenate([[q], np.geomspace(5 * q, 1.0, n - 1)])).astype(np.float32)
    lam = d.astype(np.float64) ** 2
    b = np.random.default_rng(seed).uniform(-1, 1, n).astype(np.float32)
    xs = b.astype(np.float64) / d.astype(np.float64)
    return d, lam, b, xs


def test_gp_closed_form_trajectory_and_rate_envelope():
    """Unconstrained quadratic with L_bar = L = max lam: BT accepts its first trial every
    iteration (the bound of P:180 holds for L~ >= lam_max), so Eq.(6) gives the closed form
    x_k - x* = (1 - lam/L)^k (x_0 - x*) componentwise and
    f_k - f* = 1/2 sum lam (1 - lam/L)^(2k) e0^2.  The history must follow it, stay under the
    Eq.(7) envelope (1 - mu/L)^k C_GP and decay at the sharp slope 2 log(1 - mu/L)."""
    d, lam, b, xs = _diag_quadratic()
    P = _prob(diag_csr(d), b, (4, 5, 2), 0.0, 1e-3, lo=-math.inf)
    L, mu = lam.max(), lam.min()
    res = oracle.gp(P, np.zeros(len(d)), eps=1e-30, max_iters=600, L_bar=L)
    assert [h["trials"] for h in res.history] == [1] * len(res.history)
    assert all(h["L"] == L for h in res.history)
    e0 = -xs
    ks = np.array([h["iter"] for h in res.history])
    exact = np.array([0.5 * np.sum(lam * (1 - lam / L) ** (2 * k) * e0 ** 2) for k in ks])
    gaps = np.array([h["f"] for h in res.history]) - P.f(xs)
    ok = exact > 1e-9 * exact[0]
    assert np.allclose(gaps[ok], exact[ok], rtol=1e-6, atol=0)
    C = gaps[0] / (1 - mu / L)
    assert np.all(gaps[ok] <= C * (1 - mu / L) ** ks[ok] * (1 + 1e-9))
    sel = ok & (ks > 100)
    slope = np.polyfit(ks[sel], np.log(gaps[sel]), 1)[0]
    assert abs(slope / (2 * math.log(1 - mu / L)) - 1) <= 0.05


def test_gp_keeps_L_between_iterations():
    """Isotropic quadratic with Hessian L0 I and L_bar < L0: the first BT call takes
    ceil(log_rho(L0/L_bar)) + 1 trials, and because BT is seeded with L_{k-1}
    (P:213 for UPN) every later iteration accepts its first trial.  Resetting L to
    L_bar each iteration would repeat the long search."""
    n, L0, rho = 30, 10.0, 1.3
    s = np.float32(math.sqrt(L0))
    lam = float(s) ** 2
    b = np.random.default_rng(32).uniform(-1, 1, n).astype(np.float32)
    P = _prob(diag_csr(np.full(n, s)), b, (5, 3, 2), 0.0, 1e-3, lo=-math.inf)
    res = oracle.gp(P, np.zeros(n), eps=1e-12, max_iters=50, L_bar=1.0, rho=rho)
    m = math.ceil(math.log(lam / 1.0, rho) - 1e-12)
    assert res.history[0]["trials"] == m + 1
    assert all(h["trials"] == 1 for h in res.history[1:])
    Lt = rho ** m
    assert all(h["L"] == pytest.approx(Lt, rel=1e-12) for h in res.history)
    # each iteration contracts the error by exactly (1 - lam / L~)
    xs = b.astype(np.float64) / float(s)
    gap0 = P.f(np.zeros(n)) - P.f(xs)
    for h in res.history[:5]:
        assert h["f"] - P.f(xs) == pytest.approx(gap0 * (1 - lam / Lt) ** (2 * h["iter"]),
                                                 rel=1e-9, abs=1e-300)


def test_gp_monotone_on_ct_problem():
    """GP with BT decreases f at every iteration (S:317 'objective strictly nonincreasing'),
    and L_k never decreases (seeded with L_{k-1})."""
    A = harness.siddon_separable(10, 10, 4, 6, 15)
    b = harness.simulate_data(A, harness.phantom(10, 10, 4, 3))
    P = _prob(A, b, (10, 10, 4), 0.01, 1e-2)
    res = oracle.gp(P, np.zeros(P.N), eps=1e-5, max_iters=3000)
    f = np.array([h["f"] for h in res.history])
    assert np.all(np.diff(f) <= 1e-12 * np.abs(f[1:]))
    Ls = np.array([h["L"] for h in res.history])
    assert np.all(np.diff(Ls) >= 0)


def test_gp_stop_uses_nu_equal_L():
    """C11: the stop test of GP (as UPN) evaluates G_nu at x_{k+1} with nu = L_k (Eq.(10),
    P:225-228).  On a box-constrained CT problem the recorded map equals ||G_{L_k}(x)|| at the
    returned x, which differs from ||G_1(x)||, and the decision flips exactly at exit."""
    A = harness.siddon_separable(10, 10, 4, 6, 15)
    b = harness.simulate_data(A, harness.phantom(10, 10, 4, 3))
    P = _prob(A, b, (10, 10, 4), 0.01, 1e-2, lo=0.0, hi=0.6)
    eps = 1e-3
    res = oracle.gp(P, np.zeros(P.N), eps=eps, max_iters=20000)
    assert res.converged
    L = res.history[-1]["L"]
    g = P.grad(res.x)
    gL = float(np.linalg.norm(L * (res.x - P.proj(res.x - g / L))))
    g1 = float(np.linalg.norm(res.x - P.proj(res.x - g)))
    assert res.gmap == pytest.approx(gL, rel=1e-12)
    assert abs(gL - g1) > 1e-3 * gL
    assert res.history[-1]["gmap"] <= eps * res.gmap_ref < res.history[-2]["gmap"]


# ------------------------------------------------------------ stop scaling
def test_stop_abs_per_n_divides_by_N():
    """stop when ||G_nu(x^(k))||_2 / N <= eps (N, not sqrt N; C12)."""
    assert oracle._stop(0.5, 1.0, 100, 0.01, "abs_per_n")          # 0.005 <= 0.01
    assert not oracle._stop(2.0, 1.0, 100, 0.01, "abs_per_n")      # 0.02 > 0.01
    # with sqrt(N) this would not stop: 0.5 / 10 = 0.05 > 0.01
    assert not (0.5 / math.sqrt(100) <= 0.01)
    assert oracle._stop(0.5, 100.0, 100, 0.005, "rel") and not oracle._stop(0.6, 100.0, 100, 0.005, "rel")


def test_gp_abs_per_n_stop_iteration_closed_form():
    """On the closed-form quadratic of test_gp_closed_form_trajectory_and_rate_envelope (no
    active bounds, so G_L = grad f = lam e_k), the first k with ||lam (1 - lam/L)^k e0|| / N <= eps
    is known exactly; the solver must stop there, where dividing by sqrt(N) stops later."""
    d, lam, b, xs = _diag_quadratic()
    n = len(d)
    P = _prob(diag_csr(d), b, (4, 5, 2), 0.0, 1e-3, lo=-math.inf)
    L = lam.max()
    e0 = -xs
    gk = lambda k: float(np.linalg.norm(lam * (1 - lam / L) ** k * e0))
    eps = 1e-5
    k_n = next(k for k in range(1, 10000) if gk(k) / n <= eps)
    k_sqrt = next(k for k in range(1, 10000) if gk(k) / math.sqrt(n) <= eps)
    assert k_sqrt > k_n + 10
    res = oracle.gp(P, np.zeros(n), eps=eps, stop_mode="abs_per_n", max_iters=10000, L_bar=L)
    assert res.converged and res.iters == k_n
    assert res.gmap / n <= eps
