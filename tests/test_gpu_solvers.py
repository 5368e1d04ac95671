"""Solver parity: GPU GPBB / UPN against the oracle's GPBB / UPN on
the BJ:7 workload c1 and variants.  Both results are evaluated with the ORACLE's objective;
bars from BASELINE.json north_star: relative objective gap <= 1e-5, relative image difference
<= 1e-3.  Plus invariant replay from the recorded histories."""
import math

import numpy as np
import pytest

import harness
import oracle
from tests._helpers import diag_csr, identity_csr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tvreg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1105_4002_b200 import tvreg as T
    return T


def _oracle_problem(w, **over):
    kw = dict(alpha=w.alpha, tau=w.tau, lo=w.lo, hi=w.hi)
    kw.update(over)
    return oracle.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, nthreads=4, **kw)


def _gpu_problem(T, w, **over):
    kw = dict(alpha=w.alpha, tau=w.tau, lo=w.lo, hi=w.hi)
    kw.update(over)
    return T.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, kw["alpha"], kw["tau"], kw["lo"], kw["hi"])


def _check_parity(Po, x_gpu, res_ora):
    f_gpu = Po.f(x_gpu.astype(np.float64))
    f_ora = Po.f(res_ora.x)
    gap = abs(f_gpu - f_ora) / abs(f_ora)
    diff = np.linalg.norm(x_gpu - res_ora.x) / np.linalg.norm(res_ora.x)
    assert gap <= 1e-5, gap
    assert diff <= 1e-3, diff
    return gap, diff


@pytest.fixture(scope="module")
def c1_ref(c1):
    Po = _oracle_problem(c1)
    return dict(upn=oracle.upn(Po, np.zeros(c1.N), eps=1e-6, max_iters=20000),
                gpbb=oracle.gpbb(Po, np.zeros(c1.N), eps=1e-6, max_iters=20000), P=Po)


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_solver_parity_c1(tvreg, c1, c1_ref, solver):
    P = _gpu_problem(tvreg, c1)
    x = torch.zeros(c1.N, device="cuda")
    res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6, hist_cap=25000)
    assert res.converged
    ref = c1_ref[solver]
    _check_parity(c1_ref["P"], x.cpu().numpy(), ref)
    # iteration counts within a modest factor of the oracle's (BB steps amplify rounding)
    assert 0.5 * ref.iters <= res.iters <= 2.0 * ref.iters
    assert res.gmap_rel <= 1e-6
    h = res.history
    assert len(h) == res.iters + (1 if solver == "gpbb" else 0)
    if solver == "upn":
        mus = [r["mu"] for r in h]
        Ls = [r["L"] for r in h]
        assert all(a >= b for a, b in zip(mus, mus[1:]))
        assert all(a <= b for a, b in zip(Ls, Ls[1:]))
    else:
        assert all(r["step"] > 0 for r in h)
    # the first iterations agree with the oracle's trajectory
    oh = ref.history
    for k in range(3):
        assert abs(h[k]["f"] - oh[k]["f"]) <= 1e-6 * abs(oh[k]["f"])


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_solver_parity_box_constraint(tvreg, solver):
    """c4-shaped: box Q = [0, 1], tau = 1e-2 (BJ:10) at desk size, solved to the BJ:7 tolerance
    1e-6 (UPN carries its iterates as hi + lo pairs: with fp32 iterates it stalled near 1.2e-6 on
    this problem) against an oracle reference at 1e-7."""
    w = harness.separable_workload("c4s", (24, 24, 12), 10, 35, 5, alpha=0.03, tau=1e-2, hi=1.0)
    Po = _oracle_problem(w)
    ref = getattr(oracle, solver)(Po, np.zeros(w.N), eps=1e-7, max_iters=20000)
    P = _gpu_problem(tvreg, w)
    x = torch.zeros(w.N, device="cuda")
    res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6)
    assert res.converged and ref.converged
    xg = x.cpu().numpy()
    assert xg.min() >= 0.0 and xg.max() <= 1.0
    _check_parity(Po, xg, ref)


def test_solver_identity_closed_form(tvreg):
    """A = I, alpha = 0: the minimiser is P_Q(b)."""
    n = 4 * 4 * 4
    A = identity_csr(n)
    b = np.random.default_rng(1).uniform(-1, 1, n).astype(np.float32)
    for solver in ("gpbb", "upn"):
        P = tvreg.Problem(A.row_ptr, A.col, A.val, b, (4, 4, 4), 0.0, 1e-3, 0.0, 0.5)
        x = torch.zeros(n, device="cuda")
        res = getattr(P, f"solve_{solver}")(x, eps=1e-6, max_iters=1000)
        assert res.converged
        assert np.allclose(x.cpu().numpy(), np.clip(b, 0, 0.5), atol=1e-6)


def test_abs_per_n_stop_mode_and_max_iters(tvreg, c1):
    P = _gpu_problem(tvreg, c1)
    x = torch.zeros(c1.N, device="cuda")
    res = P.solve_upn(x, max_iters=7, eps=1e-30, stop_mode=tvreg.TVR_STOP_ABS_PER_N)
    assert res.status == tvreg.TVR_NOT_CONVERGED and not res.converged and res.iters == 7
    x2 = torch.zeros(c1.N, device="cuda")
    res2 = P.solve_gpbb(x2, max_iters=5, eps=1e-30)
    assert res2.status == tvreg.TVR_NOT_CONVERGED and res2.iters == 5
    # P:228 scaling: ||G||/N, with N the voxel count
    assert abs(res.gmap_abs_per_n * c1.N - res.gmap_rel * res.gmap_ref) <= 1e-9 * res.gmap_ref


def test_gp_parity_c1(tvreg, c1):
    """GP (f1, Eq. (6) with BT steps): 150 iterations on c1 against the oracle's gp(): same L_k
    sequence, f_k to fp32-storage accuracy, monotone f, and the final iterate within the
    north_star bars."""
    Po = _oracle_problem(c1)
    ref = oracle.gp(Po, np.zeros(c1.N), eps=0.0, max_iters=150)
    P = _gpu_problem(tvreg, c1)
    x = torch.zeros(c1.N, device="cuda")
    res = P.solve_gp(x, max_iters=150, eps=0.0, hist_cap=200)
    assert not res.converged and res.iters == 150
    h, oh = res.history, ref.history
    assert len(h) == 150
    assert [r["L"] for r in h] == [r["L"] for r in oh]
    for k in range(150):
        assert abs(h[k]["f"] - oh[k]["f"]) <= 1e-6 * abs(oh[k]["f"])
    fs = [r["f"] for r in h]
    assert all(a >= b for a, b in zip(fs, fs[1:]))  # BT's sufficient decrease
    _check_parity(Po, x.cpu().numpy(), ref)


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
@pytest.mark.parametrize("case", ["c1", "box"])
def test_device_control_matches_host_control(tvreg, c1, case, solver, monkeypatch):
    """f3: a solve as one CUDA graph with conditional nodes and device control kernels takes the
    host controller's decisions in the same fp64 arithmetic: identical iterates, counts, history.
    (UPN's graph evaluates its hi + lo iterates whole from the start; the host controller switches
    to that at a gradient-map ratio of TVR_EXT_EVAL_AT, set to 1 here: from the start too.)"""
    monkeypatch.setenv("TVR_EXT_EVAL_AT", "1")
    kw = {} if case == "c1" else dict(alpha=0.03, tau=1e-2, hi=1.0)
    outs = {}
    for mode in ("host", "device"):
        P = _gpu_problem(tvreg, c1, **kw)
        P.set_control(mode)
        x = torch.zeros(c1.N, device="cuda")
        res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6,
                                            hist_cap=25000)
        outs[mode] = (res, x.clone())
        P.close()
    (rh, xh), (rd, xd) = outs["host"], outs["device"]
    assert rd.converged == rh.converged and rd.iters == rh.iters
    assert (rd.n_f, rd.n_grad, rd.n_ls) == (rh.n_f, rh.n_grad, rh.n_ls)
    assert rd.f == rh.f and rd.gmap_rel == rh.gmap_rel
    assert torch.equal(xd, xh)
    assert rd.history == rh.history


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_device_control_max_iters_and_restart(tvreg, c1, solver, monkeypatch):
    """max_iters stops the device loop like the host loop, and a second solve on the same problem
    starts from fresh controller state."""
    monkeypatch.setenv("TVR_EXT_EVAL_AT", "1")
    P = _gpu_problem(tvreg, c1)
    res = []
    for mode in ("host", "device", "device"):
        P.set_control(mode)
        x = torch.zeros(c1.N, device="cuda")
        res.append((getattr(P, f"solve_{solver}")(x, max_iters=7, eps=1e-12, hist_cap=20), x.clone()))
    for r, x in res[1:]:
        assert not r.converged and r.iters == 7
        assert len(r.history) == (8 if solver == "gpbb" else 7)
        assert r.history == res[0][0].history and torch.equal(x, res[0][1])


@pytest.fixture(scope="module")
def c2_ref():
    """The oracle's own c2 solves (BJ:8 workload, 128^3, 1.6e8 entries) to REL 1e-6: A x
    row-parallel on every host core, A^T r row-parallel over the oracle's own canonical
    transpose (SURVEY §8(d) oracle timing mode; same fp64 sums per row as the scatter)."""
    import os
    w = harness.preset("c2")
    Po = oracle.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                        nthreads=os.cpu_count() or 1).use_transpose()
    return w, Po, {}


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_solver_parity_c2(tvreg, c2_ref, solver):
    """SURVEY §8(c).4 item 3 at c2: the GPU solve (bench configuration, device-side control)
    against the oracle's solve of the same problem, both evaluated with the oracle's objective:
    relative objective gap <= 1e-5, relative image difference <= 1e-3 (BJ:5)."""
    w, Po, cache = c2_ref
    ref = getattr(oracle, solver)(Po, np.zeros(w.N), eps=1e-6, max_iters=20000)
    assert ref.converged
    P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
    x = torch.zeros(w.N, device="cuda")
    res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6)
    assert res.converged
    gap, diff = _check_parity(Po, x.cpu().numpy(), ref)
    assert 0.5 * ref.iters <= res.iters <= 2.0 * ref.iters


def test_gp_abs_per_n_stop_closed_form(tvreg):
    """P:228's stop rule ||G_nu||/N <= eps through the C ABI, on the closed-form quadratic of
    the oracle pin (tests/test_oracle_solvers.py): unconstrained f = 1/2||D x - b||^2 with
    L_bar = L = max lam, so x_k - x* = (1 - lam/L)^k (x_0 - x*) and the stop iteration is the
    first k with ||lam (1 - lam/L)^k e0|| / N <= eps; with sqrt(N) it would be far later."""
    n, q = 40, 1e-2
    d = np.sqrt(np.concatenate([[q], np.geomspace(5 * q, 1.0, n - 1)])).astype(np.float32)
    lam = d.astype(np.float64) ** 2
    b = np.random.default_rng(31).uniform(-1, 1, n).astype(np.float32)
    e0 = -(b.astype(np.float64) / d.astype(np.float64))
    L = float(lam.max())
    gk = lambda k: float(np.linalg.norm(lam * (1 - lam / L) ** k * e0))
    eps = math.sqrt(gk(499) * gk(500)) / n  # half-way between two iterates: margin over fp32
    k_n = next(k for k in range(1, 10000) if gk(k) / n <= eps)
    assert k_n == 500 and gk(k_n) / math.sqrt(n) > 5 * eps  # sqrt(N) would not stop here
    assert gk(k_n - 1) / n > 1.001 * eps and gk(k_n) / n < 0.999 * eps  # margin over fp32 storage
    A = diag_csr(d)
    P = tvreg.Problem(A.row_ptr, A.col, A.val, b, (4, 5, 2), 0.0, 1e-3, -math.inf, math.inf)
    for solver in ("gp",):
        x = torch.zeros(n, device="cuda")
        res = P.solve_gp(x, max_iters=10000, eps=eps, stop_mode=tvreg.TVR_STOP_ABS_PER_N, L0=L)
        assert res.converged and res.iters == k_n
        assert res.gmap_abs_per_n <= eps


def test_gpbb_long_nonmonotone_window(tvreg, c1):
    """f_hat of P:147 is the max over the last K + 1 accepted values for any K (the host
    controller used to keep at most 64).  K = 100 (host control: more than the device
    controller's 64 slots) runs 120 iterations, follows the oracle's GPBB with K = 100 over the
    first iterations, and is identical to K = 63 while both windows still hold every accepted
    value (iterations < 64); every accepted value lies below the max of the K + 1 before it."""
    outs = {}
    for K in (63, 100):
        P = _gpu_problem(tvreg, c1)
        P.set_control("host")
        x = torch.zeros(c1.N, device="cuda")
        res = P.solve_gpbb(x, max_iters=120, eps=0.0, K=K, hist_cap=200)
        assert res.iters == 120
        outs[K] = res.history
        P.close()
    a, b = outs[63], outs[100]
    assert a[:64] == b[:64]
    fs = [r["f"] for r in b]
    assert all(fs[k + 1] < max(fs[max(0, k - 100):k + 1]) for k in range(len(fs) - 1))
    ref = oracle.gpbb(_oracle_problem(c1), np.zeros(c1.N), eps=0.0, max_iters=5, K=100)
    for k in range(3):
        assert abs(b[k]["f"] - ref.history[k]["f"]) <= 1e-6 * abs(ref.history[k]["f"])


@pytest.mark.parametrize("alpha", [0.003, 0.03])
@pytest.mark.parametrize("solver", ["upn", "gpbb"])
def test_solver_parity_c4_recipe_desk(tvreg, solver, alpha):
    """BJ:10's c4 recipe (box [0, 1], tau = 1e-2) at 32^3 (12 views x 45 bins, 10 ellipsoids):
    the fp64 oracle's UPN converges to 1e-7 here while fp32 iterates stalled the GPU UPN near
    2e-6 (profiles/r02/c4_study.md); with hi + lo iterates the GPU solve reaches 1e-6 and matches
    the oracle's reconstruction."""
    w = harness.preset("c4", grid=(32, 32, 32), views=12, bins=45)
    Po = oracle.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, alpha, 1e-2, 0.0, 1.0)
    ref = getattr(oracle, solver)(Po, np.zeros(w.N), eps=1e-7, max_iters=20000)
    P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, alpha, 1e-2, 0.0, 1.0)
    x = torch.zeros(w.N, device="cuda")
    res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6)
    assert res.converged and ref.converged
    _check_parity(Po, x.cpu().numpy(), ref)


@pytest.mark.parametrize("solver", ["upn", "gp"])
def test_solver_parity_gather_layouts_extended(tvreg, solver, monkeypatch):
    """Non-separable rays (c5's geometry at desk size) through the int32 sliced ELL with block
    modes and the gather layouts (row-major / x-y swapped / bricks), with the extended-precision
    evaluation on from the start (the A pass also gathers the lo parts from the re-laid-out lo
    vector): the converged reconstruction against the oracle's."""
    monkeypatch.setenv("TVR_SPMV_SELL32", "3")
    monkeypatch.setenv("TVR_EXT_EVAL_AT", "1")
    grid = (32, 24, 16)
    A = harness.siddon_tilted(*grid, 12, 16, 41, 10.0)
    xt = harness.phantom(*grid, 4)
    b = harness.simulate_data(A, xt)
    alpha, tau = 0.01, 1e-2
    Po = oracle.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau, 0.0, np.inf, nthreads=4)
    P = tvreg.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau, 0.0, np.inf)
    lb = list(P.info.gather_layout_blocks)
    assert min(lb) > 0, lb
    x = torch.zeros(A.n_cols, device="cuda")
    if solver == "upn":
        ref = oracle.upn(Po, np.zeros(A.n_cols), eps=1e-6, max_iters=20000)
        res = P.solve_upn(x, max_iters=20000, eps=1e-6)
        assert res.converged and ref.converged
        _check_parity(Po, x.cpu().numpy(), ref)
    else:  # GP (Eq. (6)): 150 iterations follow the oracle's trajectory
        ref = oracle.gp(Po, np.zeros(A.n_cols), eps=0.0, max_iters=150)
        res = P.solve_gp(x, max_iters=150, eps=0.0, hist_cap=200)
        h, oh = res.history, ref.history
        assert len(h) == 150
        for k in range(150):
            assert abs(h[k]["f"] - oh[k]["f"]) <= 1e-6 * abs(oh[k]["f"])
