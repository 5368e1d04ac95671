"""Oracle: a plain, slow, obviously correct fp64 CPU reference for the paper's method.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product path (paper_1105_4002_b200/) never imports, links or executes it,
and the two share no code: no kernels, headers, helpers or constants.

Paper: Jorgensen et al., "Accelerated gradient methods for total-variation-based
CT image reconstruction" (/root/reference/PAPER.md, cited as P:line).

What it computes:
  * phi_tau(x) = 1/2 ||Ax - b||^2 + alpha * TV_tau(x)            Eq.(1)-(2)
  * grad phi_tau(x) = A^T (Ax - b) + alpha * grad TV_tau(x)
  * P_Q(v) = min(max(v, lo), hi)                                    P:119, P:246 (C22)
  * G_nu(x) = nu (x - P_Q(x - grad f(x)/nu))                        Eq.(10)
  * GPBB (Alg. 1), BT (Alg. 2), mu_k (Eq.(9)),
    UPN (Alg. 3), stopping rule with the readings C6-C14.
Heavy loops (A x, A^T y, TV) are in oracle.c; vectors here are fp64 numpy arrays
and the solver control follows the algorithms line by line.

Pins (tests/test_oracle_*.py): closed forms, finite differences, dense brute force,
exact dyadic adjointness, special-case solvers.  "parity unpinned": none of the
paper's own numbers exist (its figures are placeholders), so no
function is pinned to a printed paper value; every function here is pinned by
the mathematics instead (see DESIGN.md §Oracle pins).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2, no fast-math, OpenMP for row-parallel timing only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, f64, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        L.ora_matvec.restype = None
        L.ora_matvec.argtypes = [i64, vp, vp, vp, vp, vp, i32]
        L.ora_rmatvec_scatter.restype = None
        L.ora_rmatvec_scatter.argtypes = [i64, i64, vp, vp, vp, vp, vp]
        L.ora_transpose.restype = None
        L.ora_transpose.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp]
        L.ora_transpose_range.restype = None
        L.ora_transpose_range.argtypes = [i64, i64, vp, vp, vp, i64, i64, vp, vp, vp]
        L.ora_tv.restype = f64
        L.ora_tv.argtypes = [i32, i32, i32, vp, f64, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


# --------------------------------------------------------------- operators
def matvec(row_ptr, col, val, x, nthreads: int = 1) -> np.ndarray:
    """y = A x in fp64 (Eq.(1))."""
    x = _f64(x)
    m = len(row_ptr) - 1
    y = np.empty(m, np.float64)
    lib().ora_matvec(m, _p(row_ptr), _p(col), _p(val), _p(x), _p(y), nthreads)
    return y


def rmatvec(row_ptr, col, val, y, n: int) -> np.ndarray:
    """x = A^T y by scatter over A's rows (no transposed matrix)."""
    y = _f64(y)
    m = len(row_ptr) - 1
    x = np.empty(n, np.float64)
    lib().ora_rmatvec_scatter(m, n, _p(row_ptr), _p(col), _p(val), _p(y), _p(x))
    return x


def transpose(row_ptr, col, val, n: int):
    """Canonical A^T (rows = columns of A, entries ascending by source row; C20)."""
    m = len(row_ptr) - 1
    nnz = int(row_ptr[-1])
    rT = np.empty(n + 1, np.int64)
    cT = np.empty(nnz, np.int32)
    vT = np.empty(nnz, np.float32)
    lib().ora_transpose(m, n, _p(row_ptr), _p(col), _p(val), _p(rT), _p(cT), _p(vT))
    return rT, cT, vT


def transpose_range(row_ptr, col, val, n: int, j0: int, j1: int):
    """(rowT in full, colT[rowT[j0]:rowT[j1]], valT[rowT[j0]:rowT[j1]]) of the canonical A^T
    (same stable counting sort as transpose(); for matrices too large to transpose twice)."""
    m = len(row_ptr) - 1
    rT = np.empty(n + 1, np.int64)
    # sizes of the part come from the histogram, computed first by the same routine
    lib().ora_transpose_range(m, n, _p(row_ptr), _p(col), _p(val), 0, 0, _p(rT), None, None)
    cnt = int(rT[j1] - rT[j0])
    cT = np.empty(max(cnt, 1), np.int32)
    vT = np.empty(max(cnt, 1), np.float32)
    lib().ora_transpose_range(m, n, _p(row_ptr), _p(col), _p(val), j0, j1, _p(rT), _p(cT), _p(vT))
    return rT, cT[:cnt], vT[:cnt]


def tv(grid, x, tau: float, want_grad: bool = True):
    """(TV_tau(x), grad TV_tau(x) or None); Eq.(2) with Huber h_tau (C1-C3)."""
    nx, ny, nz = grid
    x = _f64(x)
    g = np.empty(nx * ny * nz, np.float64) if want_grad else None
    val = lib().ora_tv(nx, ny, nz, _p(x), float(tau), _p(g) if want_grad else None)
    return val, g


# ----------------------------------------------------------------- problem
class LineSearchError(RuntimeError):
    """beta < beta_min in GPBB or more than bt_max BT trials."""


class ThetaError(RuntimeError):
    """UPN theta outside (0, 1]."""


class NonFiniteError(RuntimeError):
    """Non-finite objective or gradient."""


@dataclass
class Problem:
    """phi_tau(x) = 1/2||Ax-b||^2 + alpha TV_tau(x) over Q = [lo, hi]^N (Eq.(1)).

    A is given by CSR arrays (row_ptr int64, col int32, val fp32), b fp32; all
    arithmetic in fp64.  ``nthreads`` only splits independent rows of A x."""
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    b: np.ndarray
    grid: tuple
    alpha: float
    tau: float
    lo: float = 0.0
    hi: float = math.inf
    nthreads: int = 1
    n_f: int = field(default=0, init=False)
    n_g: int = field(default=0, init=False)

    @property
    def N(self) -> int:
        nx, ny, nz = self.grid
        return nx * ny * nz

    def use_transpose(self):
        """Compute A^T y row-parallel over the oracle's own canonical transpose (the
        multi-core timing mode of SURVEY §8(d)); the default is the scatter over A's rows."""
        self._T = transpose(self.row_ptr, self.col, self.val, self.N)
        return self

    def rmatvec(self, y) -> np.ndarray:
        T = getattr(self, "_T", None)
        if T is not None:
            return matvec(T[0], T[1], T[2], y, self.nthreads)
        return rmatvec(self.row_ptr, self.col, self.val, y, self.N)

    # r = A x - b
    def residual(self, x) -> np.ndarray:
        return matvec(self.row_ptr, self.col, self.val, x, self.nthreads) - self.b.astype(np.float64)

    def fidelity(self, x) -> float:
        r = self.residual(x)
        return 0.5 * float(r @ r)

    def f(self, x) -> float:
        """phi_tau(x), Eq.(1)."""
        self.n_f += 1
        r = self.residual(x)
        t, _ = tv(self.grid, x, self.tau, want_grad=False)
        val = 0.5 * float(r @ r) + self.alpha * t
        if not math.isfinite(val):
            raise NonFiniteError("f")
        return val

    def fg(self, x):
        """(phi_tau(x), grad phi_tau(x)) = (fid + alpha TV, A^T(Ax-b) + alpha grad TV)."""
        self.n_f += 1
        self.n_g += 1
        r = self.residual(x)
        t, gt = tv(self.grid, x, self.tau, want_grad=True)
        g = self.rmatvec(r) + self.alpha * gt
        val = 0.5 * float(r @ r) + self.alpha * t
        if not (math.isfinite(val) and np.all(np.isfinite(g))):
            raise NonFiniteError("f/g")
        return val, g

    def grad(self, x) -> np.ndarray:
        return self.fg(x)[1]

    def proj(self, v) -> np.ndarray:
        """P_Q(v) = min(max(v, lo), hi) (C22)."""
        return np.minimum(np.maximum(_f64(v), self.lo), self.hi)

    def gradient_map(self, x, nu: float, g=None) -> np.ndarray:
        """G_nu(x) = nu (x - P_Q(x - nu^{-1} grad f(x))), Eq.(10) P:225-227."""
        if g is None:
            g = self.grad(x)
        return nu * (x - self.proj(x - g / nu))


def _stop(gn: float, g_ref: float, N: int, eps: float, mode: str) -> bool:
    """P:228 'stop if ||G_nu(x^(k))||_2 / N <= eps' (mode 'abs_per_n');
    mode 'rel' (BJ:7): ||G_nu(x_k)||_2 <= eps * ||G_1(x_0)||_2 (C12, C25)."""
    if mode == "abs_per_n":
        return gn / N <= eps
    return gn <= eps * g_ref


@dataclass
class Result:
    x: np.ndarray
    converged: bool
    iters: int
    f: float
    gmap: float
    gmap_ref: float
    n_f: int
    n_g: int
    n_ls: int
    history: list


# -------------------------------------------------------------- Alg. 1 GPBB
def gpbb(P: Problem, x0, max_iters: int = 10000, eps: float = 1e-6, stop_mode: str = "rel",
         K: int = 2, sigma: float = 0.1, beta0: float = 0.95, beta_min: float = 1e-10) -> Result:
    """GPBB, Alg. 1, readings C6, C11-C14, C21.

    theta_0 = 1; for k > 0 the BB step
    theta_k = ||x_k - x_{k-1}||^2 / <x_k - x_{k-1}, g_k - g_{k-1}>, kept at
    theta_{k-1} if the denominator is <= 0 or non-finite (C6).  beta = 0.95,
    x_bar = P_Q(x_k - beta theta_k g_k), f_hat = max of the last K+1 accepted
    f values (C21), loop while f(x_bar) >= f_hat - sigma g_k^T (x_k - x_bar)
     with beta <- beta^2.  The stop test runs at the top of
    iteration k with nu = 1/theta_k (C11, C14)."""
    P.n_f = P.n_g = 0
    x = P.proj(x0)
    f, g = P.fg(x)
    g_ref = float(np.linalg.norm(P.gradient_map(x, 1.0, g)))
    fhist = [f]
    theta = 1.0
    x_prev = g_prev = None
    hist = []
    n_ls = 0
    k = 0
    while True:
        if k > 0:
            dx = x - x_prev
            dg = g - g_prev
            den = float(dx @ dg)
            if den > 0.0 and math.isfinite(den):
                theta = float(dx @ dx) / den
        gn = float(np.linalg.norm((x - P.proj(x - theta * g)) / theta))
        conv = _stop(gn, g_ref, P.N, eps, stop_mode)
        if conv or k >= max_iters:
            hist.append(dict(iter=k, f=f, gmap=gn, step=theta, trials=0))
            return Result(x, conv, k, f, gn, g_ref, P.n_f, P.n_g, n_ls, hist)
        beta = beta0
        fhat = max(fhist[-(K + 1):])
        trials = 0
        while True:
            x_bar = P.proj(x - beta * theta * g)
            f_bar = P.f(x_bar)
            trials += 1
            rhs = fhat - sigma * float(g @ (x - x_bar))
            if not (f_bar >= rhs):
                break
            beta = beta * beta
            if beta < beta_min:
                raise LineSearchError(f"GPBB beta < {beta_min} at k={k}")
        n_ls += trials
        hist.append(dict(iter=k, f=f, gmap=gn, step=theta, trials=trials, f_next=f_bar,
                         armijo_rhs=rhs, beta=beta))
        x_prev, g_prev = x, g
        x = x_bar
        f = f_bar
        g = P.grad(x)
        fhist.append(f)
        k += 1


# ---------------------------------------------------------------- Alg. 2 BT
def backtrack(P: Problem, y, f_y: float, g_y, L_bar: float, rho: float = 1.3,
              bt_max: int = 200):
    """BT, Alg. 2, reading C7: L~ = L_bar; x = P_Q(y - g_y/L~); while
    f(x) > f(y) + g_y^T(x - y) + L~/2 ||x - y||^2: L~ <- rho L~.
    Returns (x, f(x), L~, trials)."""
    L = L_bar
    trials = 0
    while True:
        x = P.proj(y - g_y / L)
        fx = P.f(x)
        trials += 1
        d = x - y
        if not (fx > f_y + float(g_y @ d) + 0.5 * L * float(d @ d)):
            return x, fx, L, trials
        if trials >= bt_max:
            raise LineSearchError(f"BT exceeded {bt_max} trials")
        L = rho * L


def mu_estimate(mu_prev: float, f_x: float, f_y: float, g_y, x, y) -> float:
    """Eq.(9) with Alg. 3's pairing (C9):
    mu_k = min(mu_{k-1}, (f(x) - f(y) - grad f(y)^T (x - y)) / (1/2 ||x - y||^2));
    keep mu_{k-1} if x = y or the quotient is <= 0 or non-finite."""
    d = x - y
    dd = float(d @ d)
    if dd <= 0.0:
        return mu_prev
    M = (f_x - f_y - float(g_y @ d)) / (0.5 * dd)
    if not (M > 0.0 and math.isfinite(M)):
        return mu_prev
    return min(mu_prev, M)


def theta_root(theta_k: float, q: float) -> float:
    """Positive root of theta^2 = (1 - theta) theta_k^2 + q theta, C10."""
    a = theta_k * theta_k - q
    s = math.sqrt(a * a + 4.0 * theta_k * theta_k)
    return 2.0 * theta_k * theta_k / (a + s) if a >= 0.0 else 0.5 * (-a + s)


# --------------------------------------------------------------- Alg. 3 UPN
def upn(P: Problem, x0, max_iters: int = 10000, eps: float = 1e-6, stop_mode: str = "rel",
        L_bar: float = 1.0, mu_bar: float | None = None, rho: float = 1.3,
        bt_max: int = 200) -> Result:
    """UPN, Alg. 3 with BT (Alg. 2), readings C7-C14.

    [x1, L0] = BT(x0, L_bar); mu_0 = mu_bar (= L_bar, C8); y1 = x1; theta_1 = sqrt(mu_0/L_0).
    For k >= 1: [x_{k+1}, L_k] = BT(y_k, L_{k-1}); mu_k = min(mu_{k-1}, M(x_k, y_k));
    theta_{k+1} = positive root; beta_k = theta_k (1-theta_k)/(theta_k^2 + theta_{k+1});
    y_{k+1} = x_{k+1} + beta_k (x_{k+1} - x_k).  Stop test at x_{k+1} with nu = L_k (C11);
    also at x_1 after the first BT (C13).  f(y), grad f(y) are evaluated directly."""
    if mu_bar is None:
        mu_bar = L_bar
    P.n_f = P.n_g = 0
    x0 = P.proj(x0)
    f0, g0 = P.fg(x0)
    g_ref = float(np.linalg.norm(P.gradient_map(x0, 1.0, g0)))
    hist = []
    x1, f1, L, trials = backtrack(P, x0, f0, g0, L_bar, rho, bt_max)
    n_ls = trials
    mu = mu_bar
    theta = math.sqrt(mu / L)
    if not (0.0 < theta <= 1.0):
        raise ThetaError(f"theta_1 = {theta}")
    g1 = P.grad(x1)
    gn = float(np.linalg.norm(P.gradient_map(x1, L, g1)))
    hist.append(dict(iter=1, f=f1, gmap=gn, L=L, mu=mu, theta=theta, trials=trials))
    x_k, f_xk = x1, f1
    y, f_y, g_y = x1, f1, g1
    k = 1
    conv = _stop(gn, g_ref, P.N, eps, stop_mode)
    while not conv and k < max_iters:
        x_next, f_next, L, trials = backtrack(P, y, f_y, g_y, L, rho, bt_max)
        n_ls += trials
        mu = mu_estimate(mu, f_xk, f_y, g_y, x_k, y)
        theta_next = theta_root(theta, mu / L)
        if not (0.0 < theta_next <= 1.0) or not math.isfinite(theta_next):
            raise ThetaError(f"theta = {theta_next} at k={k}")
        beta = theta * (1.0 - theta) / (theta * theta + theta_next)
        y = x_next + beta * (x_next - x_k)
        g_next = P.grad(x_next)
        gn = float(np.linalg.norm(P.gradient_map(x_next, L, g_next)))
        k += 1
        hist.append(dict(iter=k, f=f_next, gmap=gn, L=L, mu=mu, theta=theta_next, trials=trials))
        x_k, f_xk, theta = x_next, f_next, theta_next
        conv = _stop(gn, g_ref, P.N, eps, stop_mode)
        if conv:
            break
        f_y, g_y = P.fg(y)
    return Result(x_k, conv, k, f_xk, gn, g_ref, P.n_f, P.n_g, n_ls, hist)


# -------------------------------------------------------------- Eq.(6) GP
def gp(P: Problem, x0, max_iters: int = 10000, eps: float = 1e-6, stop_mode: str = "rel",
       L_bar: float = 1.0, rho: float = 1.3, bt_max: int = 200) -> Result:
    """Gradient projection, Eq.(6), step theta_k = 1/L_k from BT.
    The paper's baseline comparator."""
    P.n_f = P.n_g = 0
    x = P.proj(x0)
    f, g = P.fg(x)
    g_ref = float(np.linalg.norm(P.gradient_map(x, 1.0, g)))
    L = L_bar
    hist = []
    n_ls = 0
    k = 0
    while True:
        x_next, f_next, L, trials = backtrack(P, x, f, g, L, rho, bt_max)
        n_ls += trials
        k += 1
        x, f = x_next, f_next
        g = P.grad(x)
        gn = float(np.linalg.norm(P.gradient_map(x, L, g)))
        hist.append(dict(iter=k, f=f, gmap=gn, L=L, trials=trials))
        conv = _stop(gn, g_ref, P.N, eps, stop_mode)
        if conv or k >= max_iters:
            return Result(x, conv, k, f, gn, g_ref, P.n_f, P.n_g, n_ls, hist)
