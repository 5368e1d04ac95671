"""Seeded synthetic inputs for the TV-reconstruction hot path (input generators only).

Builds the workloads of BASELINE.json configs c1-c5 from the
conventions of SURVEY.md §8(c): Siddon system matrix (C15), slice-major /
view-major row order (C4), additive-ellipsoid phantom (C17), noise
sigma = 0.01*||A x_true||/sqrt(m) (C16), random test point x ~ U[0,1) (seed 3).
The paper's FORBILD phantom and 3D sphere geometry are not
available; these seeded inputs stand in for them.

This module holds none of the method's arithmetic.  It is shared by oracle/ and
by the CUDA path's tests/bench, and imports neither.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "harness.cpp")
_LIB = os.path.join(_HERE, "libtvrharness.so")

SEED_PHANTOM = 1
SEED_NOISE = 2
SEED_X = 3


def build(force: bool = False) -> str:
    """Compile harness.cpp into libtvrharness.so (g++, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c++17",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, f64, vp, u64 = (ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_void_p, ctypes.c_uint64)
        L.hx_siddon2d.restype = i64
        L.hx_siddon2d.argtypes = [i32, i32, i32, i32, vp, vp, vp]
        L.hx_siddon3d.restype = i64
        L.hx_siddon3d.argtypes = [i32, i32, i32, i32, i32, i32, f64, vp, vp, vp]
        L.hx_siddon3d_views.restype = i64
        L.hx_siddon3d_views.argtypes = [i32, i32, i32, i32, i32, i32, f64, i32, i32, vp, vp, vp]
        L.hx_siddon_sphere.restype = i64
        L.hx_siddon_sphere.argtypes = [i32, i32, i32, i32, i32, i32, vp, vp, vp]
        L.hx_replicate_slices.restype = None
        L.hx_replicate_slices.argtypes = [i64, i64, vp, vp, vp, i64, i32, vp, vp, vp]
        L.hx_simulate_projections.restype = None
        L.hx_simulate_projections.argtypes = [i64, vp, vp, vp, vp, vp]
        L.hx_phantom.restype = None
        L.hx_phantom.argtypes = [i32, i32, i32, i32, u64, vp]
        L.hx_uniform.restype = None
        L.hx_uniform.argtypes = [i64, u64, vp]
        L.hx_normal.restype = None
        L.hx_normal.argtypes = [i64, u64, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------- matrices
@dataclass
class CSR:
    """CSR matrix: int64 row_ptr[m+1], int32 col[nnz], fp32 val[nnz]."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val.astype(np.float64), self.col, self.row_ptr),
                             shape=(self.n_rows, self.n_cols))


def siddon_slice(nx: int, ny: int, views: int, bins: int) -> CSR:
    """One axial slice's Siddon matrix (rows v*bins + b, cols iy*nx + ix); C15."""
    L = lib()
    m = views * bins
    rp = np.zeros(m + 1, np.int64)
    nnz = L.hx_siddon2d(nx, ny, views, bins, _p(rp), None, None)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32)
    L.hx_siddon2d(nx, ny, views, bins, _p(rp), _p(col), _p(val))
    return CSR(m, nx * ny, rp, col, val)


def siddon_separable(nx: int, ny: int, nz: int, views: int, bins: int) -> CSR:
    """Slice-separable parallel-beam matrix, slice-major rows (z*V + v)*bins + b (C4)."""
    s = siddon_slice(nx, ny, views, bins)
    m = s.n_rows * nz
    nnz = s.nnz * nz
    rp = np.empty(m + 1, np.int64)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32)
    lib().hx_replicate_slices(s.n_rows, s.nnz, _p(s.row_ptr), _p(s.col), _p(s.val),
                              nx * ny, nz, _p(rp), _p(col), _p(val))
    return CSR(m, nx * ny * nz, rp, col, val)


def siddon_tilted(nx: int, ny: int, nz: int, views: int, det_rows: int, det_cols: int,
                  phimax_deg: float = 10.0) -> CSR:
    """Non-separable geometry of c5: rays tilted in z by up to +-phimax (C15), view-major rows."""
    L = lib()
    m = views * det_rows * det_cols
    rp = np.zeros(m + 1, np.int64)
    nnz = L.hx_siddon3d(nx, ny, nz, views, det_rows, det_cols, phimax_deg, _p(rp), None, None)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32)
    L.hx_siddon3d(nx, ny, nz, views, det_rows, det_cols, phimax_deg, _p(rp), _p(col), _p(val))
    return CSR(m, nx * ny * nz, rp, col, val)


def siddon_tilted_views(nx: int, ny: int, nz: int, views: int, det_rows: int, det_cols: int,
                        phimax_deg: float, v0: int, v1: int) -> CSR:
    """Rows of views [v0, v1) of siddon_tilted (a contiguous block of its view-major rows,
    bit-identical to that block of the full matrix): one rank's part of a view-sharded run."""
    L = lib()
    m = (v1 - v0) * det_rows * det_cols
    rp = np.zeros(m + 1, np.int64)
    nnz = L.hx_siddon3d_views(nx, ny, nz, views, det_rows, det_cols, phimax_deg, v0, v1, _p(rp),
                              None, None)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32)
    L.hx_siddon3d_views(nx, ny, nz, views, det_rows, det_cols, phimax_deg, v0, v1, _p(rp), _p(col),
                        _p(val))
    return CSR(m, nx * ny * nz, rp, col, val)


def siddon_sphere(nx: int, ny: int, nz: int, views: int, det_rows: int, det_cols: int) -> CSR:
    """The paper's geometry (f2): parallel beam, view directions on a golden spiral over
    the half sphere, det_rows x det_cols unit pixels; view-major rows."""
    L = lib()
    m = views * det_rows * det_cols
    rp = np.zeros(m + 1, np.int64)
    nnz = L.hx_siddon_sphere(nx, ny, nz, views, det_rows, det_cols, _p(rp), None, None)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32)
    L.hx_siddon_sphere(nx, ny, nz, views, det_rows, det_cols, _p(rp), _p(col), _p(val))
    return CSR(m, nx * ny * nz, rp, col, val)


# ----------------------------------------------------------- vectors (C17)
def phantom(nx: int, ny: int, nz: int, n_ell: int, seed: int = SEED_PHANTOM) -> np.ndarray:
    out = np.empty(nx * ny * nz, np.float32)
    lib().hx_phantom(nx, ny, nz, n_ell, seed, _p(out))
    return out


def uniform(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().hx_uniform(n, seed, _p(out))
    return out


def normal(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().hx_normal(n, seed, _p(out))
    return out


def random_x(n: int, seed: int = SEED_X) -> np.ndarray:
    """Test point x ~ U[0,1) rounded to fp32 (SURVEY §8(d) c2 'x a random nonnegative vector')."""
    return uniform(n, seed).astype(np.float32)


def simulate_data(A: CSR, x_true: np.ndarray, noise_rel: float = 0.01,
                  seed: int = SEED_NOISE) -> np.ndarray:
    """b = A x_true + e, e ~ N(0, sigma^2) i.i.d. over all m rows,
    sigma = noise_rel*||A x_true||_2/sqrt(m) (C16; Eq.(11)).  Returns fp32."""
    y = np.empty(A.n_rows, np.float64)
    lib().hx_simulate_projections(A.n_rows, _p(A.row_ptr), _p(A.col), _p(A.val),
                                  _p(np.ascontiguousarray(x_true, np.float32)), _p(y))
    sigma = noise_rel * np.linalg.norm(y) / np.sqrt(A.n_rows)
    e = sigma * normal(A.n_rows, seed)
    return (y + e).astype(np.float32)


# ---------------------------------------------------------- workload presets
@dataclass
class Workload:
    name: str
    grid: tuple            # (nx, ny, nz)
    A: CSR
    b: np.ndarray
    x_true: np.ndarray
    alpha: float = 0.01
    tau: float = 1e-4
    lo: float = 0.0
    hi: float = float("inf")
    geometry: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        nx, ny, nz = self.grid
        return nx * ny * nz


# BASELINE.json configs (BJ:7-11)
PRESETS = {
    "c1": dict(grid=(32, 32, 32), views=12, bins=45, n_ell=6),
    "c2": dict(grid=(128, 128, 128), views=60, bins=181, n_ell=6),
    "c3": dict(grid=(256, 256, 256), views=90, bins=363, n_ell=10),
    "c4": dict(grid=(256, 256, 256), views=90, bins=363, n_ell=10, hi=1.0),
    "c5": dict(grid=(256, 256, 256), views=120, det=(256, 363), tilt=10.0, n_ell=10),
    # the paper's own experiment shape: 64^3, 55 / 19 views of 91^2
    "f2many": dict(grid=(64, 64, 64), views=55, det=(91, 91), sphere=True, n_ell=10),
    "f2few": dict(grid=(64, 64, 64), views=19, det=(91, 91), sphere=True, n_ell=10),
}


def separable_workload(name: str, grid, views: int, bins: int, n_ell: int,
                       alpha: float = 0.01, tau: float = 1e-4, lo: float = 0.0,
                       hi: float = float("inf"), noise_rel: float = 0.01) -> Workload:
    nx, ny, nz = grid
    A = siddon_separable(nx, ny, nz, views, bins)
    xt = phantom(nx, ny, nz, n_ell)
    b = simulate_data(A, xt, noise_rel)
    return Workload(name, (nx, ny, nz), A, b, xt, alpha, tau, lo, hi,
                    dict(kind="separable", views=views, bins=bins))


@dataclass
class SlabWorkload:
    """One rank's part of a weak-scaled slice-separable workload: the preset's volume repeated
    `world` times along z (global grid nx x ny x (nz world)); this rank owns slices [z0, z1) and
    their rows, columns global."""
    grid: tuple
    z0: int
    z1: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    b: np.ndarray
    alpha: float
    tau: float
    lo: float
    hi: float


def weak_slab(name: str, world: int, rank: int) -> SlabWorkload:
    """Rank `rank`'s slab of preset `name` weak-scaled over `world` ranks (separable presets):
    the phantom is drawn on the tall volume, the noise seed differs per rank."""
    p = dict(PRESETS[name])
    nx, ny, nz = p["grid"]
    A = siddon_separable(nx, ny, nz, p["views"], p["bins"])
    z0, z1 = rank * nz, (rank + 1) * nz
    plane = nx * ny
    xt = phantom(nx, ny, nz * world, p["n_ell"])[z0 * plane:z1 * plane]
    b = simulate_data(A, xt, seed=SEED_NOISE + 1000 * rank)
    col = (A.col.astype(np.int64) + z0 * plane).astype(np.int32)
    return SlabWorkload((nx, ny, nz * world), z0, z1, A.row_ptr, col, A.val, b,
                        p.get("alpha", 0.01), p.get("tau", 1e-4), p.get("lo", 0.0),
                        p.get("hi", float("inf")))


def _balanced(n: int, world: int, rank: int):
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def strong_slab(name: str, world: int, rank: int) -> SlabWorkload:
    """Rank `rank`'s part of preset `name` (slice-separable) split over `world` ranks by z-slabs
    (strong scaling): slices [z0, z1) (balanced) and exactly the rows of
    preset(name) that touch them, with global columns, and the same b (the projections are
    simulated slice by slice with the same per-row sums, so sigma and every row of b equal the
    single-process workload's).  Only the rank's rows of A are built."""
    p = dict(PRESETS[name])
    nx, ny, nz = p["grid"]
    As = siddon_slice(nx, ny, p["views"], p["bins"])
    z0, z1 = _balanced(nz, world, rank)
    plane, ms = nx * ny, As.n_rows
    xt = np.ascontiguousarray(phantom(nx, ny, nz, p["n_ell"]), np.float32)
    y = np.empty(ms * nz, np.float64)
    for z in range(nz):
        lib().hx_simulate_projections(ms, _p(As.row_ptr), _p(As.col), _p(As.val),
                                      _p(np.ascontiguousarray(xt[z * plane:(z + 1) * plane])),
                                      _p(y[z * ms:(z + 1) * ms]))
    sigma = 0.01 * np.linalg.norm(y) / np.sqrt(len(y))
    e = normal(len(y), SEED_NOISE)
    b = (y[z0 * ms:z1 * ms] + sigma * e[z0 * ms:z1 * ms]).astype(np.float32)
    nzl = z1 - z0
    rp = np.empty(ms * nzl + 1, np.int64)
    col = np.empty(As.nnz * nzl, np.int32)
    val = np.empty(As.nnz * nzl, np.float32)
    lib().hx_replicate_slices(ms, As.nnz, _p(As.row_ptr), _p(As.col), _p(As.val), plane, nzl,
                              _p(rp), _p(col), _p(val))
    col += np.int32(z0 * plane)
    return SlabWorkload((nx, ny, nz), z0, z1, rp, col, val, b, p.get("alpha", 0.01),
                        p.get("tau", 1e-4), p.get("lo", 0.0), p.get("hi", float("inf")))


@dataclass
class ViewBlock:
    """One rank's part of a view-sharded (P2) workload: views [v0, v1), their rows (global
    columns), the noise-free projections y of those rows, and the rank's z-slab [z0, z1)."""
    grid: tuple
    v0: int
    v1: int
    z0: int
    z1: int
    row0: int
    m_total: int
    A: CSR
    y: np.ndarray
    alpha: float
    tau: float
    lo: float
    hi: float

    def data(self, sum_y2: float, noise_rel: float = 0.01, seed: int = SEED_NOISE) -> np.ndarray:
        """b of the rank's rows given sum_i y_i^2 over ALL rows (e.g. an all-reduce of the ranks'
        partial sums): sigma = noise_rel sqrt(sum y^2 / m), the noise stream of all m rows (C16)."""
        sigma = noise_rel * np.sqrt(sum_y2) / np.sqrt(self.m_total)
        e = normal(self.m_total, seed)[self.row0:self.row0 + self.A.n_rows]
        return (self.y + sigma * e).astype(np.float32)


def views_block(name: str, world: int, rank: int) -> ViewBlock:
    """Rank `rank`'s views of a tilted preset (c5) split over `world` ranks (balanced view ranges,
    slabs balanced like strong_slab); only its rows are traced."""
    p = dict(PRESETS[name])
    nx, ny, nz = p["grid"]
    V, (R, C) = p["views"], p["det"]
    v0, v1 = _balanced(V, world, rank)
    z0, z1 = _balanced(nz, world, rank)
    A = siddon_tilted_views(nx, ny, nz, V, R, C, p["tilt"], v0, v1)
    xt = phantom(nx, ny, nz, p["n_ell"])
    y = np.empty(A.n_rows, np.float64)
    lib().hx_simulate_projections(A.n_rows, _p(A.row_ptr), _p(A.col), _p(A.val),
                                  _p(np.ascontiguousarray(xt, np.float32)), _p(y))
    return ViewBlock((nx, ny, nz), v0, v1, z0, z1, v0 * R * C, V * R * C, A, y,
                     p.get("alpha", 0.01), p.get("tau", 1e-4), p.get("lo", 0.0),
                     p.get("hi", float("inf")))


def preset(name: str, **over) -> Workload:
    p = dict(PRESETS[name])
    p.update(over)
    if p.get("sphere"):
        nx, ny, nz = p["grid"]
        A = siddon_sphere(nx, ny, nz, p["views"], p["det"][0], p["det"][1])
        xt = phantom(nx, ny, nz, p["n_ell"])
        b = simulate_data(A, xt)
        return Workload(name, p["grid"], A, b, xt, p.get("alpha", 0.01), p.get("tau", 1e-4),
                        p.get("lo", 0.0), p.get("hi", float("inf")),
                        dict(kind="sphere", views=p["views"], det=p["det"]))
    if "det" in p:
        nx, ny, nz = p["grid"]
        A = siddon_tilted(nx, ny, nz, p["views"], p["det"][0], p["det"][1], p["tilt"])
        xt = phantom(nx, ny, nz, p["n_ell"])
        b = simulate_data(A, xt)
        return Workload(name, p["grid"], A, b, xt, p.get("alpha", 0.01), p.get("tau", 1e-4),
                        p.get("lo", 0.0), p.get("hi", float("inf")),
                        dict(kind="tilted", views=p["views"], det=p["det"], tilt=p["tilt"]))
    return separable_workload(name, p["grid"], p["views"], p["bins"], p["n_ell"],
                              p.get("alpha", 0.01), p.get("tau", 1e-4), p.get("lo", 0.0),
                              p.get("hi", float("inf")))


def sliced_preset(name: str, **over) -> Workload:
    """A slice-separable preset (c1-c4) with ONE slice's matrix in `A` (nx*ny columns) for the
    slice-shared operator (tvr_create_sliced): the operator is I_nz (x) A.  b and x_true
    are those of preset(name) (the projections are simulated slice by slice, same rows, same
    noise), without building the nz-times larger CSR."""
    p = dict(PRESETS[name])
    p.update(over)
    if p.get("sphere") or "det" in p:
        raise ValueError(f"{name}: not slice-separable")
    nx, ny, nz = p["grid"]
    As = siddon_slice(nx, ny, p["views"], p["bins"])
    xt = np.ascontiguousarray(phantom(nx, ny, nz, p["n_ell"]), np.float32)
    plane, ms = nx * ny, As.n_rows
    y = np.empty(ms * nz, np.float64)
    for z in range(nz):
        lib().hx_simulate_projections(ms, _p(As.row_ptr), _p(As.col), _p(As.val),
                                      _p(np.ascontiguousarray(xt[z * plane:(z + 1) * plane])),
                                      _p(y[z * ms:(z + 1) * ms]))
    sigma = 0.01 * np.linalg.norm(y) / np.sqrt(len(y))
    b = (y + sigma * normal(len(y), SEED_NOISE)).astype(np.float32)
    return Workload(name, (nx, ny, nz), As, b, xt, p.get("alpha", 0.01), p.get("tau", 1e-4),
                    p.get("lo", 0.0), p.get("hi", float("inf")),
                    dict(kind="sliced", views=p["views"], bins=p["bins"]))
