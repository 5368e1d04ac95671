"""Thin ctypes binding of libtvreg (include/libtvreg.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libtvreg.so; this module never
computes anything itself and has no CPU fallback: if the shared library is missing it raises.
Device vectors are passed as torch CUDA tensors (their data_ptr()) or raw integer pointers.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# TVR_LIB_PATH: load another in-tree build (A/B timing of kernel revisions); default libtvreg.so
LIB_PATH = os.environ.get("TVR_LIB_PATH") or os.path.join(_PKG, "libtvreg.so")

# ---------------------------------------------------------------- status codes
TVR_OK = 0
TVR_NOT_CONVERGED = 1
TVR_E_ARG = -1
TVR_E_CSR = -2
TVR_E_NOT_SEPARABLE = -3
TVR_E_CUDA = -4
TVR_E_NCCL = -5
TVR_E_OOM = -6
TVR_E_NONFINITE = -7
TVR_E_LINESEARCH = -8
TVR_E_THETA = -9
STATUS_NAMES = {v: k for k, v in globals().items() if k.startswith("TVR_") and isinstance(v, int)}

TVR_SHARD_NONE = 0
TVR_SHARD_ZSLAB = 1
TVR_SHARD_VIEWS = 2
TVR_SHARD_VIEWS_REP = 3
TVR_CONTROL_HOST = 0
TVR_CONTROL_DEVICE = 1
TVR_CONTROL_AUTO = 2
TVR_STOP_REL = 0
TVR_STOP_ABS_PER_N = 1

c_i32, c_i64, c_f64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class tvr_csr(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("n_cols", c_i64), ("nnz", c_i64),
                ("row_ptr", c_vp), ("col_idx", c_vp), ("val", c_vp)]


class tvr_grid(ctypes.Structure):
    _fields_ = [("nx", c_i32), ("ny", c_i32), ("nz", c_i32)]


class tvr_dist(ctypes.Structure):
    _fields_ = [("world", c_i32), ("rank", c_i32), ("mode", c_i32), ("z0", c_i32), ("z1", c_i32),
                ("nccl_comm", c_vp), ("device", c_i32), ("cuda_stream", c_vp)]


class tvr_info(ctypes.Structure):
    _fields_ = [("m_local", c_i64), ("n_local", c_i64), ("nnz_local", c_i64), ("z0", c_i32),
                ("z1", c_i32), ("slab_staged_A", c_i32), ("slab_staged_AT", c_i32),
                ("device_bytes", c_i64), ("n_cols_local", c_i64), ("views_fused_rs", c_i32),
                ("slice_shared", c_i32), ("views_rep", c_i32), ("point_allgathers", c_i64),
                ("gather_layout_blocks", c_i64 * 3), ("dist_graph_solves", c_i64),
                ("dist_graph_exchanges", c_i64)]


class tvr_fparts(ctypes.Structure):
    _fields_ = [("fidelity", c_f64), ("tv", c_f64), ("f", c_f64)]


class tvr_gpbb_opts(ctypes.Structure):
    _fields_ = [("max_iters", c_i64), ("eps", c_f64), ("stop_mode", c_i32), ("K", c_i32),
                ("sigma", c_f64), ("beta0", c_f64), ("beta_min", c_f64)]


class tvr_upn_opts(ctypes.Structure):
    _fields_ = [("max_iters", c_i64), ("eps", c_f64), ("stop_mode", c_i32), ("L0", c_f64),
                ("mu0", c_f64), ("rho_L", c_f64), ("bt_max", c_i32)]


class tvr_gp_opts(ctypes.Structure):
    _fields_ = [("max_iters", c_i64), ("eps", c_f64), ("stop_mode", c_i32), ("L0", c_f64),
                ("rho_L", c_f64), ("bt_max", c_i32)]


class tvr_record(ctypes.Structure):
    _fields_ = [("iter", c_i64), ("f", c_f64), ("gmap_rel", c_f64), ("gmap_abs_per_n", c_f64),
                ("step_or_inv_L", c_f64), ("mu", c_f64), ("L", c_f64), ("ls_trials", c_i32),
                ("_pad", c_i32)]


class tvr_result(ctypes.Structure):
    _fields_ = [("converged", c_i32), ("_pad", c_i32), ("iters", c_i64), ("n_f", c_i64),
                ("n_grad", c_i64), ("n_ls", c_i64), ("n_records", c_i64), ("f", c_f64), ("gmap_rel", c_f64),
                ("gmap_abs_per_n", c_f64), ("gmap_ref", c_f64), ("seconds", c_f64),
                ("bytes", c_f64)]


class tvr_kernel_stat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", c_i64), ("total_ms", c_f64),
                ("bytes", c_f64)]


ALLOC_FN = ctypes.CFUNCTYPE(c_vp, ctypes.c_size_t, ctypes.c_int, c_vp, c_vp)
FREE_FN = ctypes.CFUNCTYPE(None, c_vp, ctypes.c_int, c_vp, c_vp)

# name -> (restype, argtypes): every symbol include/libtvreg.h declares
SIGNATURES = {
    "tvr_create": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(tvr_csr), c_vp, tvr_grid,
                                  c_f64, c_f64, c_f64, c_f64, ctypes.POINTER(tvr_dist)]),
    "tvr_create_sliced": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(tvr_csr), c_vp,
                                         tvr_grid, c_f64, c_f64, c_f64, c_f64,
                                         ctypes.POINTER(tvr_dist)]),
    "tvr_destroy": (None, [c_vp]),
    "tvr_get_info": (ctypes.c_int, [c_vp, ctypes.POINTER(tvr_info)]),
    "tvr_objective_grad": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(c_f64), c_vp,
                                          ctypes.POINTER(tvr_fparts)]),
    "tvr_objective_grad_host": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(c_f64), c_vp,
                                               ctypes.POINTER(tvr_fparts)]),
    "tvr_gpbb_default": (None, [ctypes.POINTER(tvr_gpbb_opts)]),
    "tvr_upn_default": (None, [ctypes.POINTER(tvr_upn_opts)]),
    "tvr_gp_default": (None, [ctypes.POINTER(tvr_gp_opts)]),
    "tvr_solve_gpbb": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(tvr_gpbb_opts),
                                      ctypes.POINTER(tvr_result), ctypes.POINTER(tvr_record), c_i64]),
    "tvr_solve_upn": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(tvr_upn_opts),
                                     ctypes.POINTER(tvr_result), ctypes.POINTER(tvr_record), c_i64]),
    "tvr_solve_gp": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(tvr_gp_opts),
                                     ctypes.POINTER(tvr_result), ctypes.POINTER(tvr_record), c_i64]),
    "tvr_residual": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(c_f64)]),
    "tvr_set_control": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "tvr_apply_AT": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "tvr_apply_A": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "tvr_tv": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(c_f64), c_vp]),
    "tvr_gradient_map": (ctypes.c_int, [c_vp, c_vp, c_f64, ctypes.POINTER(c_f64), c_vp]),
    "tvr_get_AT": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "tvr_profile_enable": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "tvr_profile_get": (ctypes.c_int, [c_vp, ctypes.POINTER(tvr_kernel_stat), ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int)]),
    "tvr_launch_count": (c_i64, [c_vp, ctypes.c_int]),
    "tvr_nccl_unique_id_size": (ctypes.c_int, []),
    "tvr_nccl_get_unique_id": (ctypes.c_int, [c_vp]),
    "tvr_nccl_comm_init": (ctypes.c_int, [ctypes.POINTER(c_vp), c_vp, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int]),
    "tvr_nccl_comm_destroy": (ctypes.c_int, [c_vp]),
    "tvr_rank_sum": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp]),
    "tvr_sell_partition": (ctypes.c_int, [c_vp, c_vp, c_i64, ctypes.c_int, ctypes.c_int, c_f64,
                                          c_f64, c_f64, c_vp]),
    "tvr_local_comm_create": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.c_int]),
    "tvr_local_comm_destroy": (ctypes.c_int, [c_vp]),
    "tvr_set_allocator": (ctypes.c_int, [ALLOC_FN, FREE_FN, c_vp]),
    "tvr_last_error": (ctypes.c_char_p, []),
    "tvr_abi_version": (ctypes.c_int, []),
}

_lib = None


def lib():
    """Load libtvreg.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libtvreg.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            try:
                fn = getattr(L, name)
            except AttributeError:
                if LIB_PATH.endswith("libtvreg.so"):
                    raise
                continue  # an older A/B build (TVR_LIB_PATH) without this entry point
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class TVRError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().tvr_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(status: int, where: str, allow=(TVR_OK,)):
    if status not in allow:
        raise TVRError(status, where)
    return status


def _ptr(t) -> int:
    """Device/host pointer of a torch tensor, numpy array or raw int."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


# -------------------------------------------------------------- torch allocator
_alloc_refs = None


def use_torch_allocator(on: bool = True):
    """Route libtvreg device allocations through the PyTorch caching allocator."""
    global _alloc_refs
    import torch
    L = lib()
    if not on:
        _check(L.tvr_set_allocator(ALLOC_FN(), FREE_FN(), None), "tvr_set_allocator")
        _alloc_refs = None
        return

    def _alloc(size, device, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(size), device=int(device),
                                                      stream=int(stream) if stream else None)
        except Exception:
            return None

    def _free(ptr, device, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    _alloc_refs = (ALLOC_FN(_alloc), FREE_FN(_free))
    _check(L.tvr_set_allocator(_alloc_refs[0], _alloc_refs[1], None), "tvr_set_allocator")


# ------------------------------------------------------------------ NCCL bootstrap
def nccl_unique_id() -> bytes:
    n = lib().tvr_nccl_unique_id_size()
    buf = ctypes.create_string_buffer(n)
    _check(lib().tvr_nccl_get_unique_id(buf), "tvr_nccl_get_unique_id")
    return buf.raw


def nccl_comm_init(uid: bytes, world: int, rank: int, device: int) -> int:
    comm = c_vp()
    _check(lib().tvr_nccl_comm_init(ctypes.byref(comm), uid, world, rank, device),
           "tvr_nccl_comm_init")
    return comm.value


def nccl_comm_destroy(comm: int):
    _check(lib().tvr_nccl_comm_destroy(comm), "tvr_nccl_comm_destroy")


def rank_sum(gathered_dev: int, world: int, n: int, out_dev: int, stream: int | None = None):
    """tvr_rank_sum: out[s] = rank-ordered sum of gathered[r * n + s] on the device (device
    pointers as ints)."""
    _check(lib().tvr_rank_sum(gathered_dev, world, n, out_dev, stream), "tvr_rank_sum")


def sell_partition(blk_steps, blk_slice, nwarps: int, grid: int, blk_cost: float = 2.0,
                   seg_cost: float = 3.0, lam: float = 0.5) -> np.ndarray:
    """tvr_sell_partition (host only): CTA block ranges of a sliced-ELL pass."""
    k = np.ascontiguousarray(blk_steps, np.int32)
    sl = np.ascontiguousarray(blk_slice, np.int32)
    tab = np.empty(grid + 1, np.int64)
    _check(lib().tvr_sell_partition(k.ctypes.data, sl.ctypes.data, len(k), nwarps, grid, blk_cost,
                                    seg_cost, lam, tab.ctypes.data), "tvr_sell_partition")
    return tab


def local_comm_create(world: int) -> int:
    """In-process thread communicator: ranks are threads of this process (tests of the
    multi-rank paths on one GPU; see include/libtvreg.h)."""
    comm = c_vp()
    _check(lib().tvr_local_comm_create(ctypes.byref(comm), world), "tvr_local_comm_create")
    return comm.value


def local_comm_destroy(comm: int):
    _check(lib().tvr_local_comm_destroy(comm), "tvr_local_comm_destroy")


# ----------------------------------------------------------------------- problem
@dataclass
class SolveResult:
    status: int
    converged: bool
    iters: int
    n_f: int
    n_grad: int
    n_ls: int
    f: float
    gmap_rel: float
    gmap_abs_per_n: float
    gmap_ref: float
    seconds: float
    bytes: float
    history: list


class Problem:
    """tvr_problem handle.  A: CSR (row_ptr int64, col int32 global voxel ids, val fp32) of this
    rank's rows (host arrays); b: fp32 host vector of the same rows."""

    def __init__(self, row_ptr, col, val, b, grid, alpha: float, tau: float, lo: float = 0.0,
                 hi: float = math.inf, *, n_cols: int | None = None, world: int = 1, rank: int = 0,
                 z0: int | None = None, z1: int | None = None, nccl_comm: int | None = None,
                 device: int = -1, stream: int | None = None, shard: str | None = None,
                 sliced: bool = False):
        """shard: None (ZSLAB when world > 1 or z0 is given, else NONE), "zslab", "views" or
        "views_rep" (VIEWS with the solvers' volume vectors replicated on every rank)
        (rows of any geometry, global columns; see tvr_dist in include/libtvreg.h).
        sliced: the CSR is ONE slice's matrix (n_cols = nx*ny) applied to every slice of the
        slab, b has m_s * slab-slices entries (tvr_create_sliced)."""
        L = lib()
        self._keep = [np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                      np.ascontiguousarray(val, np.float32), np.ascontiguousarray(b, np.float32)]
        rp, cl, vl, bb = self._keep
        nx, ny, nz = grid
        self.grid = (nx, ny, nz)
        if n_cols is None:
            n_cols = nx * ny if sliced else nx * ny * nz
        csr = tvr_csr(len(rp) - 1, n_cols, int(rp[-1]), rp.ctypes.data, cl.ctypes.data,
                      vl.ctypes.data)
        dist = None
        if shard is None:
            mode = TVR_SHARD_ZSLAB if (world > 1 or z0 is not None) else TVR_SHARD_NONE
        else:
            mode = {"none": TVR_SHARD_NONE, "zslab": TVR_SHARD_ZSLAB, "views": TVR_SHARD_VIEWS,
                    "views_rep": TVR_SHARD_VIEWS_REP}[shard]
        if mode != TVR_SHARD_NONE or stream is not None or device >= 0:
            dist = tvr_dist(world, rank, mode,
                            0 if z0 is None else z0, nz if z1 is None else z1,
                            nccl_comm, device, stream)
        h = c_vp()
        create = L.tvr_create_sliced if sliced else L.tvr_create
        _check(create(ctypes.byref(h), ctypes.byref(csr), bb.ctypes.data,
                      tvr_grid(nx, ny, nz), alpha, tau, lo, hi,
                      ctypes.byref(dist) if dist is not None else None), create.__name__)
        self._h = h
        self._keep = None  # host arrays are copied by tvr_create
        info = tvr_info()
        _check(L.tvr_get_info(h, ctypes.byref(info)), "tvr_get_info")
        self.info = info
        self.m = info.m_local
        self.n = info.n_local
        self.nnz = info.nnz_local
        self.alpha, self.tau, self.lo, self.hi = alpha, tau, lo, hi

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tvr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- gradient evaluation
    def objective_grad(self, x, g=None):
        f = c_f64()
        parts = tvr_fparts()
        _check(lib().tvr_objective_grad(self._h, _ptr(x), ctypes.byref(f), _ptr(g),
                                        ctypes.byref(parts)), "tvr_objective_grad")
        return f.value, (parts.fidelity, parts.tv)

    def objective_grad_host(self, x_host: np.ndarray, g_host: np.ndarray | None = None):
        f = c_f64()
        parts = tvr_fparts()
        _check(lib().tvr_objective_grad_host(self._h, _ptr(x_host), ctypes.byref(f), _ptr(g_host),
                                             ctypes.byref(parts)), "tvr_objective_grad_host")
        return f.value, (parts.fidelity, parts.tv)

    def residual(self, x, r):
        fid = c_f64()
        _check(lib().tvr_residual(self._h, _ptr(x), _ptr(r), ctypes.byref(fid)), "tvr_residual")
        return fid.value

    def apply_A(self, x, y):
        """y = A x (tvr_apply_A)."""
        _check(lib().tvr_apply_A(self._h, _ptr(x), _ptr(y)), "tvr_apply_A")

    def apply_AT(self, y, w):
        _check(lib().tvr_apply_AT(self._h, _ptr(y), _ptr(w)), "tvr_apply_AT")

    def tv(self, x, grad=None):
        v = c_f64()
        _check(lib().tvr_tv(self._h, _ptr(x), ctypes.byref(v), _ptr(grad)), "tvr_tv")
        return v.value

    def gradient_map(self, x, nu: float, G=None):
        v = c_f64()
        _check(lib().tvr_gradient_map(self._h, _ptr(x), nu, ctypes.byref(v), _ptr(G)),
               "tvr_gradient_map")
        return v.value

    def get_AT(self):
        """The stored transposed CSR (of the slice matrix for a slice-shared problem)."""
        s = self.info.slice_shared
        rows = self.grid[0] * self.grid[1] if s else self.info.n_cols_local
        nnz = self.nnz // s if s else self.nnz
        rp = np.empty(rows + 1, np.int64)
        cl = np.empty(nnz, np.int32)
        vl = np.empty(nnz, np.float32)
        _check(lib().tvr_get_AT(self._h, rp.ctypes.data, cl.ctypes.data, vl.ctypes.data), "tvr_get_AT")
        return rp, cl, vl

    # ---- solvers
    def set_control(self, mode: str):
        """Solver control: "device" (one CUDA graph per solve), "host", or "auto" (default: device
        below 2^28 matrix entries); SURVEY f3."""
        _check(lib().tvr_set_control(self._h, {"host": TVR_CONTROL_HOST, "device": TVR_CONTROL_DEVICE,
                                               "auto": TVR_CONTROL_AUTO}[mode]), "tvr_set_control")

    def _solve(self, fn, opts, x, hist_cap):
        res = tvr_result()
        hist = (tvr_record * hist_cap)() if hist_cap else None
        st = fn(self._h, _ptr(x), ctypes.byref(opts), ctypes.byref(res), hist, hist_cap)
        _check(st, fn.__name__, allow=(TVR_OK, TVR_NOT_CONVERGED))
        h = []
        for i in range(min(hist_cap, res.n_records) if hist_cap else 0):
            r = hist[i]
            h.append(dict(iter=r.iter, f=r.f, gmap_rel=r.gmap_rel, gmap_abs_per_n=r.gmap_abs_per_n,
                          step=r.step_or_inv_L, mu=r.mu, L=r.L, trials=r.ls_trials))
        return SolveResult(st, bool(res.converged), res.iters, res.n_f, res.n_grad, res.n_ls, res.f,
                           res.gmap_rel, res.gmap_abs_per_n, res.gmap_ref, res.seconds, res.bytes, h)

    def solve_gpbb(self, x, max_iters=10000, eps=1e-6, stop_mode=TVR_STOP_REL, K=2, sigma=0.1,
                   beta0=0.95, beta_min=1e-10, hist_cap=0) -> SolveResult:
        o = tvr_gpbb_opts(max_iters, eps, stop_mode, K, sigma, beta0, beta_min)
        return self._solve(lib().tvr_solve_gpbb, o, x, hist_cap)

    def solve_upn(self, x, max_iters=10000, eps=1e-6, stop_mode=TVR_STOP_REL, L0=1.0, mu0=None,
                  rho_L=1.3, bt_max=200, hist_cap=0) -> SolveResult:
        o = tvr_upn_opts(max_iters, eps, stop_mode, L0, L0 if mu0 is None else mu0, rho_L, bt_max)
        return self._solve(lib().tvr_solve_upn, o, x, hist_cap)

    def solve_gp(self, x, max_iters=10000, eps=1e-6, stop_mode=TVR_STOP_REL, L0=1.0, rho_L=1.3,
                 bt_max=200, hist_cap=0) -> SolveResult:
        """Gradient projection with BT steps (the paper's comparator, Eq. (6))."""
        o = tvr_gp_opts(max_iters, eps, stop_mode, L0, rho_L, bt_max)
        return self._solve(lib().tvr_solve_gp, o, x, hist_cap)

    def get_info(self) -> tvr_info:
        """tvr_get_info now (self.info is the snapshot taken at creation)."""
        info = tvr_info()
        _check(lib().tvr_get_info(self._h, ctypes.byref(info)), "tvr_get_info")
        return info

    # ---- timing
    def profile(self, on: bool = True):
        _check(lib().tvr_profile_enable(self._h, 1 if on else 0), "tvr_profile_enable")

    def kernel_stats(self) -> dict:
        arr = (tvr_kernel_stat * 16)()
        n = ctypes.c_int()
        _check(lib().tvr_profile_get(self._h, arr, 16, ctypes.byref(n)), "tvr_profile_get")
        return {arr[i].name.decode(): dict(launches=arr[i].launches, ms=arr[i].total_ms,
                                           bytes=arr[i].bytes) for i in range(n.value)}

    def launch_count(self, reset: bool = False) -> int:
        return int(lib().tvr_launch_count(self._h, 1 if reset else 0))
