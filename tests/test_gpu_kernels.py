"""Kernel parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element
(SURVEY.md §8(c).4).  Bars: bit-exact for the transposed CSR index arrays and for dyadic-exact
SpMV inputs; relative L2 <= 1e-6 for single passes (fp32 output rounding is 6e-8); <= 1e-5 for a
full gradient (BASELINE.json north_star)."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def make(T, A, b, grid, alpha=0.01, tau=1e-4, lo=0.0, hi=math.inf):
    return T.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau, lo, hi)


# ------------------------------------------------------------------ a3: A^T
@pytest.mark.parametrize("which", ["c1", "random_ragged", "tilted", "sphere"])
def test_transpose_bit_exact(tvreg, which, c1):
    if which == "c1":
        A, grid = c1.A, c1.grid
    elif which == "random_ragged":
        A, grid = random_csr(301, 7 * 5 * 3, 0.2, seed=3, empty_rows=11), (7, 5, 3)
    elif which == "sphere":
        A, grid = harness.siddon_sphere(14, 12, 10, 9, 19, 21), (14, 12, 10)
    else:
        A, grid = harness.siddon_tilted(12, 10, 9, 7, 9, 13, 10.0), (12, 10, 9)
    P = make(tvreg, A, np.zeros(A.n_rows, np.float32), grid)
    rT, cT, vT = P.get_AT()
    oT = oracle.transpose(A.row_ptr, A.col, A.val, A.n_cols)
    assert np.array_equal(rT, oT[0])
    assert np.array_equal(cT, oT[1])
    assert np.array_equal(vT.view(np.uint32), oT[2].view(np.uint32))


def test_transpose_bit_exact_c2(tvreg):
    A = harness.siddon_separable(128, 128, 128, 60, 181)
    P = make(tvreg, A, np.zeros(A.n_rows, np.float32), (128, 128, 128))
    assert P.info.slab_staged_A >= 1 and P.info.slab_staged_AT >= 1
    rT, cT, vT = P.get_AT()
    oT = oracle.transpose(A.row_ptr, A.col, A.val, A.n_cols)
    assert np.array_equal(rT, oT[0]) and np.array_equal(cT, oT[1])
    assert np.array_equal(vT.view(np.uint32), oT[2].view(np.uint32))


# --------------------------------------------------------------- a1 / a2
def _dyadic_separable(nx, ny, nz, V, nb):
    A = harness.siddon_separable(nx, ny, nz, V, nb)
    A.val = (np.maximum(1, np.rint(A.val.astype(np.float64) * 1024)) / 1024).astype(np.float32)
    return A


@pytest.mark.parametrize("kind", ["separable", "random"])
def test_spmv_dyadic_bitwise(tvreg, kind):
    """Values k/1024 and integer vectors in [0, 8]: every partial sum is exact, so the GPU's
    r = Ax - b and w = A^T r must equal the oracle bitwise in any summation order (App. A.4)."""
    rng = np.random.default_rng(1)
    if kind == "separable":
        A, grid = _dyadic_separable(40, 24, 6, 9, 31), (40, 24, 6)
    else:
        A, grid = random_csr(500, 9 * 8 * 7, 0.05, seed=2, dyadic=True, empty_rows=9), (9, 8, 7)
    x = rng.integers(0, 9, A.n_cols).astype(np.float32)
    b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    P = make(tvreg, A, b, grid)
    r = torch.empty(A.n_rows, device="cuda")
    fid = P.residual(dev(x), r)
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x) - b
    assert np.array_equal(host(r).astype(np.float64), r_ora)
    assert fid == 0.5 * float(r_ora @ r_ora)
    y = rng.integers(0, 9, A.n_rows).astype(np.float32)
    w = torch.empty(A.n_cols, device="cuda")
    P.apply_AT(dev(y), w)
    w_ora = oracle.rmatvec(A.row_ptr, A.col, A.val, y, A.n_cols)
    assert np.array_equal(host(w).astype(np.float64), w_ora)


@pytest.mark.parametrize("cfg", ["c1", "ragged", "random"])
def test_spmv_real_values(tvreg, cfg, c1):
    rng = np.random.default_rng(4)
    if cfg == "c1":
        A, grid = c1.A, c1.grid
    elif cfg == "ragged":
        A, grid = harness.siddon_separable(37, 29, 11, 13, 47), (37, 29, 11)
    else:
        A, grid = random_csr(700, 10 * 9 * 8, 0.1, seed=5, empty_rows=20), (10, 9, 8)
    x = rng.random(A.n_cols).astype(np.float32)
    b = rng.random(A.n_rows).astype(np.float32)
    P = make(tvreg, A, b, grid)
    r = torch.empty(A.n_rows, device="cuda")
    fid = P.residual(dev(x), r)
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x) - b
    assert rel(host(r), r_ora) <= 1e-6
    assert abs(fid - 0.5 * r_ora @ r_ora) <= 1e-12 * (0.5 * r_ora @ r_ora)
    empty = np.diff(A.row_ptr) == 0
    if empty.any():   # rays that miss the volume: r_i = -b_i exactly
        assert np.array_equal(host(r)[empty], -b[empty])
    w = torch.empty(A.n_cols, device="cuda")
    P.apply_AT(dev(b), w)
    assert rel(host(w), oracle.rmatvec(A.row_ptr, A.col, A.val, b, A.n_cols)) <= 1e-6


# -------------------------------------------------------------------- TV
# row-tiled stencil (K voxels per lane, 7 owned rows per tile): K = 1 (32, 31, 1, 2 wide),
# K = 2 (64), K = 4 (128 with ragged tiles, 100 and 96 with idle lanes), K = 8 (256, 200);
# the 32x8 xy-tile kernel where K does not divide nx (37)
@pytest.mark.parametrize("grid", [(32, 32, 32), (37, 29, 19), (31, 7, 16), (1, 1, 5), (64, 3, 2),
                                  (2, 1, 1), (128, 20, 9), (100, 15, 7), (96, 8, 3), (256, 9, 5),
                                  (200, 13, 4)])
@pytest.mark.parametrize("tau", [1e-4, 1e-1])
def test_tv_value_and_gradient(tvreg, grid, tau):
    N = grid[0] * grid[1] * grid[2]
    rng = np.random.default_rng(N)
    x = rng.random(N).astype(np.float32)
    A = random_csr(3, N, 0.5, seed=1)
    P = make(tvreg, A, np.zeros(3, np.float32), grid, tau=tau)
    g = torch.empty(N, device="cuda")
    v = P.tv(dev(x), g)
    v_ora, g_ora = oracle.tv(grid, x, tau)
    assert abs(v - v_ora) <= 1e-12 * max(1.0, abs(v_ora))
    assert rel(host(g), g_ora) <= 1e-6


def test_tv_piecewise_constant_phantom(tvreg):
    """Flat regions (t = 0 < tau: quadratic branch and zero gradient) next to edges."""
    grid = (40, 36, 20)
    x = harness.phantom(*grid, 6)
    A = random_csr(3, x.size, 0.5, seed=1)
    P = make(tvreg, A, np.zeros(3, np.float32), grid, tau=1e-4)
    g = torch.empty(x.size, device="cuda")
    v = P.tv(dev(x), g)
    v_ora, g_ora = oracle.tv(grid, x, 1e-4)
    assert abs(v - v_ora) <= 1e-12 * v_ora
    assert rel(host(g), g_ora) <= 1e-6


# ------------------------------------------------------- full gradient (a1+a2+a4)
def test_objective_grad_c1(tvreg, c1):
    x = harness.random_x(c1.N)
    P = make(tvreg, c1.A, c1.b, c1.grid, c1.alpha, c1.tau)
    g = torch.empty(c1.N, device="cuda")
    f, (fid, tv) = P.objective_grad(dev(x), g)
    Po = oracle.Problem(c1.A.row_ptr, c1.A.col, c1.A.val, c1.b, c1.grid, c1.alpha, c1.tau)
    fo, go = Po.fg(x)
    assert abs(f - fo) <= 1e-10 * fo
    assert rel(host(g), go) <= 1e-5
    # determinism: ten reruns are bitwise identical
    g0 = host(g).copy()
    for _ in range(10):
        f2, _ = P.objective_grad(dev(x), g)
        assert f2 == f and np.array_equal(host(g), g0)
    # host API (e2e path) returns the same numbers
    gh = np.empty(c1.N, np.float32)
    fh, _ = P.objective_grad_host(x, gh)
    assert fh == f and np.array_equal(gh, g0)
    # value-only call
    fv, _ = P.objective_grad(dev(x), None)
    assert fv == f


def test_objective_grad_c2_full_size(tvreg):
    """BJ:8 workload at full size in the bench's launch configuration: relative L2 <= 1e-5."""
    w = harness.preset("c2")
    x = harness.random_x(w.N)
    P = make(tvreg, w.A, w.b, w.grid, w.alpha, w.tau)
    assert P.info.slab_staged_A >= 1 and P.info.slab_staged_AT >= 1
    g = torch.empty(w.N, device="cuda")
    f, (fid, tv) = P.objective_grad(dev(x), g)
    Po = oracle.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, nthreads=8)
    fo, go = Po.fg(x)
    assert abs(f - fo) <= 1e-9 * fo
    assert rel(host(g), go) <= 1e-5
    # separately: A pass and A^T pass at <= 1e-6
    r = torch.empty(w.A.n_rows, device="cuda")
    P.residual(dev(x), r)
    ro = oracle.matvec(w.A.row_ptr, w.A.col, w.A.val, x, 8) - w.b
    assert rel(host(r), ro) <= 1e-6
    wt = torch.empty(w.N, device="cuda")
    P.apply_AT(r, wt)
    rT = oracle.transpose(w.A.row_ptr, w.A.col, w.A.val, w.N)
    assert rel(host(wt), oracle.matvec(*rT, host(r), 8)) <= 1e-6


def test_gradient_map(tvreg, c1):
    x = harness.random_x(c1.N) - 0.3
    P = make(tvreg, c1.A, c1.b, c1.grid, c1.alpha, c1.tau)
    G = torch.empty(c1.N, device="cuda")
    nrm = P.gradient_map(dev(x), 7.0, G)
    Po = oracle.Problem(c1.A.row_ptr, c1.A.col, c1.A.val, c1.b, c1.grid, c1.alpha, c1.tau)
    Go = Po.gradient_map(x.astype(np.float64), 7.0)
    assert rel(host(G), Go) <= 1e-5
    assert abs(nrm - np.linalg.norm(Go)) <= 1e-5 * np.linalg.norm(Go)


@pytest.mark.parametrize("cfg", ["c1", "ragged"])
def test_per_row_kernels_bitwise(tvreg, cfg, c1, monkeypatch):
    """The int32 per-row SpMV with the slice window staged in shared memory and with global
    gathers use the same per-row summation order, so r, 1/2||r||^2 and A^T r agree bitwise; the
    16-bit-column kernel (8-entry chunks) agrees to fp32 rounding."""
    if cfg == "c1":
        A, b, grid = c1.A, c1.b, c1.grid
    else:
        A = harness.siddon_separable(37, 29, 11, 13, 47)
        b = np.random.default_rng(2).random(A.n_rows).astype(np.float32)
        grid = (37, 29, 11)
    x = dev(harness.random_x(A.n_cols))
    outs = {}
    for mode in ("reg", "global", "reg16"):
        monkeypatch.setenv("TVR_SPMV_STAGE", "0" if mode == "global" else "1")
        monkeypatch.setenv("TVR_IDX16", "1" if mode == "reg16" else "0")
        P = make(tvreg, A, b, grid)
        assert P.info.slab_staged_A == {"reg": 1, "global": 0, "reg16": 1}[mode]
        r = torch.empty(A.n_rows, device="cuda")
        fid = P.residual(x, r)
        w = torch.empty(A.n_cols, device="cuda")
        P.apply_AT(r, w)
        outs[mode] = (host(r).copy(), fid, host(w).copy())
        if mode == "reg16":   # the 16-bit device columns expand back to the canonical A^T
            rT, cT, vT = P.get_AT()
            oT = oracle.transpose(A.row_ptr, A.col, A.val, A.n_cols)
            assert np.array_equal(cT, oT[1]) and np.array_equal(rT, oT[0])
        P.close()
    assert np.array_equal(outs["global"][0], outs["reg"][0])
    # the fp64 sum of r^2 is split differently over CTAs: equal to rounding only
    assert abs(outs["global"][1] - outs["reg"][1]) <= 1e-13 * outs["reg"][1]
    assert np.array_equal(outs["global"][2], outs["reg"][2])
    assert rel(outs["reg16"][0], outs["reg"][0]) <= 1e-7
    assert abs(outs["reg16"][1] - outs["reg"][1]) <= 1e-13 * outs["reg"][1]
    assert rel(outs["reg16"][2], outs["reg"][2]) <= 1e-7


def _row_length_zoo(n_cols, seed):
    """Rows of 0, 1, 2, 3, 7, 8, 9, 31, 255, 256, 257 and 600 entries in random order, dyadic
    values: rows inside one chunk, rows ending on chunk / tile edges, rows spanning several
    256-entry tiles, empty rows."""
    rng = np.random.default_rng(seed)
    lens = rng.permutation(np.repeat([0, 1, 2, 3, 7, 8, 9, 31, 255, 256, 257, 600], 6))
    rp, cols, vals = [0], [], []
    for L in lens:
        c = np.sort(rng.choice(n_cols, size=L, replace=False))
        cols.extend(c.tolist())
        vals.extend((rng.integers(1, 2049, size=L) / 1024.0).tolist())
        rp.append(rp[-1] + L)
    return SmallCSR(rp, cols, vals, n_cols)


@pytest.mark.parametrize("cfg", ["c1", "ragged", "zoo"])
def test_spmv_variants_against_oracle(tvreg, cfg, c1, monkeypatch):
    """Every SpMV layout the library can pick for a slice-structured matrix (sliced ELL with the
    staged window, global gathers, int32 columns, the padded per-row kernel) against the oracle:
    bitwise on dyadic data (the zoo of row lengths 0 .. 600: rows inside one chunk, on chunk
    edges, spanning many chunks, empty rows), to fp32 rounding otherwise."""
    rng = np.random.default_rng(11)
    if cfg == "c1":
        A, grid = c1.A, c1.grid
        x = harness.random_x(A.n_cols)
        b = c1.b
    elif cfg == "ragged":
        A, grid = harness.siddon_separable(37, 29, 11, 13, 47), (37, 29, 11)
        x = harness.random_x(A.n_cols)
        b = rng.random(A.n_rows).astype(np.float32)
    else:
        grid = (16, 16, 4)
        A = _row_length_zoo(16 * 16 * 4, 3)
        x = rng.integers(0, 9, A.n_cols).astype(np.float32)
        b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    modes = {"sell": {}, "global": {"TVR_SPMV_STAGE": "0"}, "int32": {"TVR_IDX16": "0"},
             "perrow": {"TVR_SPMV_SELL": "0"}}
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
    w_ora = oracle.rmatvec(A.row_ptr, A.col, A.val, b.astype(np.float64), A.n_cols)
    for mode, env in modes.items():
        for k in ("TVR_SPMV_STAGE", "TVR_IDX16", "TVR_SPMV_SELL"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        P = make(tvreg, A, b, grid)
        r = torch.empty(A.n_rows, device="cuda")
        fid = P.residual(dev(x), r)
        w = torch.empty(A.n_cols, device="cuda")
        P.apply_AT(dev(b), w)
        rh, wh = host(r).astype(np.float64), host(w).astype(np.float64)
        P.close()
        if cfg == "zoo":  # dyadic: exact
            assert np.array_equal(rh, r_ora), mode
            assert np.array_equal(wh, w_ora), mode
            assert fid == 0.5 * float(r_ora @ r_ora), mode
        assert rel(rh, r_ora) <= 1e-6 and rel(wh, w_ora) <= 1e-6, mode


def _separable_zoo(nx, ny, nz, seed):
    """Slice-major rows, each inside one z slice, of 0, 1, 2, 3, 7, 8, 9, 31, 255 and nx*ny
    entries (capped at the slice), dyadic values: row-length mixes for the sliced-ELL blocks
    (empty rows, partial last blocks, rows padded to a longer block neighbour)."""
    rng = np.random.default_rng(seed)
    plane = nx * ny
    rp, cols, vals = [0], [], []
    for z in range(nz):
        lens = rng.permutation(np.repeat([0, 1, 2, 3, 7, 8, 9, 31, min(255, plane), plane], 5))
        for L in lens:
            c = z * plane + np.sort(rng.choice(plane, size=L, replace=False))
            cols.extend(c.tolist())
            vals.extend((rng.integers(1, 2049, size=L) / 1024.0).tolist())
            rp.append(rp[-1] + L)
    return SmallCSR(rp, cols, vals, plane * nz)


@pytest.mark.parametrize("cfg", ["c1", "ragged", "zoo", "zoo_global", "zoo_half"])
def test_sell_spmv(tvreg, cfg, c1, monkeypatch):
    """The sliced-ELL kernel (spmv16s_kernel; the default for slice-structured matrices) against
    the oracle, for both passes: exact on dyadic data (every row length class, empty rows, partial
    blocks; staged, global-gather and partly staged windows), fp32 rounding otherwise; and
    against the padded per-row kernel (TVR_SPMV_SELL=0)."""
    rng = np.random.default_rng(12)
    if cfg == "c1":
        A, grid = c1.A, c1.grid
        x = harness.random_x(A.n_cols)
        b = c1.b
    elif cfg == "ragged":
        A, grid = harness.siddon_separable(37, 29, 11, 13, 47), (37, 29, 11)
        x = harness.random_x(A.n_cols)
        b = rng.random(A.n_rows).astype(np.float32)
    else:
        grid = (16, 16, 4)
        A = _separable_zoo(16, 16, 4, 5)
        x = rng.integers(0, 9, A.n_cols).astype(np.float32)
        b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    if cfg == "zoo_global":
        monkeypatch.setenv("TVR_SPMV_STAGE", "0")
        monkeypatch.setenv("TVR_SPMV_HALF", "0")
    if cfg == "zoo_half":  # 1 KB budget: offsets >= 224 of the 256-entry window from global memory
        monkeypatch.setenv("TVR_SPMV_STAGE", "0")
        monkeypatch.setenv("TVR_SPMV_HALF_KB", "1")
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
    w_ora = oracle.rmatvec(A.row_ptr, A.col, A.val, b.astype(np.float64), A.n_cols)
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("TVR_SPMV_SELL", mode)
        P = make(tvreg, A, b, grid)
        r = torch.empty(A.n_rows, device="cuda")
        fid = P.residual(dev(x), r)
        w = torch.empty(A.n_cols, device="cuda")
        P.apply_AT(dev(b), w)
        outs[mode] = (host(r).astype(np.float64), fid, host(w).astype(np.float64))
        P.close()
    r, fid, w = outs["1"]
    if cfg.startswith("zoo"):
        assert np.array_equal(r, r_ora) and np.array_equal(w, w_ora)
        assert fid == 0.5 * float(r_ora @ r_ora)
    else:
        assert rel(r, r_ora) <= 1e-6 and rel(w, w_ora) <= 1e-6
        assert abs(fid - 0.5 * float(r_ora @ r_ora)) <= 1e-6 * fid
    assert rel(r, outs["0"][0]) <= 1e-7 and rel(w, outs["0"][2]) <= 1e-7


@pytest.mark.parametrize("cfg,floats", [("zoo", "96"), ("zoo", "128"), ("c1", "300"), ("c1", "512")])
def test_sell_column_parts(tvreg, cfg, floats, c1, monkeypatch):
    """Windows larger than shared memory cut into column parts (the c3 A pass): each row's
    entries split at the part boundaries, one sliced-ELL pass per part with the fp64 row sum
    carried between passes; forced here on small windows (TVR_SELL_PART_FLOATS).  Exact on dyadic
    data (rows spanning every part, empty parts), fp32 rounding otherwise, and the e2e pipeline's
    gradient equals the device one."""
    monkeypatch.setenv("TVR_SPMV_STAGE", "0")
    monkeypatch.setenv("TVR_SELL_PART_FLOATS", floats)
    rng = np.random.default_rng(13)
    if cfg == "zoo":
        grid = (16, 16, 4)
        A = _separable_zoo(16, 16, 4, 6)
        x = rng.integers(0, 9, A.n_cols).astype(np.float32)
        b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    else:
        A, grid = c1.A, c1.grid
        x = harness.random_x(A.n_cols)
        b = c1.b
    P = make(tvreg, A, b, grid)
    r = torch.empty(A.n_rows, device="cuda")
    fid = P.residual(dev(x), r)
    w = torch.empty(A.n_cols, device="cuda")
    P.apply_AT(dev(b), w)
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
    w_ora = oracle.rmatvec(A.row_ptr, A.col, A.val, b.astype(np.float64), A.n_cols)
    rr, ww = host(r).astype(np.float64), host(w).astype(np.float64)
    if cfg == "zoo":
        assert np.array_equal(rr, r_ora) and np.array_equal(ww, w_ora)
        assert fid == 0.5 * float(r_ora @ r_ora)
    else:
        assert rel(rr, r_ora) <= 1e-6 and rel(ww, w_ora) <= 1e-6
        assert abs(fid - 0.5 * float(r_ora @ r_ora)) <= 1e-6 * fid
    g = torch.empty(A.n_cols, device="cuda")
    f, _ = P.objective_grad(dev(x), g)
    xh = torch.from_numpy(np.ascontiguousarray(x, np.float32)).pin_memory()
    gh = torch.empty(A.n_cols, dtype=torch.float32).pin_memory()
    fh, _ = P.objective_grad_host(xh.numpy(), gh.numpy())
    assert torch.equal(gh, g.cpu()) and abs(fh - f) <= 1e-13 * abs(f)
    P.close()


@pytest.mark.parametrize("cfg", ["zoo", "sphere", "tilted", "layouts"])
@pytest.mark.parametrize("mode", ["0", "1", "2", "3"])
def test_sell32_spmv(tvreg, cfg, mode, monkeypatch):
    """Int32 sliced ELL for non-separable matrices (spmv32s_kernel; TVR_SPMV_SELL32 = 0 none,
    1 the A^T pass, 2 both in lane mode, 3 the A pass with per-block lane / row modes): exact on
    dyadic data with rows of every length class, the oracle to fp32 rounding on the paper's
    sphere geometry and on tilted rays (c5's geometry)."""
    monkeypatch.setenv("TVR_SPMV_SELL32", mode)
    rng = np.random.default_rng(21)
    if cfg == "zoo":
        grid = (16, 16, 4)
        A = _row_length_zoo(16 * 16 * 4, 9)
        x = rng.integers(0, 9, A.n_cols).astype(np.float32)
        b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    elif cfg == "sphere":
        grid = (24, 24, 24)
        A = harness.siddon_sphere(24, 24, 24, 7, 33, 33)
        x = harness.random_x(A.n_cols)
        b = rng.random(A.n_rows).astype(np.float32)
    elif cfg == "tilted":
        grid = (20, 20, 20)
        A = harness.siddon_tilted(20, 20, 20, 9, 20, 29, 10.0)
        x = harness.random_x(A.n_cols)
        b = rng.random(A.n_rows).astype(np.float32)
    else:  # tilted rays on a grid whose xy planes tile into 8x4 bricks: the gather layouts
        grid = (32, 24, 16)
        A = harness.siddon_tilted(32, 24, 16, 12, 16, 41, 10.0)
        x = harness.random_x(A.n_cols)
        b = rng.random(A.n_rows).astype(np.float32)
    P = make(tvreg, A, b, grid)
    if mode == "3" and cfg == "layouts":  # every layout is chosen by some block of rays
        lb = list(P.info.gather_layout_blocks)
        assert sum(lb) == (A.n_rows + 31) // 32 and min(lb) > 0, lb
    r = torch.empty(A.n_rows, device="cuda")
    fid = P.residual(dev(x), r)
    w = torch.empty(A.n_cols, device="cuda")
    P.apply_AT(dev(b), w)
    P.close()
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
    w_ora = oracle.rmatvec(A.row_ptr, A.col, A.val, b.astype(np.float64), A.n_cols)
    rr, ww = host(r).astype(np.float64), host(w).astype(np.float64)
    if cfg == "zoo":
        assert np.array_equal(rr, r_ora) and np.array_equal(ww, w_ora)
        assert fid == 0.5 * float(r_ora @ r_ora)
    else:
        assert rel(rr, r_ora) <= 1e-6 and rel(ww, w_ora) <= 1e-6
        assert abs(fid - 0.5 * float(r_ora @ r_ora)) <= 1e-6 * fid


@pytest.mark.parametrize("cap", [1024, 300, 128])
def test_window_parts_match_oracle(tvreg, c1, cap, monkeypatch):
    """Slice windows cut into parts (the c3 A pass path): rows' entries split at part boundaries,
    fp64 partial sums carried between parts; dyadic data makes the result exact."""
    monkeypatch.setenv("TVR_PART_CAP", str(cap))
    A = _dyadic_separable(32, 32, 6, 12, 45)
    rng = np.random.default_rng(7)
    x = rng.integers(0, 9, A.n_cols).astype(np.float32)
    b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    P = make(tvreg, A, b, (32, 32, 6))
    assert P.info.slab_staged_A == 1 and P.info.slab_staged_AT == 1
    r = torch.empty(A.n_rows, device="cuda")
    fid = P.residual(dev(x), r)
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x) - b
    assert np.array_equal(host(r).astype(np.float64), r_ora)
    assert fid == 0.5 * float(r_ora @ r_ora)
    w = torch.empty(A.n_cols, device="cuda")
    P.apply_AT(dev(b), w)
    assert np.array_equal(host(w).astype(np.float64), oracle.rmatvec(A.row_ptr, A.col, A.val, b, A.n_cols))
    rT, cT, vT = P.get_AT()
    oT = oracle.transpose(A.row_ptr, A.col, A.val, A.n_cols)
    assert np.array_equal(rT, oT[0]) and np.array_equal(cT, oT[1])
    assert np.array_equal(vT.view(np.uint32), oT[2].view(np.uint32))


# ------------------------------------------------------- VIEWS mode (§8(e) P2) on one GPU
def test_views_mode_one_rank_matches_unsharded(tvreg):
    grid = (12, 10, 9)
    A = harness.siddon_tilted(*grid, 8, 9, 13, 10.0)
    b = harness.simulate_data(A, harness.phantom(*grid, 3))
    x = dev(harness.random_x(A.n_cols))
    P0 = make(tvreg, A, b, grid)
    P1 = tvreg.Problem(A.row_ptr, A.col, A.val, b, grid, 0.01, 1e-4, 0.0, math.inf, shard="views",
                       z0=0, z1=grid[2])
    assert P1.info.n_cols_local == A.n_cols
    g0 = torch.empty_like(x)
    g1 = torch.empty_like(x)
    f0, _ = P0.objective_grad(x, g0)
    f1, _ = P1.objective_grad(x, g1)
    assert f0 == f1
    assert torch.equal(g0, g1)


def test_views_row_blocks_sum_to_full_AT(tvreg):
    """Per-rank pieces of P2 on one GPU: each view block's A_p^T y_p spans the whole volume and
    their sum is A^T y; each block's residual is its rows of A x - b."""
    from paper_1105_4002_b200.dist import local_views
    grid = (12, 10, 9)
    views = 8
    A = harness.siddon_tilted(*grid, views, 9, 13, 10.0)
    b = harness.simulate_data(A, harness.phantom(*grid, 3))
    xh = harness.random_x(A.n_cols)
    y = harness.normal(A.n_rows, 7).astype(np.float32)
    w_sum = np.zeros(A.n_cols)
    for rank in range(3):
        lv = local_views(A.row_ptr, A.col, A.val, b, grid, views, 3, rank)
        P = tvreg.Problem(lv.row_ptr, lv.col, lv.val, lv.b, grid, 0.01, 1e-4, 0.0, math.inf,
                          shard="views", z0=0, z1=grid[2])
        w = torch.empty(A.n_cols, device="cuda")
        P.apply_AT(dev(y[lv.row0:lv.row1]), w)
        w_sum += host(w)
        r = torch.empty(lv.row1 - lv.row0, device="cuda")
        P.residual(dev(xh), r)
        ro = oracle.matvec(lv.row_ptr, lv.col, lv.val, xh.astype(np.float64)) - lv.b
        assert rel(host(r), ro) <= 1e-6
    wo = oracle.rmatvec(A.row_ptr, A.col, A.val, y.astype(np.float64), A.n_cols)
    assert rel(w_sum, wo) <= 1e-6


def test_objective_grad_sphere_geometry(tvreg):
    """f2: the paper's geometry (parallel beam, directions over the sphere) is
    non-separable: int32 columns, global gathers; gradient parity with the oracle."""
    grid = (20, 18, 16)
    A = harness.siddon_sphere(*grid, 9, 29, 29)
    b = harness.simulate_data(A, harness.phantom(*grid, 4))
    x = harness.random_x(A.n_cols)
    P = make(tvreg, A, b, grid)
    assert P.info.slab_staged_A == 0
    g = torch.empty(A.n_cols, device="cuda")
    f, _ = P.objective_grad(dev(x), g)
    Po = oracle.Problem(A.row_ptr, A.col, A.val, b, grid, 0.01, 1e-4)
    fo, go = Po.fg(x.astype(np.float64))
    assert abs(f - fo) <= 1e-9 * abs(fo)
    assert rel(host(g), go) <= 1e-5


@pytest.mark.parametrize("chunks", ["1", "3", "4"])
def test_objective_grad_host_pipeline(tvreg, c1, chunks, monkeypatch):
    """e2e API with pinned host buffers: x goes up and g comes down per slab chunk while other
    chunks compute.  The gradient is the unchunked one element for element; f matches to the
    rounding of the per-chunk sums."""
    monkeypatch.setenv("TVR_E2E_CHUNKS", chunks)
    P = make(tvreg, c1.A, c1.b, c1.grid, alpha=c1.alpha, tau=c1.tau)
    x = harness.random_x(c1.N)
    g = torch.empty(c1.N, device="cuda")
    f, (fid, tv) = P.objective_grad(dev(x), g)
    xh = torch.from_numpy(x.copy()).pin_memory()
    gh = torch.empty(c1.N, dtype=torch.float32).pin_memory()
    for _ in range(3):
        fh, (fidh, tvh) = P.objective_grad_host(xh.numpy(), gh.numpy())
        assert torch.equal(gh, g.cpu())
        assert abs(fh - f) <= 1e-13 * abs(f) and abs(tvh - tv) <= 1e-13 * abs(tv)
    fv, _ = P.objective_grad_host(xh.numpy(), None)  # value only
    assert abs(fv - f) <= 1e-13 * abs(f)


@pytest.mark.parametrize("kb", ["4", "6"])
def test_partly_staged_window_matches_staged(tvreg, kb, monkeypatch):
    """Windows larger than shared memory stage their first part and gather the rest from global
    memory (the c3 A pass); forced here on a small slice: results bitwise equal to the fully
    staged kernel (same summation order) and to the oracle on dyadic data."""
    grid = (48, 40, 5)
    A = _dyadic_separable(*grid, 10, 61)
    rng = np.random.default_rng(5)
    x = rng.integers(0, 9, A.n_cols).astype(np.float32)
    b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    outs = {}
    for mode in ("staged", "half"):
        monkeypatch.delenv("TVR_SPMV_STAGE", raising=False)
        monkeypatch.delenv("TVR_SPMV_HALF_KB", raising=False)
        if mode == "half":
            monkeypatch.setenv("TVR_SPMV_STAGE", "0")
            monkeypatch.setenv("TVR_SPMV_HALF_KB", kb)
        P = make(tvreg, A, b, grid)
        r = torch.empty(A.n_rows, device="cuda")
        fid = P.residual(dev(x), r)
        w = torch.empty(A.n_cols, device="cuda")
        P.apply_AT(dev(b), w)
        outs[mode] = (host(r).copy(), fid, host(w).copy())
        P.close()
    assert np.array_equal(outs["half"][0], outs["staged"][0])
    assert np.array_equal(outs["half"][2], outs["staged"][2])
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
    assert np.array_equal(outs["half"][0].astype(np.float64), r_ora)
    assert outs["half"][1] == 0.5 * float(r_ora @ r_ora)


def _full_vector_parity(T, w, x):
    """r = A x - b and g = grad phi(x) of the whole workload element by element against the
    oracle (fp64 from the same fp32 inputs): residual rows per element to fp32 rounding, g to the
    fp32 rounding of r (an A^T row sums ~100-250 terms of the fp32-stored residual), relative L2
    <= 1e-6 for both (the BJ:5 bar for a gradient is 1e-5); f to the fp64 sums' rounding."""
    import os
    P = make(T, w.A, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
    g = torch.empty(w.N, device="cuda")
    f, (fid, tv) = P.objective_grad(dev(x), g)
    r = torch.empty(w.A.n_rows, device="cuda")
    fid2 = P.residual(dev(x), r)
    rh, gh = host(r).astype(np.float64), host(g).astype(np.float64)
    P.close()
    del r, g
    torch.cuda.empty_cache()
    Po = oracle.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                        nthreads=os.cpu_count() or 1)
    ro = Po.residual(x)
    rms_r = np.sqrt(np.mean(ro * ro))
    assert np.all(np.abs(rh - ro) <= 1e-7 * np.abs(ro) + 1e-9 * rms_r)
    assert rel(rh, ro) <= 1e-6
    assert abs(fid - 0.5 * float(ro @ ro)) <= 1e-10 * fid and abs(fid2 - fid) <= 1e-12 * fid
    fo, go = Po.fg(x)
    assert abs(f - fo) <= 1e-10 * abs(fo)
    rms_g = np.sqrt(np.mean(go * go))
    err = np.abs(gh - go) / (np.abs(go) + 1e-2 * rms_g)
    assert err.max() <= 1e-5, (int(err.argmax()), float(err.max()))
    assert rel(gh, go) <= 1e-6
    return P


def test_objective_grad_c3_full_vector(tvreg):
    """BJ:9 workload (256^3, 1.9e9 entries) at full size in the bench's launch configuration
    (16-bit sliced ELL, A pass in two column parts, A^T on one 1024-thread CTA per SM): every
    row of r and every voxel of g against the oracle."""
    w = harness.preset("c3")
    _full_vector_parity(tvreg, w, harness.random_x(w.N))


@pytest.fixture(scope="module")
def c5():
    return harness.preset("c5")


def test_objective_grad_c5_full_vector(tvreg, c5):
    """BJ configs[4] (non-separable 256^3, rays tilted up to 10 deg, 2.67e9 entries) at full size
    in the bench's launch configuration (int32 sliced ELL: A with per-block lane / row modes, A^T
    in lane mode): every row of r and every voxel of g against the oracle."""
    _full_vector_parity(tvreg, c5, harness.random_x(c5.N))


def test_transpose_bit_exact_c5(tvreg, c5):
    """a3 where it is riskiest: c5 has more than 2^31 entries (int64 rowT values up to 2.67e9).
    rowT in full, and colT / valT bit for bit over four whole column ranges (the first and last
    voxels, and ranges straddling entry offsets 2^31 and nnz - 2^28) against the oracle's stable
    counting sort."""
    A = c5.A
    assert A.nnz > 2 ** 31
    P = make(tvreg, A, np.zeros(A.n_rows, np.float32), c5.grid)
    rT, cT, vT = P.get_AT()
    P.close()
    N = A.n_cols
    rows = []
    for off in (2 ** 31, A.nnz - 2 ** 28):
        j = int(np.searchsorted(rT, off, side="right")) - 1
        rows.append((max(0, j - 20000), min(N, j + 20000)))
    ranges = [(0, 40000), *rows, (N - 40000, N)]
    for j0, j1 in ranges:
        oT = oracle.transpose_range(A.row_ptr, A.col, A.val, N, j0, j1)
        if j0 == 0:
            assert np.array_equal(rT, oT[0])
        s, e = int(rT[j0]), int(rT[j1])
        assert np.array_equal(cT[s:e], oT[1])
        assert np.array_equal(vT[s:e].view(np.uint32), oT[2].view(np.uint32))
