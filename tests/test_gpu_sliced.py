"""Slice-shared operator (tvr_create_sliced): for slice-invariant geometry the
device stores one slice's matrix A_s and applies A = I_nz (x) A_s.  Checked against the oracle on
the expanded matrix (exact on dyadic data), against the stored-operator problem (per-row results
bitwise: both run the same sliced-ELL blocks), through the solvers, the host-buffer pipeline and
the z-slab path with the thread communicator."""
import threading

import numpy as np
import pytest

import harness
import oracle
from paper_1105_4002_b200.dist import local_slab
from tests._helpers import SmallCSR

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tvreg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1105_4002_b200 import tvreg as T
    return T


def slice_of(A, grid):
    """Rows of slice 0 of a slice-major separable CSR: the slice matrix (in-slice columns)."""
    nz = grid[2]
    ms = A.n_rows // nz
    k = int(A.row_ptr[ms])
    return SmallCSR(A.row_ptr[:ms + 1], A.col[:k], A.val[:k], grid[0] * grid[1])


def expand(As, nz):
    """I_nz (x) A_s as a CSR (the operator tvr_create_sliced applies)."""
    plane, ms, k = As.n_cols, As.n_rows, As.nnz
    rp = np.concatenate([[0]] + [As.row_ptr[1:] + z * k for z in range(nz)])
    col = np.concatenate([As.col + z * plane for z in range(nz)])
    val = np.tile(As.val, nz)
    return SmallCSR(rp, col, val, plane * nz)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dyadic_slice(nx, ny, seed):
    """A slice matrix with rows of 0..nx*ny entries and dyadic values (exact fp64 sums)."""
    rng = np.random.default_rng(seed)
    plane = nx * ny
    lens = rng.permutation(np.repeat([0, 1, 3, 7, 8, 9, 31, min(255, plane), plane], 4))
    rp, cols, vals = [0], [], []
    for L in lens:
        cols.extend(np.sort(rng.choice(plane, size=L, replace=False)).tolist())
        vals.extend((rng.integers(1, 2049, size=L) / 1024.0).tolist())
        rp.append(rp[-1] + L)
    return SmallCSR(rp, cols, vals, plane)


def test_sliced_matches_oracle_dyadic(tvreg):
    """A x - b, A^T y and the gradient on the expanded operator: exact on dyadic data."""
    grid = (16, 16, 5)
    As = dyadic_slice(16, 16, 3)
    A = expand(As, grid[2])
    rng = np.random.default_rng(4)
    x = rng.integers(0, 9, A.n_cols).astype(np.float32)
    b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    y = rng.integers(-4, 5, A.n_rows).astype(np.float32)
    P = tvreg.Problem(As.row_ptr, As.col, As.val, b, grid, 0.01, 1e-4, sliced=True)
    assert P.info.slice_shared == grid[2] and P.m == A.n_rows and P.nnz == A.nnz
    r = torch.empty(A.n_rows, device="cuda")
    fid = P.residual(dev(x), r)
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
    assert np.array_equal(r.cpu().numpy().astype(np.float64), r_ora)
    assert fid == 0.5 * float(r_ora @ r_ora)
    w = torch.empty(A.n_cols, device="cuda")
    P.apply_AT(dev(y), w)
    w_ora = oracle.rmatvec(A.row_ptr, A.col, A.val, y.astype(np.float64), A.n_cols)
    assert np.array_equal(w.cpu().numpy().astype(np.float64), w_ora)
    # the stored transpose is A_s's, bit-exact against the oracle's counting-sort transpose
    rpT, colT, valT = P.get_AT()
    o_rp, o_col, o_val = oracle.transpose(As.row_ptr, As.col, As.val, As.n_cols)
    assert np.array_equal(rpT, o_rp) and np.array_equal(colT, o_col)
    assert np.array_equal(valT.view(np.uint32), np.asarray(o_val, np.float32).view(np.uint32))
    P.close()


@pytest.mark.parametrize("cfg,zg", [("c1", "1"), ("c1", "2"), ("c1", "3"), ("c1", "4"),
                                    ("ragged", "2"), ("ragged", "4")])
def test_sliced_equals_stored_operator(tvreg, cfg, zg, monkeypatch):
    """Same problem through tvr_create (expanded CSR) and tvr_create_sliced (its slice), one or
    several slices per pass (TVR_SLICE_Z; ragged: 11 slices, a partial last group): the
    residual, A^T r and the gradient agree bitwise (same blocks, same per-row order); f to the
    rounding of the fp64 block-partial order; both match the oracle gradient."""
    monkeypatch.setenv("TVR_SLICE_Z", zg)
    if cfg == "c1":
        w = harness.preset("c1")
        A, grid, b = w.A, w.grid, w.b
        alpha, tau = w.alpha, w.tau
    else:
        grid = (37, 29, 11)
        A = harness.siddon_separable(37, 29, 11, 13, 47)
        b = np.random.default_rng(5).random(A.n_rows).astype(np.float32)
        alpha, tau = 0.02, 1e-3
    As = slice_of(A, grid)
    Ae = expand(As, grid[2])
    assert np.array_equal(Ae.row_ptr, A.row_ptr) and np.array_equal(Ae.col, A.col)
    x = harness.random_x(A.n_cols)
    P0 = tvreg.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau)
    P1 = tvreg.Problem(As.row_ptr, As.col, As.val, b, grid, alpha, tau, sliced=True)
    out = []
    for P in (P0, P1):
        r = torch.empty(A.n_rows, device="cuda")
        fid = P.residual(dev(x), r)
        g = torch.empty(A.n_cols, device="cuda")
        f, (fidg, tv) = P.objective_grad(dev(x), g)
        out.append((r.cpu(), fid, g.cpu(), f, tv))
    assert torch.equal(out[0][0], out[1][0])
    assert torch.equal(out[0][2], out[1][2])
    assert abs(out[0][1] - out[1][1]) <= 1e-13 * out[0][1]
    assert abs(out[0][3] - out[1][3]) <= 1e-13 * out[0][3]
    Po = oracle.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau)
    fo, go = Po.fg(x.astype(np.float64))
    assert abs(out[1][3] - fo) <= 1e-9 * abs(fo)
    assert rel(out[1][2].numpy(), go) <= 1e-5
    P0.close()
    P1.close()


def test_sliced_solvers_match_stored(tvreg):
    """GPBB and UPN on the slice-shared operator reach the stored operator's solution."""
    w = harness.preset("c1")
    As = slice_of(w.A, w.grid)
    res = {}
    for sliced in (False, True):
        if sliced:
            P = tvreg.Problem(As.row_ptr, As.col, As.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                              sliced=True)
        else:
            P = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
        for solver in ("gpbb", "upn"):
            x = torch.zeros(w.N, device="cuda")
            r = getattr(P, f"solve_{solver}")(x, eps=1e-6, max_iters=5000)
            assert r.converged, (sliced, solver)
            res[(sliced, solver)] = (r.f, x.cpu().numpy())
        P.close()
    for solver in ("gpbb", "upn"):
        f0, x0 = res[(False, solver)]
        f1, x1 = res[(True, solver)]
        assert abs(f1 - f0) <= 1e-6 * abs(f0)
        assert rel(x1, x0) <= 1e-3


@pytest.mark.parametrize("zg", ["1", "3"])
def test_sliced_host_pipeline(tvreg, zg, monkeypatch):
    """The host-buffer API (slab chunks overlapped with PCIe, chunk boundaries on slice-group
    boundaries) on the slice-shared operator gives the device API's gradient element for
    element."""
    monkeypatch.setenv("TVR_SLICE_Z", zg)
    w = harness.preset("c1")
    As = slice_of(w.A, w.grid)
    P = tvreg.Problem(As.row_ptr, As.col, As.val, w.b, w.grid, w.alpha, w.tau, sliced=True)
    x = harness.random_x(w.N)
    g = torch.empty(w.N, device="cuda")
    f, _ = P.objective_grad(dev(x), g)
    xh = torch.from_numpy(x.copy()).pin_memory()
    gh = torch.empty(w.N, dtype=torch.float32).pin_memory()
    fh, _ = P.objective_grad_host(xh.numpy(), gh.numpy())
    assert torch.equal(gh, g.cpu())
    assert abs(fh - f) <= 1e-13 * abs(f)
    P.close()


def _run_ranks(world, fn):
    out, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("zg", ["2", "4"])
def test_sliced_zslab_two_ranks(tvreg, zg, monkeypatch):
    """Z-slab ranks (thread communicator) each holding the same slice matrix and their slab's
    rows of b: the gradient is the one-rank sliced gradient bitwise, f to the rank-ordered sum
    (6 slices per rank: with 4 slices per pass the last group is partial)."""
    monkeypatch.setenv("TVR_SLICE_Z", zg)
    w = harness.separable_workload("t", (20, 18, 12), 9, 29, 3, alpha=0.02, tau=1e-2)
    As = slice_of(w.A, w.grid)
    plane = w.grid[0] * w.grid[1]
    x = harness.random_x(w.N)
    P1 = tvreg.Problem(As.row_ptr, As.col, As.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                       sliced=True)
    g1 = torch.empty(w.N, device="cuda")
    f1, _ = P1.objective_grad(dev(x), g1)
    world = 2
    comm = tvreg.local_comm_create(world)
    ms = As.n_rows

    def rank_fn(r):
        sl = local_slab(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, world, r)
        bl = np.ascontiguousarray(w.b[sl.z0 * ms:sl.z1 * ms])
        P = tvreg.Problem(As.row_ptr, As.col, As.val, bl, w.grid, w.alpha, w.tau, w.lo, w.hi,
                          world=world, rank=r, z0=sl.z0, z1=sl.z1, nccl_comm=comm, sliced=True)
        xl = dev(x[sl.z0 * plane:sl.z1 * plane])
        g = torch.empty(P.n, device="cuda")
        f, _ = P.objective_grad(xl, g)
        P.close()
        return sl.z0, f, g.cpu()

    res = _run_ranks(world, rank_fn)
    tvreg.local_comm_destroy(comm)
    assert res[0][1] == res[1][1]
    assert abs(res[0][1] - f1) <= 1e-13 * abs(f1)
    g = torch.cat([t[2] for t in sorted(res, key=lambda t: t[0])])
    assert torch.equal(g, g1.cpu())
    P1.close()


@pytest.mark.parametrize("floats", ["96", "128"])
def test_sliced_column_parts(tvreg, floats, monkeypatch):
    """Slice-shared operator whose slice window is cut into column parts (the c3 x-slice case),
    forced on a 256-voxel slice: exact on dyadic data for both passes and the fidelity."""
    monkeypatch.setenv("TVR_SPMV_STAGE", "0")
    monkeypatch.setenv("TVR_SELL_PART_FLOATS", floats)
    grid = (16, 16, 5)
    As = dyadic_slice(16, 16, 7)
    A = expand(As, grid[2])
    rng = np.random.default_rng(8)
    x = rng.integers(0, 9, A.n_cols).astype(np.float32)
    b = rng.integers(0, 9, A.n_rows).astype(np.float32)
    P = tvreg.Problem(As.row_ptr, As.col, As.val, b, grid, 0.01, 1e-4, sliced=True)
    r = torch.empty(A.n_rows, device="cuda")
    fid = P.residual(dev(x), r)
    w = torch.empty(A.n_cols, device="cuda")
    P.apply_AT(dev(b), w)
    P.close()
    r_ora = oracle.matvec(A.row_ptr, A.col, A.val, x.astype(np.float64)) - b
    w_ora = oracle.rmatvec(A.row_ptr, A.col, A.val, b.astype(np.float64), A.n_cols)
    assert np.array_equal(r.cpu().numpy().astype(np.float64), r_ora)
    assert np.array_equal(w.cpu().numpy().astype(np.float64), w_ora)
    assert fid == 0.5 * float(r_ora @ r_ora)
