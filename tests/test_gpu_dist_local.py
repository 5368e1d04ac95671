"""Multi-rank library paths on one GPU: ranks are host threads sharing the
in-process thread communicator (tvr_local_comm_create), each with its own tvr_problem on the
same device.  Exercises the z-slab halo exchange, halo recomputation of trial / momentum points,
the rank-ordered scalar sum, the VIEWS all-gather / reduce-scatter and the distributed solvers
through the C ABI, against the one-rank problem and against the oracle (SURVEY §8(c).4 item 4:
the P-rank run matches the 1-GPU run, and the same parity bars against the oracle hold)."""
import math
import threading

import numpy as np
import pytest

import harness
import oracle
from paper_1105_4002_b200.dist import local_slab, local_views

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tvreg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1105_4002_b200 import tvreg as T
    return T


def _run_ranks(world, fn):
    """fn(rank) in `world` threads; re-raises the first failure."""
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


def _oracle(A, b, grid, alpha, tau, lo=0.0, hi=math.inf):
    return oracle.Problem(A.row_ptr, A.col, A.val, b, grid, alpha, tau, lo, hi)


def _solve_parity(Po, x_gpu, f_gpu, solver, eps):
    """BJ:5 converged-reconstruction parity: the oracle's own solve to the same eps; both
    objectives evaluated with the oracle's evaluator; gap <= 1e-5, image difference <= 1e-3."""
    ref = getattr(oracle, solver)(Po, np.zeros(Po.N), eps=eps, max_iters=20000)
    assert ref.converged
    xg = x_gpu.double().numpy()
    fg = Po.f(xg)
    assert abs(fg - f_gpu) <= 1e-6 * abs(fg)            # the solver's f is the oracle's at its x
    assert abs(fg - ref.f) <= 1e-5 * abs(ref.f)
    assert np.linalg.norm(xg - ref.x) <= 1e-3 * np.linalg.norm(ref.x)


def _separable():
    return harness.separable_workload("t", (20, 18, 12), 9, 29, 3, alpha=0.02, tau=1e-2)


@pytest.mark.parametrize("world", [2, 3])
def test_zslab_gradient_equals_one_rank(tvreg, world):
    w = _separable()
    plane = w.grid[0] * w.grid[1]
    x = harness.random_x(w.N)
    P1 = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
    g1 = torch.empty(w.N, device="cuda")
    f1, _ = P1.objective_grad(torch.from_numpy(x).cuda(), g1)
    comm = tvreg.local_comm_create(world)

    def rank_fn(r):
        sl = local_slab(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, world, r)
        P = tvreg.Problem(sl.row_ptr, sl.col, sl.val, sl.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                          n_cols=w.N, world=world, rank=r, z0=sl.z0, z1=sl.z1, nccl_comm=comm)
        xl = torch.from_numpy(np.ascontiguousarray(x[sl.z0 * plane:sl.z1 * plane])).cuda()
        g = torch.empty(P.n, device="cuda")
        f, _ = P.objective_grad(xl, g)
        return sl.z0, f, g.cpu()

    res = _run_ranks(world, rank_fn)
    tvreg.local_comm_destroy(comm)
    fs = [r[1] for r in res]
    assert all(f == fs[0] for f in fs)                # every rank sees the same f
    assert abs(fs[0] - f1) <= 1e-13 * abs(f1)         # rank-ordered partial sums
    g = torch.cat([r[2] for r in sorted(res, key=lambda t: t[0])])
    assert torch.equal(g, g1.cpu())                   # per-voxel results are the one-rank ones
    # and against the oracle (BJ:5: single gradient to relative L2 <= 1e-5)
    fo, go = _oracle(w.A, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi).fg(x)
    assert abs(fs[0] - fo) <= 1e-9 * abs(fo)
    assert np.linalg.norm(g.double().numpy() - go) <= 1e-6 * np.linalg.norm(go)


@pytest.mark.parametrize("world", [2, 3])
def test_views_gradient_matches_one_rank(tvreg, world):
    grid, views = (14, 12, 10), 9
    A = harness.siddon_tilted(*grid, views, 7, 17, 10.0)
    b = harness.simulate_data(A, harness.phantom(*grid, 3))
    x = harness.random_x(A.n_cols)
    plane = grid[0] * grid[1]
    P1 = tvreg.Problem(A.row_ptr, A.col, A.val, b, grid, 0.01, 1e-3)
    g1 = torch.empty(A.n_cols, device="cuda")
    f1, _ = P1.objective_grad(torch.from_numpy(x).cuda(), g1)
    comm = tvreg.local_comm_create(world)

    def rank_fn(r):
        lv = local_views(A.row_ptr, A.col, A.val, b, grid, views, world, r)
        P = tvreg.Problem(lv.row_ptr, lv.col, lv.val, lv.b, grid, 0.01, 1e-3, world=world, rank=r,
                          z0=lv.z0, z1=lv.z1, nccl_comm=comm, shard="views")
        xl = torch.from_numpy(np.ascontiguousarray(x[lv.z0 * plane:lv.z1 * plane])).cuda()
        g = torch.empty(P.n, device="cuda")
        f, _ = P.objective_grad(xl, g)
        return lv.z0, f, g.cpu()

    res = _run_ranks(world, rank_fn)
    tvreg.local_comm_destroy(comm)
    fs = [r[1] for r in res]
    assert all(f == fs[0] for f in fs)
    assert abs(fs[0] - f1) <= 1e-12 * abs(f1)
    g = torch.cat([r[2] for r in sorted(res, key=lambda t: t[0])]).double()
    # A^T r is summed over ranks in fp32: agreement to fp32 rounding
    assert (g - g1.cpu().double()).norm() <= 1e-6 * g1.cpu().double().norm()
    fo, go = _oracle(A, b, grid, 0.01, 1e-3).fg(x)
    assert abs(fs[0] - fo) <= 1e-9 * abs(fo)
    assert np.linalg.norm(g.numpy() - go) <= 1e-6 * np.linalg.norm(go)


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_zslab_solvers_match_one_rank(tvreg, solver):
    """The distributed solvers (host control, rank-ordered scalars) against the one-rank solve:
    every rank takes the same branches; the objective and iterate agree to the scalar sums'
    rounding (which can shift a line-search decision late in the run)."""
    world = 2
    w = _separable()
    plane = w.grid[0] * w.grid[1]
    P1 = tvreg.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
    x1 = torch.zeros(w.N, device="cuda")
    r1 = getattr(P1, f"solve_{solver}")(x1, max_iters=20000, eps=1e-6)
    comm = tvreg.local_comm_create(world)

    def rank_fn(r):
        sl = local_slab(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, world, r)
        P = tvreg.Problem(sl.row_ptr, sl.col, sl.val, sl.b, w.grid, w.alpha, w.tau, w.lo, w.hi,
                          n_cols=w.N, world=world, rank=r, z0=sl.z0, z1=sl.z1, nccl_comm=comm)
        x = torch.zeros(P.n, device="cuda")
        res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6)
        return sl.z0, res, x.cpu()

    out = _run_ranks(world, rank_fn)
    tvreg.local_comm_destroy(comm)
    its = [o[1].iters for o in out]
    assert all(i == its[0] for i in its) and all(o[1].converged for o in out)
    f = out[0][1].f
    assert abs(f - r1.f) <= 1e-6 * abs(r1.f)
    x = torch.cat([o[2] for o in sorted(out, key=lambda t: t[0])]).double()
    assert (x - x1.cpu().double()).norm() <= 1e-3 * x1.cpu().double().norm()
    assert 0.8 * r1.iters <= its[0] <= 1.25 * r1.iters
    _solve_parity(_oracle(w.A, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi), x, f, solver, 1e-6)


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_views_solvers_match_oracle(tvreg, solver):
    """Distributed solve in VIEWS mode (P2: tilted rays, rows sharded by views, A^T r
    reduce-scattered to slabs) against the oracle's solve of the whole problem."""
    world = 2
    grid, views = (14, 12, 10), 9
    A = harness.siddon_tilted(*grid, views, 7, 17, 10.0)
    b = harness.simulate_data(A, harness.phantom(*grid, 3))
    alpha, tau = 0.01, 1e-2
    comm = tvreg.local_comm_create(world)

    def rank_fn(r):
        lv = local_views(A.row_ptr, A.col, A.val, b, grid, views, world, r)
        P = tvreg.Problem(lv.row_ptr, lv.col, lv.val, lv.b, grid, alpha, tau, world=world, rank=r,
                          z0=lv.z0, z1=lv.z1, nccl_comm=comm, shard="views")
        x = torch.zeros(P.n, device="cuda")
        res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6)
        return lv.z0, res, x.cpu()

    out = _run_ranks(world, rank_fn)
    tvreg.local_comm_destroy(comm)
    its = [o[1].iters for o in out]
    assert all(i == its[0] for i in its) and all(o[1].converged for o in out)
    x = torch.cat([o[2] for o in sorted(out, key=lambda t: t[0])])
    _solve_parity(_oracle(A, b, grid, alpha, tau), x, out[0][1].f, solver, 1e-6)


@pytest.mark.parametrize("world", [2, 3])
def test_views_fused_reduce_scatter_matches_collective(tvreg, world, monkeypatch):
    """VIEWS A^T with the fused reduce-scatter (the kernel stores each row into its owner's
    inbox, the owner sums the inboxes in rank order) equals the collective reduce-scatter
    bitwise (same fp32 sums in rank order), and the distributed gradient matches one rank."""
    grid, views = (14, 12, 10), 9
    A = harness.siddon_tilted(*grid, views, 7, 17, 10.0)
    b = harness.simulate_data(A, harness.phantom(*grid, 3))
    x = harness.random_x(A.n_cols)
    plane = grid[0] * grid[1]
    outs = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("TVR_FUSED_RS", fused)
        comm = tvreg.local_comm_create(world)

        def rank_fn(r):
            lv = local_views(A.row_ptr, A.col, A.val, b, grid, views, world, r)
            P = tvreg.Problem(lv.row_ptr, lv.col, lv.val, lv.b, grid, 0.01, 1e-3, world=world,
                              rank=r, z0=lv.z0, z1=lv.z1, nccl_comm=comm, shard="views")
            assert P.info.views_fused_rs == int(fused)
            xl = torch.from_numpy(np.ascontiguousarray(x[lv.z0 * plane:lv.z1 * plane])).cuda()
            g = torch.empty(P.n, device="cuda")
            vals = [P.objective_grad(xl, g)[0] for _ in range(3)]  # repeated passes reuse inboxes
            return lv.z0, vals, g.cpu()

        res = _run_ranks(world, rank_fn)
        tvreg.local_comm_destroy(comm)
        outs[fused] = (res[0][1], torch.cat([r[2] for r in sorted(res, key=lambda t: t[0])]))
    assert outs["1"][0] == outs["0"][0]
    assert torch.equal(outs["1"][1], outs["0"][1])


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("solver", ["gpbb", "upn", "gp"])
def test_views_rep_solvers_equal_views(tvreg, world, solver):
    """VIEWS_REP (x, g and the trial / momentum points kept whole on every rank: the points are
    formed redundantly outside the slab, the gradient's slab is all-gathered once per gradient,
    the A pass reads the whole point without an all-gather) takes exactly the steps of VIEWS
    (the all-gather of the point before every A pass): identical iterations, objective and
    iterate, bitwise; the gradient too.  Against the oracle's solve of the whole problem."""
    grid, views = (14, 12, 10), 9
    A = harness.siddon_tilted(*grid, views, 7, 17, 10.0)
    b = harness.simulate_data(A, harness.phantom(*grid, 3))
    alpha, tau = 0.01, 1e-2
    x0 = harness.random_x(A.n_cols)
    plane = grid[0] * grid[1]
    iters = {"gpbb": 20000, "upn": 20000, "gp": 300}[solver]
    outs = {}
    for shard in ("views", "views_rep"):
        comm = tvreg.local_comm_create(world)

        def rank_fn(r):
            lv = local_views(A.row_ptr, A.col, A.val, b, grid, views, world, r)
            P = tvreg.Problem(lv.row_ptr, lv.col, lv.val, lv.b, grid, alpha, tau, world=world,
                              rank=r, z0=lv.z0, z1=lv.z1, nccl_comm=comm, shard=shard)
            xl = torch.from_numpy(np.ascontiguousarray(x0[lv.z0 * plane:lv.z1 * plane])).cuda()
            g = torch.empty(P.n, device="cuda")
            f, _ = P.objective_grad(xl, g)
            n0 = P.get_info().point_allgathers
            assert n0 == 1 and P.info.views_rep == (shard == "views_rep")  # a caller's slab
            x = torch.zeros(P.n, device="cuda")
            res = getattr(P, f"solve_{solver}")(x, max_iters=iters, eps=1e-6)
            # VIEWS all-gathers the point before every A pass (at least one per objective
            # evaluation), VIEWS_REP never in a solve
            ng = P.get_info().point_allgathers - n0
            assert ng == 0 if shard == "views_rep" else ng >= res.n_f
            return lv.z0, (f, res.iters, res.f, res.n_f, res.converged), g.cpu(), x.cpu()

        res = _run_ranks(world, rank_fn)
        tvreg.local_comm_destroy(comm)
        res.sort(key=lambda t: t[0])
        assert all(r[1] == res[0][1] for r in res)  # every rank: the same branches and values
        outs[shard] = (res[0][1], torch.cat([r[2] for r in res]), torch.cat([r[3] for r in res]))
    assert outs["views_rep"][0] == outs["views"][0]
    assert torch.equal(outs["views_rep"][1], outs["views"][1])
    assert torch.equal(outs["views_rep"][2], outs["views"][2])
    if solver != "gp":
        assert outs["views_rep"][0][4]
        _solve_parity(_oracle(A, b, grid, alpha, tau), outs["views_rep"][2],
                      outs["views_rep"][0][2], solver, 1e-6)
