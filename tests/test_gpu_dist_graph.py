"""f3 at world > 1: a solve as ONE CUDA graph with the NCCL
exchanges captured in it -- the scalar all-gather (+ halo send / recv) group per decision point,
the rank-ordered sum taken by a device kernel, halo planes of trial / momentum points recomputed
from device-side step parameters.

One GPU is all this build has, and two NCCL ranks cannot share a device, so the pieces are checked
where they can run: (1) the rank-ordered device sum against the host's sequential sum, bitwise, at
world 1..8; (2) the whole captured path (ncclAllGather inside the conditional WHILE bodies, the
device sum feeding the control kernels) on a ONE-rank NCCL communicator (TVR_DIST_GRAPH_FORCE=1),
bitwise against host control, and against the oracle's converged
reconstruction; (3) the halo-fill kernels with a device-side step against the host-parameter
launch, through the thread communicator's host-control solves (tests/test_gpu_dist_local.py) --
the same kernels, `dparam` null.  The multi-rank send / recv itself has not run on hardware."""
import numpy as np
import pytest

import harness
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tvreg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1105_4002_b200 import tvreg as T
    return T


@pytest.fixture(scope="module")
def nccl1(tvreg):
    """A one-rank NCCL communicator owned by the library (no torch.distributed needed)."""
    comm = tvreg.nccl_comm_init(tvreg.nccl_unique_id(), 1, 0, 0)
    yield comm
    tvreg.nccl_comm_destroy(comm)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_rank_sum_is_the_hosts_sequential_sum(tvreg, world):
    """a7 / a9: out[s] = ((0 + a_0s) + a_1s) + ... in rank order, bitwise the host controller's
    sum (csrc/dist.cu reduce_gathered_scalars), on values whose sum depends on the order."""
    n = 16
    rng = np.random.default_rng(7 + world)
    a = rng.standard_normal((world, n)) * 10.0 ** rng.integers(-8, 9, size=(world, n))
    want = np.zeros(n)
    for r in range(world):
        want = want + a[r]  # sequential, rank order
    g = torch.from_numpy(a.copy()).cuda()
    out = torch.full((n,), np.nan, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    tvreg.rank_sum(g.data_ptr(), world, n, out.data_ptr())
    got = out.cpu().numpy()
    assert np.array_equal(got, want)
    if world >= 3:  # the order matters on this data: a reversed sum differs somewhere
        rev = np.zeros(n)
        for r in reversed(range(world)):
            rev = rev + a[r]
        assert not np.array_equal(rev, want)


def _problem(T, w, comm=None, **kw):
    args = dict(alpha=w.alpha, tau=w.tau, lo=w.lo, hi=w.hi)
    args.update(kw)
    extra = {}
    if comm is not None:
        extra = dict(world=1, rank=0, z0=0, z1=w.grid[2], nccl_comm=comm, shard="zslab")
    return T.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, args["alpha"], args["tau"],
                     args["lo"], args["hi"], **extra)


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
@pytest.mark.parametrize("case", ["c1", "box"])
def test_captured_nccl_graph_equals_host_control(tvreg, nccl1, c1, case, solver, monkeypatch):
    """The distributed solver graph on a one-rank NCCL communicator: every trial's scalars go
    through the captured ncclAllGather and the device rank sum before the control kernel reads
    them.  Iterates, counts and history are bitwise those of host control on the same problem."""
    monkeypatch.setenv("TVR_EXT_EVAL_AT", "1")
    kw = {} if case == "c1" else dict(alpha=0.03, tau=1e-2, hi=1.0)
    P = _problem(tvreg, c1, comm=nccl1, **kw)
    P.set_control("host")
    xh = torch.zeros(c1.N, device="cuda")
    rh = getattr(P, f"solve_{solver}")(xh, max_iters=20000, eps=1e-6, hist_cap=25000)
    P.close()

    monkeypatch.setenv("TVR_DIST_GRAPH_FORCE", "1")
    P = _problem(tvreg, c1, comm=nccl1, **kw)
    P.set_control("device")
    xd = torch.zeros(c1.N, device="cuda")
    rd = getattr(P, f"solve_{solver}")(xd, max_iters=20000, eps=1e-6, hist_cap=25000)
    info = P.get_info()
    P.close()
    assert info.dist_graph_solves == 1
    # one captured exchange per trial and one per accepted gradient (UPN's x_1 runs before the graph)
    assert info.dist_graph_exchanges >= 2 * (rd.iters - 1)
    assert rd.converged and rh.converged and rd.iters == rh.iters
    assert (rd.n_f, rd.n_grad, rd.n_ls) == (rh.n_f, rh.n_grad, rh.n_ls)
    assert rd.f == rh.f and rd.gmap_rel == rh.gmap_rel
    assert torch.equal(xd, xh)
    assert rd.history == rh.history


def test_captured_nccl_graph_not_taken_without_force(tvreg, nccl1, c1, monkeypatch):
    """Without the force switch a one-rank communicator keeps the plain one-GPU graph."""
    monkeypatch.delenv("TVR_DIST_GRAPH_FORCE", raising=False)
    P = _problem(tvreg, c1, comm=nccl1)
    P.set_control("device")
    x = torch.zeros(c1.N, device="cuda")
    P.solve_gpbb(x, max_iters=5, eps=1e-12)
    assert P.get_info().dist_graph_solves == 0
    P.close()


@pytest.mark.parametrize("solver", ["gpbb", "upn"])
def test_captured_nccl_graph_vs_oracle(tvreg, nccl1, c1, solver, monkeypatch):
    """The captured path's converged reconstruction against the ORACLE's (BJ:5 bars: relative
    objective gap <= 1e-5, relative image difference <= 1e-3)."""
    monkeypatch.setenv("TVR_DIST_GRAPH_FORCE", "1")
    Po = oracle.Problem(c1.A.row_ptr, c1.A.col, c1.A.val, c1.b, c1.grid, c1.alpha, c1.tau, c1.lo,
                        c1.hi, nthreads=4)
    ref = getattr(oracle, solver)(Po, np.zeros(c1.N), max_iters=20000, eps=1e-6)
    P = _problem(tvreg, c1, comm=nccl1)
    P.set_control("device")
    x = torch.zeros(c1.N, device="cuda")
    res = getattr(P, f"solve_{solver}")(x, max_iters=20000, eps=1e-6)
    assert P.get_info().dist_graph_solves == 1
    P.close()
    assert res.converged and ref.converged
    xg = x.cpu().numpy().astype(np.float64)
    gap = abs(Po.f(xg) - Po.f(ref.x)) / abs(Po.f(ref.x))
    diff = np.linalg.norm(xg - ref.x) / np.linalg.norm(ref.x)
    assert gap <= 1e-5, gap
    assert diff <= 1e-3, diff
