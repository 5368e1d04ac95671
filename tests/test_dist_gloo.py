"""Multi-rank z-slab decomposition on CPU (gloo, world size 2 and 3): the partition logic of
paper_1105_4002_b200/dist.py, the halo-exchange pattern of csrc/dist.cu (plane 0 to rank-1,
plane nzl-1 to rank+1) and the rank-ordered scalar sum, checked against the unsharded oracle
gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import harness
import oracle
from paper_1105_4002_b200.dist import local_slab, local_views, row_slices, slab_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_bounds_cover_and_balance():
    for nz in (5, 32, 128):
        for world in (1, 2, 3, 4, 8):
            if world > nz:
                continue
            b = [slab_bounds(nz, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == nz
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [z1 - z0 for z0, z1 in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_bounds(3, 4, 0)


def test_local_slabs_partition_rows():
    w = harness.separable_workload("t", (12, 10, 7), 6, 17, 3)
    A = w.A
    sl = row_slices(A.row_ptr, A.col, 120)
    for world in (2, 3):
        parts = [local_slab(A.row_ptr, A.col, A.val, w.b, w.grid, world, r, sl) for r in range(world)]
        assert parts[0].row0 == 0 and parts[-1].row1 == A.n_rows
        assert all(parts[i].row1 == parts[i + 1].row0 for i in range(world - 1))
        assert np.array_equal(np.concatenate([p.b for p in parts]), w.b)
        for p in parts:
            assert p.row_ptr[0] == 0 and p.row_ptr[-1] == len(p.col)
            if len(p.col):
                assert p.col.min() >= p.z0 * 120 and p.col.max() < p.z1 * 120


def test_row_slices_rejects_non_separable():
    A = harness.siddon_tilted(8, 8, 6, 4, 5, 9, 10.0)
    with pytest.raises(ValueError):
        row_slices(A.row_ptr, A.col, 64)


def _halo_exchange(v, plane, rank, world):
    """Same pattern as csrc/dist.cu: own planes v[plane:-plane]; halos v[:plane], v[-plane:]."""
    reqs = []
    nzl = v.numel() // plane - 2
    if rank > 0:
        reqs.append(dist.isend(v[plane:2 * plane].clone(), rank - 1))
        buf_lo = torch.empty(plane, dtype=v.dtype)
        reqs.append(dist.irecv(buf_lo, rank - 1))
    if rank < world - 1:
        reqs.append(dist.isend(v[nzl * plane:(nzl + 1) * plane].clone(), rank + 1))
        buf_hi = torch.empty(plane, dtype=v.dtype)
        reqs.append(dist.irecv(buf_hi, rank + 1))
    for r in reqs:
        r.wait()
    if rank > 0:
        v[:plane] = buf_lo
    if rank < world - 1:
        v[(nzl + 1) * plane:] = buf_hi


def _rank_ordered_sum(vals, world):
    t = torch.tensor(vals, dtype=torch.float64)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    acc = torch.zeros_like(t)
    for o in out:   # rank order, as dist_sum_scalars
        acc += o
    return acc.numpy()


def _tv_slab(xl, nxy, z0, z1, tau, rank, world):
    """Owned TV value and TV gradient of a slab from its halo-exchanged volume (csrc/tv.cu's
    decomposition: planes [z0, z1), the upper halo supplying dz of the last owned plane)."""
    nx, ny = nxy
    plane = nx * ny
    nzl = z1 - z0
    v = torch.zeros((nzl + 2) * plane, dtype=torch.float64)
    v[plane:(nzl + 1) * plane] = torch.from_numpy(xl)
    _halo_exchange(v, plane, rank, world)
    vz0 = z0 - (1 if rank > 0 else 0)
    vz1 = z1 + (1 if rank < world - 1 else 0)
    lo = plane if rank > 0 else 0
    ext = v.numpy()[plane - lo:(nzl + 1) * plane + (plane if rank < world - 1 else 0)]
    _, g_ext = oracle.tv((nx, ny, vz1 - vz0), ext, tau)
    g_tv = g_ext[lo:lo + nzl * plane]
    up = ext[lo:]
    tv_own = oracle.tv((nx, ny, len(up) // plane), up, tau, False)[0]
    if rank < world - 1:
        tv_own -= oracle.tv((nx, ny, 1), up[-plane:], tau, False)[0]
    return tv_own, g_tv


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = harness.separable_workload("t", (11, 9, 8), 7, 19, 3, alpha=0.02, tau=1e-2)
        nx, ny, nz = w.grid
        plane = nx * ny
        x = harness.random_x(w.N)
        sl = local_slab(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, world, rank)
        nzl = sl.z1 - sl.z0
        # local residual / fidelity / A^T r (columns made slab-local as tvr_create does)
        col_loc = (sl.col - sl.z0 * plane).astype(np.int32)
        xl = x[sl.z0 * plane:sl.z1 * plane].astype(np.float64)
        r = oracle.matvec(sl.row_ptr, col_loc, sl.val, xl) - sl.b.astype(np.float64)
        wl = oracle.rmatvec(sl.row_ptr, col_loc, sl.val, r, nzl * plane)
        tv_own, g_tv = _tv_slab(xl, (nx, ny), sl.z0, sl.z1, w.tau, rank, world)
        s = _rank_ordered_sum([float(r @ r), tv_own], world)
        g_loc = wl + w.alpha * g_tv
        f = 0.5 * s[0] + w.alpha * s[1]
        q.put((rank, sl.z0, sl.z1, f, g_loc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gradient_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = harness.separable_workload("t", (11, 9, 8), 7, 19, 3, alpha=0.02, tau=1e-2)
    Po = oracle.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, w.alpha, w.tau)
    f, g = Po.fg(harness.random_x(w.N))
    plane = 11 * 9
    fs = [r[3] for r in res]
    assert all(fi == fs[0] for fi in fs)          # bitwise identical on every rank
    assert abs(fs[0] - f) <= 1e-12 * abs(f)
    gs = np.concatenate([r[4] for r in res])
    assert [r[1] for r in res][0] == 0 and res[-1][2] == 8
    assert np.allclose(gs, g, rtol=1e-12, atol=1e-12 * np.abs(g).max())
    assert gs.size == plane * 8


# ---------------------------------------------------------------- P2: views sharding
# csrc/dist.cu's VIEWS mode: all-gather of the point (ragged slabs: one broadcast per rank),
# local A pass over the rank's views with global columns, full-volume A_p^T r_p, reduce to each
# slab's owner (ragged: one reduce per rank), then the z-slab TV as in P1.
_TILT = dict(grid=(10, 9, 8), views=6, det=(5, 13), tilt=10.0)


def _tilted():
    nx, ny, nz = _TILT["grid"]
    A = harness.siddon_tilted(nx, ny, nz, _TILT["views"], *_TILT["det"], _TILT["tilt"])
    b = harness.simulate_data(A, harness.phantom(nx, ny, nz, 3))
    return A, b


def test_local_views_partition_rows():
    A, b = _tilted()
    for world in (2, 3, 4):
        parts = [local_views(A.row_ptr, A.col, A.val, b, _TILT["grid"], _TILT["views"], world, r)
                 for r in range(world)]
        assert parts[0].row0 == 0 and parts[-1].row1 == A.n_rows
        assert all(parts[i].row1 == parts[i + 1].row0 for i in range(world - 1))
        assert parts[0].z0 == 0 and parts[-1].z1 == _TILT["grid"][2]
        assert np.array_equal(np.concatenate([p.b for p in parts]), b)
        assert np.array_equal(np.concatenate([p.col for p in parts]), A.col)
    with pytest.raises(ValueError):
        local_views(A.row_ptr, A.col, A.val, b, _TILT["grid"], 7, 2, 0)


def _views_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, b = _tilted()
        nx, ny, nz = _TILT["grid"]
        plane, N = nx * ny, nx * ny * nz
        alpha, tau = 0.02, 1e-2
        lv = local_views(A.row_ptr, A.col, A.val, b, _TILT["grid"], _TILT["views"], world, rank)
        bounds = [slab_bounds(nz, world, r) for r in range(world)]
        x = harness.random_x(N).astype(np.float64)
        xl = x[lv.z0 * plane:lv.z1 * plane].copy()
        # all-gather the point: one broadcast per rank into its slab of the full buffer
        full = torch.zeros(N, dtype=torch.float64)
        for r, (z0, z1) in enumerate(bounds):
            piece = torch.from_numpy(xl) if r == rank else torch.zeros((z1 - z0) * plane, dtype=torch.float64)
            dist.broadcast(piece, src=r)
            full[z0 * plane:z1 * plane] = piece
        r_loc = oracle.matvec(lv.row_ptr, lv.col, lv.val, full.numpy()) - lv.b.astype(np.float64)
        w_part = torch.from_numpy(oracle.rmatvec(lv.row_ptr, lv.col, lv.val, r_loc, N))
        # reduce-scatter: each slab summed onto its owner
        w_slab = None
        for r, (z0, z1) in enumerate(bounds):
            piece = w_part[z0 * plane:z1 * plane].clone()
            dist.reduce(piece, dst=r)
            if r == rank:
                w_slab = piece.numpy()
        tv_own, g_tv = _tv_slab(xl, (nx, ny), lv.z0, lv.z1, tau, rank, world)
        s = _rank_ordered_sum([float(r_loc @ r_loc), tv_own], world)
        q.put((rank, lv.z0, lv.z1, 0.5 * s[0] + alpha * s[1], w_slab + alpha * g_tv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_views_sharded_gradient_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_views_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, b = _tilted()
    Po = oracle.Problem(A.row_ptr, A.col, A.val, b, _TILT["grid"], 0.02, 1e-2)
    f, g = Po.fg(harness.random_x(A.n_cols))
    fs = [r[3] for r in res]
    assert all(fi == fs[0] for fi in fs)
    assert abs(fs[0] - f) <= 1e-12 * abs(f)
    gs = np.concatenate([r[4] for r in res])
    assert gs.size == g.size
    assert np.allclose(gs, g, rtol=1e-12, atol=1e-12 * np.abs(g).max())


def test_weak_slab_tiles_a_tall_volume():
    """bench.py's weak scaling (harness.weak_slab): rank r owns slices [r nz, (r+1) nz) of a
    volume world times taller, with the preset's slice matrix and global columns."""
    w = harness.preset("c1")
    nx, ny, nz = w.grid
    plane = nx * ny
    for world in (1, 2, 3):
        for rank in range(world):
            sl = harness.weak_slab("c1", world, rank)
            assert sl.grid == (nx, ny, nz * world) and (sl.z0, sl.z1) == (rank * nz, (rank + 1) * nz)
            assert np.array_equal(sl.row_ptr, w.A.row_ptr) and np.array_equal(sl.val, w.A.val)
            assert np.array_equal(sl.col, w.A.col + rank * nz * plane)
            assert sl.b.shape == (w.A.n_rows,)
    assert np.array_equal(harness.weak_slab("c1", 1, 0).b, w.b)  # world 1: the c1 workload itself


# --------------------------------------------- bench.py's per-rank strong-scaling generators
_TINY_SEP = dict(grid=(12, 10, 9), views=7, bins=17, n_ell=3)
_TINY_TILT = dict(grid=(10, 9, 8), views=6, det=(5, 13), tilt=10.0, n_ell=3)


def _strong_worker(rank, world, port, q):
    """As bench.py's large_config_line at N > 1: each rank builds only its own rows
    (harness.strong_slab / harness.views_block, the noise sigma of the views from an all-reduced
    sum of y^2), then the P1 / P2 exchanges of csrc/dist.cu, here with the oracle's arithmetic."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        harness.PRESETS["tiny_sep"] = _TINY_SEP
        harness.PRESETS["tiny_tilt"] = _TINY_TILT
        alpha, tau = 0.01, 1e-2
        out = {}
        # P1: z-slab rows of the separable preset
        sl = harness.strong_slab("tiny_sep", world, rank)
        nx, ny, nz = sl.grid
        plane = nx * ny
        x = harness.random_x(nx * ny * nz).astype(np.float64)
        xl = x[sl.z0 * plane:sl.z1 * plane]
        col_loc = (sl.col - sl.z0 * plane).astype(np.int32)
        r = oracle.matvec(sl.row_ptr, col_loc, sl.val, xl) - sl.b.astype(np.float64)
        wl = oracle.rmatvec(sl.row_ptr, col_loc, sl.val, r, (sl.z1 - sl.z0) * plane)
        tv_own, g_tv = _tv_slab(xl, (nx, ny), sl.z0, sl.z1, tau, rank, world)
        s = _rank_ordered_sum([float(r @ r), tv_own], world)
        out["sep"] = (sl.z0, 0.5 * s[0] + alpha * s[1], wl + alpha * g_tv)
        # P2: view blocks of the tilted preset
        vb = harness.views_block("tiny_tilt", world, rank)
        s2 = torch.tensor([float(vb.y @ vb.y)], dtype=torch.float64)
        dist.all_reduce(s2)
        b = vb.data(float(s2.item()))
        nx, ny, nz = vb.grid
        plane, N = nx * ny, nx * ny * nz
        bounds = [slab_bounds(nz, world, q_) for q_ in range(world)]
        assert bounds[rank] == (vb.z0, vb.z1)
        x = harness.random_x(N).astype(np.float64)
        r = oracle.matvec(vb.A.row_ptr, vb.A.col, vb.A.val, x) - b.astype(np.float64)
        w_part = torch.from_numpy(oracle.rmatvec(vb.A.row_ptr, vb.A.col, vb.A.val, r, N))
        w_slab = None
        for q_, (z0, z1) in enumerate(bounds):
            piece = w_part[z0 * plane:z1 * plane].clone()
            dist.reduce(piece, dst=q_)
            if q_ == rank:
                w_slab = piece.numpy()
        tv_own, g_tv = _tv_slab(x[vb.z0 * plane:vb.z1 * plane], (nx, ny), vb.z0, vb.z1, tau,
                                rank, world)
        s = _rank_ordered_sum([float(r @ r), tv_own], world)
        out["tilt"] = (vb.z0, 0.5 * s[0] + alpha * s[1], w_slab + alpha * g_tv)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strong_scaling_generators_match_unsharded(world, monkeypatch):
    """The per-rank rows bench.py builds for its N > 1 strong-scaling lines (c3 by z-slabs, c5 by
    views) assemble, through the sharded exchanges, the oracle gradient of the single-process
    workload (same rows, same b, same sigma)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    monkeypatch.setitem(harness.PRESETS, "tiny_sep", _TINY_SEP)
    monkeypatch.setitem(harness.PRESETS, "tiny_tilt", _TINY_TILT)
    for key, name in (("sep", "tiny_sep"), ("tilt", "tiny_tilt")):
        w = harness.preset(name)
        Po = oracle.Problem(w.A.row_ptr, w.A.col, w.A.val, w.b, w.grid, 0.01, 1e-2)
        f, g = Po.fg(harness.random_x(w.N))
        parts = sorted([r[1][key] for r in res], key=lambda t: t[0])
        fs = [p_[1] for p_ in parts]
        assert all(fi == fs[0] for fi in fs)
        assert abs(fs[0] - f) <= 1e-12 * abs(f), key
        gs = np.concatenate([p_[2] for p_ in parts])
        assert np.allclose(gs, g, rtol=1e-12, atol=1e-12 * np.abs(g).max()), key
