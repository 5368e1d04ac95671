"""C-ABI checks that need no GPU: libtvreg.so loads, exports every symbol include/libtvreg.h
declares, and tvr_create's host-side validation returns the documented status codes before it
touches a device."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_1105_4002_b200 import tvreg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "libtvreg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tvr_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = tvreg.lib()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(tvreg.SIGNATURES), set(names) ^ set(tvreg.SIGNATURES)
    assert L.tvr_abi_version() == 6


def test_defaults_match_the_paper():
    o = tvreg.tvr_gpbb_opts()
    tvreg.lib().tvr_gpbb_default(ctypes.byref(o))
    assert (o.K, o.sigma, o.beta0) == (2, 0.1, 0.95)
    u = tvreg.tvr_upn_opts()
    tvreg.lib().tvr_upn_default(ctypes.byref(u))
    assert (u.L0, u.mu0, u.rho_L, u.bt_max) == (1.0, 1.0, 1.3, 200)


def _create(rp, col, val, b, grid=(2, 2, 1), alpha=0.01, tau=1e-3, lo=0.0, hi=math.inf, **kw):
    return tvreg.Problem(np.asarray(rp), np.asarray(col), np.asarray(val), np.asarray(b), grid,
                         alpha, tau, lo, hi, **kw)


@pytest.mark.parametrize("case,status", [
    (dict(rp=[0, 2, 1], col=[0, 1], val=[1, 1], b=[0, 0]), tvreg.TVR_E_CSR),      # decreasing row_ptr
    (dict(rp=[0, 2], col=[1, 1], val=[1, 1], b=[0]), tvreg.TVR_E_CSR),            # duplicate column
    (dict(rp=[0, 2], col=[2, 1], val=[1, 1], b=[0]), tvreg.TVR_E_CSR),            # descending
    (dict(rp=[0, 1], col=[4], val=[1], b=[0]), tvreg.TVR_E_CSR),                  # out of range
    (dict(rp=[0, 1], col=[0], val=[np.nan], b=[0]), tvreg.TVR_E_CSR),             # non-finite value
    (dict(rp=[1, 1], col=[0], val=[1], b=[0]), tvreg.TVR_E_CSR),                  # row_ptr[0] != 0
    (dict(rp=[0, 1], col=[0], val=[1], b=[np.inf]), tvreg.TVR_E_ARG),             # non-finite b
    (dict(rp=[0, 1], col=[0], val=[1], b=[0], tau=0.0), tvreg.TVR_E_ARG),         # tau <= 0
    (dict(rp=[0, 1], col=[0], val=[1], b=[0], alpha=-1.0), tvreg.TVR_E_ARG),      # alpha < 0
    (dict(rp=[0, 1], col=[0], val=[1], b=[0], lo=1.0, hi=0.0), tvreg.TVR_E_ARG),  # lo >= hi
])
def test_create_validation_statuses(case, status):
    with pytest.raises(tvreg.TVRError) as e:
        _create(**case)
    assert e.value.status == status


def test_create_slab_rejects_rows_outside_the_slab():
    # 2x2x2 grid, rank 1 of 2 owns slice z=1 (voxels 4..7); a row touching voxel 0 is not
    # separable.  The CSR check runs on the host before any collective or CUDA call.
    comm = tvreg.local_comm_create(2)
    try:
        with pytest.raises(tvreg.TVRError) as e:
            _create([0, 2], [0, 5], [1, 1], [0], grid=(2, 2, 2), world=2, rank=1, z0=1, z1=2,
                    nccl_comm=comm)
        assert e.value.status == tvreg.TVR_E_NOT_SEPARABLE
    finally:
        tvreg.local_comm_destroy(comm)


@pytest.mark.parametrize("shard", ["zslab", "views"])
def test_create_single_rank_must_own_every_slice(shard):
    """world == 1 with a partial slab: no neighbour fills the TV halo planes, so
    tvr_create rejects it in every shard mode."""
    with pytest.raises(tvreg.TVRError) as e:
        _create([0, 1], [5], [1], [0], grid=(2, 2, 2), shard=shard, z0=1, z1=2)
    assert e.value.status == tvreg.TVR_E_ARG


@pytest.mark.parametrize("kw", [
    dict(shard="views", z0=1, z1=2),                  # one VIEWS rank must own every slice
    dict(shard="views", world=2, rank=0, z0=0, z1=1),  # world > 1 needs an NCCL communicator
    dict(shard="views", z0=0, z1=3),                  # slab past nz
    dict(shard="zslab", world=2, rank=2, z0=0, z1=1, nccl_comm=1),  # rank out of range
])
def test_create_views_mode_validation(kw):
    # host-side checks, before any CUDA call: a tilted row (voxels 0 and 5) is fine in VIEWS mode
    with pytest.raises(tvreg.TVRError) as e:
        _create([0, 2], [0, 5], [1, 1], [0], grid=(2, 2, 2), **kw)
    assert e.value.status == tvreg.TVR_E_ARG


@pytest.mark.parametrize("case,status", [
    (dict(n_cols=8), tvreg.TVR_E_ARG),                       # n_cols must be nx*ny (one slice)
    (dict(shard="views", world=1, z0=0, z1=2), tvreg.TVR_E_ARG),  # VIEWS unsupported
    (dict(col=[5]), tvreg.TVR_E_CSR),                        # column outside the slice
    (dict(b=[0, 0, np.inf]), tvreg.TVR_E_ARG),               # b has m_s * nz entries, all finite
])
def test_create_sliced_validation(case, status):
    """tvr_create_sliced (f4): host-side checks before any CUDA call; the slice matrix has
    nx*ny columns and b one row block per slice."""
    args = dict(rp=[0, 1], col=[1], val=[1.0], b=[0.0, 0.0], grid=(2, 2, 2))
    kw = {k: v for k, v in case.items() if k not in args}
    args.update({k: v for k, v in case.items() if k in args})
    if "b" in case and len(case["b"]) == 3:
        args["grid"] = (2, 2, 3)
    with pytest.raises(tvreg.TVRError) as e:
        _create(args["rp"], args["col"], args["val"], args["b"], grid=args["grid"], sliced=True, **kw)
    assert e.value.status == status
