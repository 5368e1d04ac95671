"""Partitioning and NCCL bootstrap for multi-GPU runs.

P1 (z-slab, slice-separable geometry): a rank owns slices [z0, z1) and the rows of A whose
voxels lie there.  P2 (views, any geometry, e.g. c5's tilted rays): a rank owns a contiguous
range of projection views (rows view-major, C4) with global columns, plus a z-slab of every
volume vector.

Host-side plumbing only: which slices / views and rows a rank owns, extraction of its local
CSR, and creation of the library's NCCL communicator from a unique id broadcast over a
torch.distributed process group.  The exchanges themselves (halo send/recv, rank-ordered
scalar sum, and in P2 the all-gather of the point and reduce-scatter of A^T r) run inside
libtvreg (csrc/dist.cu).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def slab_bounds(nz: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slices [z0, z1) of rank `rank` (ranks ordered along z)."""
    if world > nz:
        raise ValueError(f"cannot split {nz} slices over {world} ranks")
    base, extra = divmod(nz, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def row_slices(row_ptr: np.ndarray, col: np.ndarray, plane: int) -> np.ndarray:
    """Slice of every row (from its first column); empty rows inherit the previous row's slice.
    Raises if a row spans two slices or rows are not slice-major (not slab-separable)."""
    m = len(row_ptr) - 1
    s, e = row_ptr[:-1], row_ptr[1:]
    nonempty = e > s
    first = np.full(m, -1, np.int64)
    last = np.full(m, -1, np.int64)
    first[nonempty] = col[s[nonempty]] // plane
    last[nonempty] = col[e[nonempty] - 1] // plane
    if np.any(first != last):
        raise ValueError("a row of A spans two z-slices: geometry is not slice-separable")
    # forward-fill empty rows
    idx = np.where(nonempty, np.arange(m), 0)
    np.maximum.accumulate(idx, out=idx)
    sl = first[idx]
    sl[sl < 0] = 0
    if np.any(np.diff(sl) < 0):
        raise ValueError("rows are not slice-major")
    return sl


@dataclass
class LocalSlab:
    z0: int
    z1: int
    row0: int
    row1: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    b: np.ndarray


def local_slab(row_ptr, col, val, b, grid, world: int, rank: int, slices=None) -> LocalSlab:
    """Rank's slices and the contiguous block of A's rows (and b) that touch them.  Columns stay
    global (tvr_create makes them slab-local)."""
    nx, ny, nz = grid
    z0, z1 = slab_bounds(nz, world, rank)
    sl = row_slices(row_ptr, col, nx * ny) if slices is None else slices
    r0 = int(np.searchsorted(sl, z0, side="left"))
    r1 = int(np.searchsorted(sl, z1, side="left"))
    if rank == 0:
        r0 = 0
    if rank == world - 1:
        r1 = len(row_ptr) - 1
    e0, e1 = int(row_ptr[r0]), int(row_ptr[r1])
    return LocalSlab(z0, z1, r0, r1, (row_ptr[r0:r1 + 1] - e0).astype(np.int64),
                     col[e0:e1], val[e0:e1], b[r0:r1])


@dataclass
class LocalViews:
    v0: int
    v1: int
    z0: int
    z1: int
    row0: int
    row1: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    b: np.ndarray


def local_views(row_ptr, col, val, b, grid, n_views: int, world: int, rank: int) -> LocalViews:
    """P2: the rank's views [v0, v1) (balanced like slab_bounds), their rows (view-major: view v
    owns rows [v R, (v+1) R), R = m / n_views) with GLOBAL columns, and the rank's z-slab of the
    volume vectors."""
    m = len(row_ptr) - 1
    if n_views <= 0 or m % n_views:
        raise ValueError(f"{m} rows are not {n_views} equal views")
    R = m // n_views
    v0, v1 = slab_bounds(n_views, world, rank)
    z0, z1 = slab_bounds(grid[2], world, rank)
    r0, r1 = v0 * R, v1 * R
    e0, e1 = int(row_ptr[r0]), int(row_ptr[r1])
    return LocalViews(v0, v1, z0, z1, r0, r1, (row_ptr[r0:r1 + 1] - e0).astype(np.int64),
                      col[e0:e1], val[e0:e1], b[r0:r1])


def nccl_comm_from_process_group(world: int, rank: int, device: int) -> int:
    """ncclUniqueId from rank 0, broadcast over the default torch.distributed group; returns the
    library-owned ncclComm_t (as an int) for tvr_dist.nccl_comm."""
    import torch
    import torch.distributed as dist

    from . import tvreg

    n = tvreg.lib().tvr_nccl_unique_id_size()
    if rank == 0:
        uid = torch.tensor(list(tvreg.nccl_unique_id()), dtype=torch.uint8)
    else:
        uid = torch.zeros(n, dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        uid = uid.cuda(device)
    dist.broadcast(uid, src=0)
    return tvreg.nccl_comm_init(bytes(uid.cpu().tolist()), world, rank, device)
