"""Host logic of the sliced-ELL plan (no GPU): the CTA block ranges by simulated makespan
(tvr_sell_partition).  The checks use an independent Python simulation of the
kernel's schedule -- a CTA walks its range slice segment by slice segment, its warps take the
segment's blocks in stored order, a barrier between segments."""
import heapq

import numpy as np
import pytest

from paper_1105_4002_b200 import tvreg


def _makespan(k, sl, b0, b1, nwarps, blk_cost, seg_cost):
    """List-scheduled time of blocks [b0, b1) (independent re-implementation)."""
    t = 0.0
    i = b0
    while i < b1:
        j = i
        while j < b1 and sl[j] == sl[i]:
            j += 1
        free = [0.0] * nwarps
        heapq.heapify(free)
        end = 0.0
        for q in range(i, j):
            f = heapq.heappop(free) + k[q] + blk_cost
            end = max(end, f)
            heapq.heappush(free, f)
        t += seg_cost + end
        i = j
    return t


def _c2_like(nslices=16, blocks=340, seed=0):
    """Blocks of a slice sorted by length, longest first (like the stored sliced-ELL blocks)."""
    rng = np.random.default_rng(seed)
    k = np.sort(rng.integers(2, 33, size=blocks))[::-1]
    return np.tile(k, nslices).astype(np.int32), np.repeat(np.arange(nslices), blocks).astype(np.int32)


@pytest.mark.parametrize("lam", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("grid", [1, 7, 19, 148])
def test_partition_is_a_cover(lam, grid):
    k, sl = _c2_like(nslices=5, blocks=100)
    tab = tvreg.sell_partition(k, sl, 32, grid, lam=lam)
    assert tab[0] == 0 and tab[-1] == len(k) and len(tab) == grid + 1
    assert np.all(np.diff(tab) >= 0)


def test_partition_uniform_blocks_one_slice_is_even():
    """Equal blocks in one slice: every CTA gets the same number of rounds of its warps."""
    k = np.full(4 * 8 * 10, 5, np.int32)
    sl = np.zeros(len(k), np.int32)
    tab = tvreg.sell_partition(k, sl, 8, 4, lam=1.0)
    rounds = [-(-int(n) // 8) for n in np.diff(tab)]
    assert max(rounds) == 10 and sum(np.diff(tab)) == len(k)


def test_partition_beats_work_sum_split_on_makespan():
    """On slice-structured blocks the largest simulated CTA time of the makespan partition is
    below that of the equal-work-sum split (the split the kernels search for themselves): ranges
    that end a few long blocks into the next slice are what it avoids."""
    k, sl = _c2_like(nslices=32, blocks=340)
    grid, nw, bc, sc = 37, 32, 2.0, 3.0
    tab = tvreg.sell_partition(k, sl, nw, grid, bc, sc, 1.0)
    worst = max(_makespan(k, sl, int(tab[c]), int(tab[c + 1]), nw, bc, sc) for c in range(grid))
    cum = np.concatenate([[0], np.cumsum(k + bc)])
    ws = [int(np.searchsorted(cum, cum[-1] * c / grid)) for c in range(grid)] + [len(k)]
    worst_ws = max(_makespan(k, sl, ws[c], ws[c + 1], nw, bc, sc) for c in range(grid))
    ideal = cum[-1] / (grid * nw)
    assert worst < worst_ws
    assert worst <= 1.15 * ideal + sc + k.max() + bc
    # and every CTA has work
    assert np.all(np.diff(tab) > 0)


def test_partition_rejects_bad_arguments():
    k = np.ones(4, np.int32)
    with pytest.raises(Exception):
        tvreg.sell_partition(k, k, 0, 4)
    with pytest.raises(Exception):
        tvreg.sell_partition(k, k, 32, 4, lam=1.5)
