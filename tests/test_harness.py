"""Pins of the seeded input generators (harness/): Siddon geometry,
phantom and RNG (C17), noise model (C16).  CPU only."""
import math
import os

import numpy as np
import pytest

import harness

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_counts():
    rows = []
    for line in open(os.path.join(GOLDEN, "siddon_counts.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, *nums = line.split()
        rows.append((name, *map(int, nums)))
    return rows


@pytest.mark.parametrize("row", _golden_counts(), ids=lambda r: r[0])
def test_siddon_slice_counts(row):
    name, nx, ny, V, nb, nnz, empty, maxrow, nz, total = row
    s = harness.siddon_slice(nx, ny, V, nb)
    lens = np.diff(s.row_ptr)
    assert s.nnz == nnz
    assert int((lens == 0).sum()) == empty
    assert int(lens.max()) == maxrow
    assert s.nnz * nz == total


def _chord(nx, ny, V, nb, v, b):
    """Closed-form length of ray (v, b) inside the half-open box [-nx/2, nx/2) x [-ny/2, ny/2)."""
    if v == 0:
        c, s = 1.0, 0.0
    elif 2 * v == V:
        c, s = 0.0, 1.0
    else:
        th = math.pi * v / V
        c, s = math.cos(th), math.sin(th)
    sb = b - 0.5 * (nb - 1)
    p = (-s * sb, c * sb)
    d = (c, s)
    n = (nx, ny)
    t0, t1 = -math.inf, math.inf
    for a in range(2):
        lo, hi = -0.5 * n[a], 0.5 * n[a]
        if d[a] == 0.0:
            if not (lo <= p[a] < hi):
                return 0.0
        else:
            ta, tb = (lo - p[a]) / d[a], (hi - p[a]) / d[a]
            t0, t1 = max(t0, min(ta, tb)), min(t1, max(ta, tb))
    return max(0.0, t1 - t0)


@pytest.mark.parametrize("cfg", [(32, 32, 12, 45), (20, 12, 7, 31), (16, 16, 8, 23)])
def test_siddon_row_sum_is_chord_length(cfg):
    nx, ny, V, nb = cfg
    s = harness.siddon_slice(nx, ny, V, nb)
    for i in range(s.n_rows):
        v, b = divmod(i, nb)
        seg = s.val[s.row_ptr[i]:s.row_ptr[i + 1]].astype(np.float64)
        chord = _chord(nx, ny, V, nb, v, b)
        # each fp32 entry carries <= 2^-24 relative rounding
        assert abs(seg.sum() - chord) <= 1e-12 + len(seg) * 2.0 ** -24 * max(1.0, seg.max(initial=0)), (i, seg.sum(), chord)


def test_siddon_axis_aligned_rays_unit_entries_and_structure():
    nx = ny = 32
    V, nb = 12, 45
    s = harness.siddon_slice(nx, ny, V, nb)
    for v in (0, V // 2):
        rows = slice(s.row_ptr[v * nb], s.row_ptr[(v + 1) * nb])
        assert np.all(s.val[rows] == 1.0)
    # strictly ascending, in-range columns within every row
    for i in range(s.n_rows):
        c = s.col[s.row_ptr[i]:s.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
        assert c.size == 0 or (c.min() >= 0 and c.max() < nx * ny)
    # at 0 deg the ray with s_b = -16 runs along voxel row iy = 0 (half-open rule)
    b = 22 - 16
    c = s.col[s.row_ptr[b]:s.row_ptr[b + 1]]
    assert np.array_equal(c, np.arange(32, dtype=np.int32))


def test_separable_replication_layout():
    A = harness.siddon_separable(8, 6, 5, 4, 11)
    s = harness.siddon_slice(8, 6, 4, 11)
    assert A.n_rows == 5 * s.n_rows and A.nnz == 5 * s.nnz
    for z in range(5):
        r0, r1 = z * s.n_rows, (z + 1) * s.n_rows
        seg = slice(A.row_ptr[r0], A.row_ptr[r1])
        assert np.array_equal(A.col[seg], s.col + z * 48)
        assert np.array_equal(A.val[seg], s.val)


def test_tilted_geometry_row_sums_and_layout():
    A = harness.siddon_tilted(12, 10, 8, 5, 6, 9, 10.0)
    assert A.n_rows == 5 * 6 * 9
    for i in range(A.n_rows):
        c = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    # zero tilt reduces to a stack of 2D slices: every row's columns lie in one slice
    A0 = harness.siddon_tilted(8, 8, 4, 3, 4, 11, 0.0)
    for i in range(A0.n_rows):
        c = A0.col[A0.row_ptr[i]:A0.row_ptr[i + 1]]
        if c.size:
            assert len(set((c // 64).tolist())) == 1


def test_splitmix64_reference_stream():
    # SplitMix64 (Steele, Lea, Flood 2014) with seed 0: first outputs are
    # 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4; uniform() = (z >> 11) * 2^-53.
    u = harness.uniform(2, 0)
    assert u[0] == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53
    assert u[1] == (0x6E789E6AA1B965F4 >> 11) * 2.0 ** -53


def test_normal_moments_and_phantom_range():
    z = harness.normal(200000, 7)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    x = harness.phantom(24, 24, 24, 6)
    assert x.dtype == np.float32 and x.min() >= 0.0 and x.max() <= 1.0
    assert (x > 0).mean() > 0.05
    assert np.array_equal(x, harness.phantom(24, 24, 24, 6))


def test_noise_level_rule(c1):
    A = c1.A
    y = A.to_scipy() @ c1.x_true.astype(np.float64)
    e = c1.b.astype(np.float64) - y
    # sigma = 0.01 ||A x_true|| / sqrt(m): ||e|| ~= 0.01 ||A x_true|| (C16)
    assert abs(np.linalg.norm(e) / np.linalg.norm(y) - 0.01) < 0.001


def _box_chord(p0, d, n):
    """Length of p0 + t d (|d| = 1) inside the centred box prod [-n_a/2, n_a/2] (slab method)."""
    t0, t1 = -np.inf, np.inf
    for a in range(3):
        h = 0.5 * n[a]
        if d[a] == 0.0:
            if not (-h <= p0[a] <= h):
                return 0.0
            continue
        ta, tb = sorted(((-h - p0[a]) / d[a], (h - p0[a]) / d[a]))
        t0, t1 = max(t0, ta), min(t1, tb)
    return max(0.0, t1 - t0)


def test_sphere_geometry_row_sums_are_box_chords():
    """f2: every row of the golden-spiral parallel-beam matrix sums to the length of its
    ray inside the volume (closed form by slabs), so Siddon drops or duplicates no segment."""
    nx, ny, nz, V, R, C = 6, 5, 4, 7, 9, 11
    A = harness.siddon_sphere(nx, ny, nz, V, R, C)
    assert A.n_rows == V * R * C and A.n_cols == nx * ny * nz
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    sums = np.bincount(rows, weights=A.val.astype(np.float64), minlength=A.n_rows)
    golden = np.pi * (3.0 - np.sqrt(5.0))
    for i in range(A.n_rows):
        v, r, c = i // (R * C), (i // C) % R, i % C
        ct = 1.0 - (v + 0.5) / V
        st = np.sqrt(1.0 - ct * ct)
        d = np.array([st * np.cos(golden * v), st * np.sin(golden * v), ct])
        a = np.array([0.0, 0.0, 1.0]) if abs(ct) < 0.9 else np.array([1.0, 0.0, 0.0])
        u = np.cross(a, d)
        u /= np.linalg.norm(u)
        w = np.cross(d, u)
        p0 = (c - 0.5 * (C - 1)) * u + (r - 0.5 * (R - 1)) * w
        assert abs(sums[i] - _box_chord(p0, d, (nx, ny, nz))) <= 1e-5, i
    # columns strictly ascending within rows, lengths positive
    for i in range(A.n_rows):
        cs = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
        assert np.all(np.diff(cs) > 0)
    assert np.all(A.val > 0)


def test_f2_presets_match_the_paper_sizes():
    """64^3 voxels, 55 or 19 views of 91^2 pixels (m = 455,455 / 157,339 rows)."""
    for name, views in (("f2many", 55), ("f2few", 19)):
        p = harness.PRESETS[name]
        assert p["grid"] == (64, 64, 64) and p["views"] == views and p["det"] == (91, 91)
    assert 55 * 91 * 91 == 455455 and 19 * 91 * 91 == 157339


def test_sliced_preset_is_the_separable_preset():
    """sliced_preset (f4 inputs): its slice matrix, replicated over the slices, is preset's CSR
    entry for entry, and b / x_true are preset's bit for bit."""
    w = harness.preset("c1")
    s = harness.sliced_preset("c1")
    nx, ny, nz = w.grid
    plane, ms, k = nx * ny, s.A.n_rows, s.A.nnz
    assert s.A.n_cols == plane and ms * nz == w.A.n_rows and k * nz == w.A.nnz
    for z in (0, 1, nz - 1):
        rows = w.A.row_ptr[z * ms:(z + 1) * ms + 1]
        assert np.array_equal(rows - rows[0], s.A.row_ptr)
        seg = slice(int(rows[0]), int(rows[-1]))
        assert np.array_equal(w.A.col[seg] - z * plane, s.A.col)
        assert np.array_equal(w.A.val[seg].view(np.uint32), s.A.val.view(np.uint32))
    assert np.array_equal(w.b.view(np.uint32), s.b.view(np.uint32))
    assert np.array_equal(np.asarray(w.x_true, np.float32), s.x_true)


def test_strong_slab_is_the_presets_rows(monkeypatch):
    """strong_slab (per-rank generator of a z-slab-sharded run) reproduces exactly the rows of
    A and b of the single-process workload for its slices (rows (z V + v) bins + b, C4)."""
    monkeypatch.setitem(harness.PRESETS, "tiny", dict(grid=(20, 18, 12), views=9, bins=29, n_ell=3))
    full = harness.preset("tiny")
    ms = 9 * 29
    for world in (1, 2, 3, 5):
        seen = 0
        for r in range(world):
            s = harness.strong_slab("tiny", world, r)
            r0, r1 = s.z0 * ms, s.z1 * ms
            e0, e1 = full.A.row_ptr[r0], full.A.row_ptr[r1]
            assert np.array_equal(s.row_ptr, full.A.row_ptr[r0:r1 + 1] - e0)
            assert np.array_equal(s.col, full.A.col[e0:e1])
            assert np.array_equal(s.val.view(np.uint32), full.A.val[e0:e1].view(np.uint32))
            assert np.array_equal(s.b.view(np.uint32), full.b[r0:r1].view(np.uint32))
            seen += s.z1 - s.z0
        assert seen == 12


def test_views_block_is_the_presets_rows(monkeypatch):
    """views_block traces only a rank's views; its rows equal that block of the full tilted
    matrix, and b assembled from the ranks' partial sums of y^2 equals the preset's b."""
    monkeypatch.setitem(harness.PRESETS, "tinyt",
                        dict(grid=(14, 12, 10), views=9, det=(7, 17), tilt=10.0, n_ell=3))
    full = harness.preset("tinyt")
    for world in (1, 2, 3):
        parts = [harness.views_block("tinyt", world, r) for r in range(world)]
        rows = [(p.row0, p.row0 + p.A.n_rows) for p in parts]
        assert rows[0][0] == 0 and rows[-1][1] == full.A.n_rows
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        for p, (r0, r1) in zip(parts, rows):
            e0, e1 = full.A.row_ptr[r0], full.A.row_ptr[r1]
            assert np.array_equal(p.A.row_ptr, full.A.row_ptr[r0:r1 + 1] - e0)
            assert np.array_equal(p.A.col, full.A.col[e0:e1])
            assert np.array_equal(p.A.val.view(np.uint32), full.A.val[e0:e1].view(np.uint32))
        s2 = sum(float(p.y @ p.y) for p in parts)
        b = np.concatenate([p.data(s2) for p in parts])
        assert np.array_equal(b.view(np.uint32), full.b.view(np.uint32))
