"""c5 A-pass gather locality (offline, CPU): for one view of the c5 geometry, the number of
distinct 128-byte lines of x each 32-lane gather instruction touches (the L1TEX wavefronts that
bound the pass, profiles/r02/c5_raw.csv: l1tex throughput 88 %), for the int32 sliced-ELL modes
(lane: one ray per lane, 4-entry chunks; row: 8 lanes per ray, 4 rays) and for candidate layouts.
usage: python scripts/c5_lines.py [view ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import harness  # noqa: E402

NX = NY = NZ = 256


def blocks(A, order_key=None):
    """yield 32 x L arrays of columns (-1 pad) for consecutive 32-row blocks"""
    rp, col = A.row_ptr, A.col
    m = A.n_rows
    for b0 in range(0, m - 31, 32):
        lens = rp[b0 + 1:b0 + 33] - rp[b0:b0 + 32]
        L = int(lens.max())
        if L == 0:
            continue
        M = np.full((32, L), -1, np.int64)
        for i in range(32):
            c = col[rp[b0 + i]:rp[b0 + i + 1]].astype(np.int64)
            if order_key is not None:
                c = np.sort(order_key(c))
            M[i, :len(c)] = c
        yield M


def distinct_per_column(lines):
    """lines: 32 x S (line ids, -1 = inactive): distinct valid ids per column"""
    s = np.sort(lines, axis=0)
    valid = s >= 0
    new = np.ones_like(s, bool)
    new[1:] = s[1:] != s[:-1]
    return (new & valid).sum(axis=0)


def lane_mode(M):
    # gather instruction k of step t: lane l reads entry 4t + k of its ray
    lines = np.where(M >= 0, M // 32, -1)
    d = distinct_per_column(lines)
    return d.sum(), (M >= 0).any(axis=0).sum()


def row_mode(M):
    # 4 rays at a time; lane j of a ray holds entries 32t + 4j .. +3; instruction k: entries
    # 32t + 4j + k for j = 0..7 of each of the 4 rays
    tot = ins = 0
    for g in range(0, 32, 4):
        R = M[g:g + 4]
        L = R.shape[1]
        T = (L + 31) // 32
        P = np.full((4, T * 32), -1, np.int64)
        P[:, :L] = R
        P = P.reshape(4, T, 8, 4)  # ray, window, lane, k
        lines = np.where(P >= 0, P // 32, -1).transpose(0, 2, 1, 3).reshape(32, T * 4)
        d = distinct_per_column(lines)
        tot += d.sum()
        ins += (lines >= 0).any(axis=0).sum()
    return tot, ins


def xy_swap(c):
    z, r = np.divmod(c, NX * NY)
    y, x = np.divmod(r, NX)
    return (z * NX + x) * NY + y


def brick(bx, by, bz):
    def f(c):
        z, r = np.divmod(c, NX * NY)
        y, x = np.divmod(r, NX)
        bi = ((z // bz) * (NY // by) + (y // by)) * (NX // bx) + (x // bx)
        return (bi * bz + z % bz) * (by * bx) + (y % by) * bx + (x % bx)
    return f


LAYOUTS = (("xy", None), ("yx", xy_swap), ("b442", brick(4, 4, 2)), ("b8x4", brick(8, 4, 1)))


def main():
    views = [int(v) for v in sys.argv[1:]] or [0, 15, 30, 45, 60, 75, 90, 105]
    tot = {}
    for v in views:
        vb = harness.views_block("c5", 120, v)
        A = vb.A
        per = {}
        best_all = 0
        nnz = 0
        mats = {name: list(blocks(A, key)) for name, key in LAYOUTS}
        for bi in range(len(mats["xy"])):
            cand = []
            for name, _ in LAYOUTS:
                M = mats[name][bi]
                a, _ = lane_mode(M)
                b, _ = row_mode(M)
                per.setdefault(name + "_lane", 0)
                per.setdefault(name + "_row", 0)
                per[name + "_lane"] += a
                per[name + "_row"] += b
                cand += [a, b]
            per.setdefault("xy_best", 0)
            per["xy_best"] += min(cand[0], cand[1])
            per.setdefault("xy_yx_best", 0)
            per["xy_yx_best"] += min(cand[:4])
            best_all += min(cand)
            nnz += (mats["xy"][bi] >= 0).sum()
        per["all_best"] = best_all
        f = lambda t: 32.0 * t / nnz  # noqa: E731  lines per 32-lane gather instruction
        print(f"view {v:3d}: " + "  ".join(f"{k} {f(t):5.2f}" for k, t in per.items()), flush=True)
        for k, t in per.items():
            tot[k] = tot.get(k, 0) + t
        tot["nnz"] = tot.get("nnz", 0) + nnz
    print("all   : " + "  ".join(f"{k} {32.0 * t / tot['nnz']:5.2f}" for k, t in tot.items() if k != "nnz"))


if __name__ == "__main__":
    main()
