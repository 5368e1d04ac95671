"""Shared-memory bank-conflict model of the staged 16-bit SpMV gather (spmv16_kernel).

Replays the warp access pattern of one slice (LPR lanes per row, 32 / LPR rows per warp, chunks
of 8 entries at 8-aligned starts, one LDS per (chunk, q), masked lanes reading index 0) and
counts shared-memory wavefronts = max over banks of distinct words, for candidate swizzles.
usage: python scripts/bank_sim.py [nx views bins]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import harness

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
views = int(sys.argv[2]) if len(sys.argv) > 2 else 60
bins = int(sys.argv[3]) if len(sys.argv) > 3 else 181


def swizzles():
    def ident(c):
        return c

    def pad32(c):  # current: c + c/32
        return c + (c >> 5)

    def pad128x4(c):
        return c + 4 * (c >> 7)

    def xor5(c):  # permute 4-word groups inside a 32-word row by the row number
        return c ^ (((c >> 5) & 7) << 2)

    def xor_mix(c):
        r = c >> 5
        return c ^ (((r ^ (r >> 3) ^ (r >> 6)) & 7) << 2)

    def xor_mix2(c):
        r = c >> 5
        return c ^ (((r ^ (r >> 2) ^ (r >> 5) ^ (r >> 8)) & 7) << 2)

    def xor_full(c):  # full 5-bit XOR (breaks 16-byte groups)
        r = c >> 5
        return c ^ ((r ^ (r >> 5)) & 31)

    return dict(ident=ident, pad32=pad32, pad128x4=pad128x4, xor5=xor5, xor_mix=xor_mix,
                xor_mix2=xor_mix2, xor_full=xor_full)


def simulate(rp, col, lpr, sw):
    m = len(rp) - 1
    rows_per_warp = 32 // lpr
    total = 0
    ideal = 0
    for w0 in range(0, m - rows_per_warp + 1, rows_per_warp):
        rows = range(w0, w0 + rows_per_warp)
        kb = [rp[r] & ~7 for r in rows]
        nch = [((rp[r + 1] - kb[i]) + 8 * lpr - 1) // (8 * lpr) for i, r in enumerate(rows)]
        for ch in range(max(nch)):
            for q in range(8):
                addrs = []
                for i, r in enumerate(rows):
                    for lane in range(lpr):
                        k = kb[i] + ch * 8 * lpr + 8 * lane + q
                        if ch < nch[i] and rp[r] <= k < rp[r + 1]:
                            addrs.append(sw(int(col[k])))
                        else:
                            addrs.append(sw(0))
                a = np.unique(np.array(addrs))
                total += np.bincount(a & 31, minlength=32).max()
                ideal += 1
    return total, ideal


def main():
    A = harness.siddon_slice(nx, nx, views, bins)
    S = A.to_scipy().tocsc()
    AT_rp, AT_col = S.indptr.astype(np.int64), S.indices.astype(np.int64)
    for name, sw in swizzles().items():
        ta, ia = simulate(A.row_ptr, A.col, 8, sw)
        tt, it = simulate(AT_rp, AT_col, 4, sw)
        print(f"{name:10s} A: {ta / ia:.3f} wavefronts/LDS   A^T: {tt / it:.3f}", flush=True)


if __name__ == "__main__":
    main()
