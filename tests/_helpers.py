"""Small test-only helpers: random sparse matrices and dense brute-force assemblies."""
import numpy as np


class SmallCSR:
    def __init__(self, row_ptr, col, val, n_cols):
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        self.col = np.ascontiguousarray(col, np.int32)
        self.val = np.ascontiguousarray(val, np.float32)
        self.n_rows = len(row_ptr) - 1
        self.n_cols = n_cols

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    def dense(self):
        """Brute-force dense assembly by explicit loops (fp64)."""
        M = np.zeros((self.n_rows, self.n_cols))
        for i in range(self.n_rows):
            for k in range(self.row_ptr[i], self.row_ptr[i + 1]):
                M[i, self.col[k]] += float(self.val[k])
        return M


def random_csr(m, n, density, seed, dyadic=False, empty_rows=0):
    """Random CSR with strictly ascending columns.  dyadic=True gives values k/1024,
    1 <= k <= 2048, so every fp32 partial sum with integer vectors in [0, 8] is exact."""
    rng = np.random.default_rng(seed)
    rp = [0]
    cols, vals = [], []
    dead = set(rng.choice(m, size=empty_rows, replace=False).tolist()) if empty_rows else set()
    for i in range(m):
        if i in dead:
            rp.append(rp[-1])
            continue
        mask = rng.random(n) < density
        c = np.nonzero(mask)[0]
        if dyadic:
            v = rng.integers(1, 2049, size=c.size) / 1024.0
        else:
            v = rng.uniform(0.05, 1.5, size=c.size)
        cols.extend(c.tolist())
        vals.extend(v.tolist())
        rp.append(rp[-1] + c.size)
    return SmallCSR(rp, cols, vals, n)


def identity_csr(n, scale=1.0):
    return SmallCSR(np.arange(n + 1), np.arange(n), np.full(n, scale, np.float32), n)


def diag_csr(d):
    n = len(d)
    return SmallCSR(np.arange(n + 1), np.arange(n), np.asarray(d, np.float32), n)


def dense_D(nx, ny, nz):
    """Explicit 3N x N forward-difference matrix with Neumann last faces (C3), built
    entry by entry; rows (3j, 3j+1, 3j+2) are D_j's x, y, z components."""
    N = nx * ny * nz
    D = np.zeros((3 * N, N))
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                j = (iz * ny + iy) * nx + ix
                if ix < nx - 1:
                    D[3 * j, j + 1] = 1.0
                    D[3 * j, j] = -1.0
                if iy < ny - 1:
                    D[3 * j + 1, j + nx] = 1.0
                    D[3 * j + 1, j] = -1.0
                if iz < nz - 1:
                    D[3 * j + 2, j + nx * ny] = 1.0
                    D[3 * j + 2, j] = -1.0
    return D
