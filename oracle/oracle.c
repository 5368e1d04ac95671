/* oracle.c — plain, slow, obviously correct fp64 CPU reference for the TV
 * reconstruction hot path.  TEST INFRASTRUCTURE ONLY: it may be used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference arm, never by the product path.  It shares no code with
 * paper_1105_4002_b200/ (the CUDA path) and includes none of its headers.
 *
 * Every quantity is computed in fp64 from the fp32 inputs promoted exactly
 * (SURVEY.md §8(c) C5).  Citations: PAPER.md line numbers (P:n).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* y = A x, y_i = sum_k A_ik x_k : the operand of the fidelity term
 * 1/2 ||Ax - b||^2 of Eq. (1).  Sequential per-row sum.
 * Rows are independent; nthreads > 1 only splits rows (timing). */
void ora_matvec(int64_t m, const int64_t *row_ptr, const int32_t *col, const float *val,
                const double *x, double *y, int nthreads) {
  (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s += (double)val[k] * x[col[k]];
    y[i] = s;
  }
}

/* x = A^T y by scatter over the rows of A: x_j = sum_i A_ij y_i.  Uses no
 * transposed matrix, so it checks the transpose independently. */
void ora_rmatvec_scatter(int64_t m, int64_t n, const int64_t *row_ptr, const int32_t *col,
                         const float *val, const double *y, double *x) {
  for (int64_t j = 0; j < n; ++j) x[j] = 0.0;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) x[col[k]] += (double)val[k] * y[i];
}

/* Canonical transposed CSR by a sequential (stable) counting sort: row j of
 * A^T holds the (i, A_ij) with col = j in ascending i; values moved bit for bit
 * (SURVEY §8(a) a3, §8(c) C20). */
void ora_transpose(int64_t m, int64_t n, const int64_t *row_ptr, const int32_t *col,
                   const float *val, int64_t *rowT, int32_t *colT, float *valT) {
  for (int64_t j = 0; j <= n; ++j) rowT[j] = 0;
  for (int64_t k = 0; k < row_ptr[m]; ++k) rowT[col[k] + 1] += 1;
  for (int64_t j = 0; j < n; ++j) rowT[j + 1] += rowT[j];
  int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t j = 0; j < n; ++j) next[j] = rowT[j];
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      int64_t p = next[col[k]]++;
      colT[p] = (int32_t)i;
      valT[p] = val[k];
    }
  free(next);
}

/* Huber-smoothed isotropic TV, Eq. (2) with h_tau:
 *   TV_tau(x) = sum_j h_tau(t_j),  t_j = ||D_j x||_2,
 *   h_tau(t) = t - tau/2 if t >= tau, t^2/(2 tau) otherwise,
 * D_j x = forward differences (x_{j+ex}-x_j, x_{j+ey}-x_j, x_{j+ez}-x_j), a
 * component being 0 when j lies on the last face of that axis (C3).
 * If grad != NULL it receives  sum_j D_j^T (D_j x / max(t_j, tau))  (C2, C23),
 * assembled by scattering each D_j^T u_j in ascending j.
 * Layout: x fastest, then y, then z (C4). */
double ora_tv(int nx, int ny, int nz, const double *x, double tau, double *grad) {
  const int64_t sx = 1, sy = nx, sz = (int64_t)nx * ny;
  const int64_t N = sz * nz;
  if (grad)
    for (int64_t j = 0; j < N; ++j) grad[j] = 0.0;
  double tv = 0.0;
  for (int iz = 0; iz < nz; ++iz)
    for (int iy = 0; iy < ny; ++iy)
      for (int ix = 0; ix < nx; ++ix) {
        const int64_t j = iz * sz + iy * sy + ix;
        const double dx = (ix < nx - 1) ? x[j + sx] - x[j] : 0.0;
        const double dy = (iy < ny - 1) ? x[j + sy] - x[j] : 0.0;
        const double dz = (iz < nz - 1) ? x[j + sz] - x[j] : 0.0;
        const double t = sqrt(dx * dx + dy * dy + dz * dz);
        tv += (t >= tau) ? t - 0.5 * tau : t * t / (2.0 * tau);
        if (grad) {
          const double den = (t > tau) ? t : tau;
          const double ux = dx / den, uy = dy / den, uz = dz / den;
          grad[j] -= ux + uy + uz;
          if (ix < nx - 1) grad[j + sx] += ux;
          if (iy < ny - 1) grad[j + sy] += uy;
          if (iz < nz - 1) grad[j + sz] += uz;
        }
      }
  return tv;
}

/* The canonical transposed CSR of ora_transpose restricted to the rows j0 <= j < j1 of A^T
 * (columns of A): rowT[0..n] in full (histogram of the columns + exclusive scan, as above) and
 * the entries of rows j0..j1-1, i.e. positions rowT[j0] .. rowT[j1]-1 of colT / valT, written to
 * colT_part / valT_part at offset p - rowT[j0].  Same stable counting sort (rows of A visited in
 * ascending i), so the part is bit-identical to the slice of the full transpose; it lets a test
 * check a matrix whose full transpose does not fit in host memory twice (c5, > 2^31 entries). */
void ora_transpose_range(int64_t m, int64_t n, const int64_t *row_ptr, const int32_t *col,
                         const float *val, int64_t j0, int64_t j1, int64_t *rowT,
                         int32_t *colT_part, float *valT_part) {
  for (int64_t j = 0; j <= n; ++j) rowT[j] = 0;
  for (int64_t k = 0; k < row_ptr[m]; ++k) rowT[col[k] + 1] += 1;
  for (int64_t j = 0; j < n; ++j) rowT[j + 1] += rowT[j];
  const int64_t base = rowT[j0];
  int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(j1 > j0 ? j1 - j0 : 1));
  for (int64_t j = j0; j < j1; ++j) next[j - j0] = rowT[j];
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const int64_t c = col[k];
      if (c < j0 || c >= j1) continue;
      int64_t p = next[c - j0]++;
      colT_part[p - base] = (int32_t)i;
      valT_part[p - base] = val[k];
    }
  free(next);
}
