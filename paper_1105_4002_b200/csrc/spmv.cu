// CSR SpMV passes of the gradient evaluation.
//
//  a1  r = A v - b, 1/2||r||^2        (Eq. (1); once per line-search / BT trial)
//  a2  w = A^T r  (stored transposed CSR, no atomics)
//  a6  sum ((1+beta) r1 - beta r0)^2   (UPN momentum residual by linearity)
//
// Both SpMVs use LPR lanes per row, 128-bit streaming loads of 4 column indices and 4 values
// per lane over a 16-byte-aligned window masked at the row edges, fp64 accumulation and a
// fixed-order butterfly.  Work is split into nnz-balanced row items; a persistent grid of
// CTAs walks contiguous item ranges.  For slice-separable matrices (every row of A touches one
// z-slice; rows slice-major) the gather vector of the current slice is staged in shared memory
// once per slice change, so the x[col] / r[colT] gathers hit smem instead of L1/L2.
#include "common.cuh"
#include "kernels.h"

namespace tvr {

// Shared-memory index of slice-local column c.  MODE 0: identity; MODE 1: rows of nx voxels
// padded to a pitch of pitch (nx a power of two, shift = log2 nx) so that y-direction rays
// (column stride nx) spread over the 32 banks.
template <int MODE>
__device__ __forceinline__ int smem_index(int c, int shift, int extra) {
  if constexpr (MODE == 0) return c;
  else return c + (c >> shift) * extra;
}

template <int LPR, bool STAGED, int PADMODE>
__global__ void __launch_bounds__(512) spmv_kernel(SpmvArgs a) {
  extern __shared__ float stage[];
  const int lane = threadIdx.x & (LPR - 1);
  const int grp = threadIdx.x / LPR;
  const int ngrp = blockDim.x / LPR;
  const int64_t it0 = (a.nitems * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t it1 = (a.nitems * (int64_t)(blockIdx.x + 1)) / gridDim.x;
  int cur_slice = -1;
  int64_t win_lo = 0;
  double sq = 0.0;
  for (int64_t it = it0; it < it1; ++it) {
    if constexpr (STAGED) {
      const int z = a.item_slice[it];
      if (z != cur_slice) {
        __syncthreads();
        win_lo = a.win_lo[z];
        const int len = a.win_len[z];
        const float* src = a.src + win_lo;
        for (int i = threadIdx.x; i < len; i += blockDim.x)
          stage[smem_index<PADMODE>(i, a.pad_shift, a.pad_extra)] = __ldg(src + i);
        __syncthreads();
        cur_slice = z;
      }
    }
    const int64_t r0 = a.item_row[it], r1 = a.item_row[it + 1];
    for (int64_t base = r0; base < r1; base += ngrp) {
      const int64_t row = base + grp;
      double acc = 0.0;
      if (row < r1) {
        const int64_t s = a.rp[row], e = a.rp[row + 1];
        for (int64_t k0 = (s & ~int64_t(3)) + 4 * lane; k0 < e; k0 += 4 * LPR) {
          const int4 c = ld_stream_i4(a.col + k0);
          const float4 v = ld_stream_f4(a.val + k0);
          const int cc[4] = {c.x, c.y, c.z, c.w};
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int64_t k = k0 + q;
            if (k >= s && k < e) {
              float xv;
              if constexpr (STAGED)
                xv = stage[smem_index<PADMODE>(cc[q] - (int)win_lo, a.pad_shift, a.pad_extra)];
              else
                xv = __ldg(a.src + cc[q]);
              acc = fma((double)vv[q], (double)xv, acc);
            }
          }
        }
      }
      acc = group_sum<LPR>(acc);
      if (row < r1 && lane == 0) {
        if (a.b) {
          const double r = acc - (double)a.b[row];
          a.out[row] = (float)r;
          sq += r * r;
        } else {
          a.out[row] = (float)acc;
        }
      }
    }
  }
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// a6: s = sum_i ((1+beta) r1_i - beta r0_i)^2 in fp64 (no vector written: only f(y) needs it).
__global__ void momentum_resid_kernel(int64_t m, const float* __restrict__ r1,
                                      const float* __restrict__ r0, double beta, double* partials,
                                      unsigned* counter, double* scal) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
    const double ry = (1.0 + beta) * (double)r1[i] - beta * (double)r0[i];
    s += ry * ry;
  }
  double v[1] = {s};
  reduce_to_scalars<1>(v, partials, counter, scal);
}

// x <- P_Q(x) = min(max(x, lo), hi) over n entries.
__global__ void project_kernel(int64_t n, float* x, double lo, double hi) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    x[i] = (float)clampd((double)x[i], lo, hi);
}

// G = nu (x - P_Q(x - g/nu)); sum G^2.
__global__ void gradient_map_kernel(int64_t n, const float* __restrict__ x,
                                    const float* __restrict__ g, double nu, double lo, double hi,
                                    float* G, double* partials, unsigned* counter, double* scal) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double xv = x[i];
    const double gm = nu * (xv - clampd(xv - (double)g[i] / nu, lo, hi));
    if (G) G[i] = (float)gm;
    s += gm * gm;
  }
  double v[1] = {s};
  reduce_to_scalars<1>(v, partials, counter, scal);
}

// ----------------------------------------------------------------- launchers
template <int LPR, bool STAGED, int PADMODE>
static cudaError_t launch_spmv_t(const SpmvArgs& a, int grid, int block, size_t smem,
                                 cudaStream_t st) {
  auto k = spmv_kernel<LPR, STAGED, PADMODE>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<grid, block, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_spmv(const SpmvArgs& a, int lpr, bool staged, int padmode, int grid, int block,
                        size_t smem, cudaStream_t st) {
#define TVR_SPMV_CASE(L)                                                            \
  if (lpr == L) {                                                                   \
    if (!staged) return launch_spmv_t<L, false, 0>(a, grid, block, 0, st);          \
    if (padmode == 0) return launch_spmv_t<L, true, 0>(a, grid, block, smem, st);   \
    return launch_spmv_t<L, true, 1>(a, grid, block, smem, st);                     \
  }
  TVR_SPMV_CASE(32)
  TVR_SPMV_CASE(16)
  TVR_SPMV_CASE(8)
#undef TVR_SPMV_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_momentum_resid(int64_t m, const float* r1, const float* r0, double beta,
                                  double* partials, unsigned* counter, double* scal, int grid,
                                  cudaStream_t st) {
  momentum_resid_kernel<<<grid, 256, 0, st>>>(m, r1, r0, beta, partials, counter, scal);
  return cudaGetLastError();
}

cudaError_t launch_project(int64_t n, float* x, double lo, double hi, int grid, cudaStream_t st) {
  project_kernel<<<grid, 256, 0, st>>>(n, x, lo, hi);
  return cudaGetLastError();
}

cudaError_t launch_gradient_map(int64_t n, const float* x, const float* g, double nu, double lo,
                                double hi, float* G, double* partials, unsigned* counter,
                                double* scal, int grid, cudaStream_t st) {
  gradient_map_kernel<<<grid, 256, 0, st>>>(n, x, g, nu, lo, hi, G, partials, counter, scal);
  return cudaGetLastError();
}

}  // namespace tvr
