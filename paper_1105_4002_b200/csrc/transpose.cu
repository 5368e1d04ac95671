// Device construction of the canonical transposed CSR.
//
// rowT[j+1]-rowT[j] = |{k : col_k = j}|; row j of A^T lists the (i, A_ij) with col = j in
// ascending source row i; values are moved bit for bit.  Integer work only, so the result is
// bit-exact and independent of scheduling:
//   1. histogram of column indices (integer atomics)
//   2. exclusive int64 scan -> rowT
//   3. scatter (i, val) into per-row slots via integer atomic cursors (order arbitrary)
//   4. per-row rank sort by source row (keys are unique: columns are strictly ascending
//      within each row of A, so row i contributes at most once to any column)
#include "common.cuh"
#include "kernels.h"

namespace tvr {

__global__ void col_histogram_kernel(int64_t nnz, const int32_t* __restrict__ col,
                                     int32_t* __restrict__ cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += stride)
    atomicAdd(&cnt[col[k]], 1);
}

// Block-local exclusive scan of int32 counts into int64, plus per-block totals.
constexpr int kScanBlock = 1024;
__global__ void scan_blocks_kernel(int64_t n, const int32_t* __restrict__ cnt,
                                   int64_t* __restrict__ out, int64_t* __restrict__ block_tot) {
  __shared__ int64_t s[kScanBlock];
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  const int64_t v = (i < n) ? cnt[i] : 0;
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < kScanBlock; o <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t t = (threadIdx.x >= o) ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  if (i < n) out[i] = s[threadIdx.x] - v;  // exclusive
  if (threadIdx.x == kScanBlock - 1) block_tot[blockIdx.x] = s[kScanBlock - 1];
}

// Sequential exclusive scan of the (few thousand) block totals by one thread.
__global__ void scan_totals_kernel(int64_t nb, int64_t* tot, int64_t* grand) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t run = 0;
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t t = tot[b];
      tot[b] = run;
      run += t;
    }
    *grand = run;
  }
}

__global__ void scan_add_kernel(int64_t n, int64_t* __restrict__ out,
                                const int64_t* __restrict__ block_off) {
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  if (i < n) out[i] += block_off[blockIdx.x];
}

// One warp per row of A: scatter its entries into the rows of A^T.
__global__ void scatter_kernel(int64_t m, const int64_t* __restrict__ rp,
                               const int32_t* __restrict__ col, const float* __restrict__ val,
                               const int64_t* __restrict__ rowT, int32_t* __restrict__ cursor,
                               int32_t* __restrict__ colT, float* __restrict__ valT) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < m; i += nwarps) {
    const int64_t s = rp[i], e = rp[i + 1];
    for (int64_t k = s + lane; k < e; k += 32) {
      const int32_t j = col[k];
      const int64_t pos = rowT[j] + atomicAdd(&cursor[j], 1);
      colT[pos] = (int32_t)i;
      valT[pos] = val[k];
    }
  }
}

// One warp per row of A^T: rank sort (rank = #keys smaller), write to the output arrays.
__global__ void row_rank_sort_kernel(int64_t n, const int64_t* __restrict__ rowT,
                                     const int32_t* __restrict__ ci, const float* __restrict__ vi,
                                     int32_t* __restrict__ co, float* __restrict__ vo) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    const int64_t s = rowT[j], e = rowT[j + 1];
    for (int64_t a = s + lane; a < e; a += 32) {
      const int32_t key = ci[a];
      int64_t rank = 0;
      for (int64_t b = s; b < e; ++b) rank += (ci[b] < key);
      co[s + rank] = key;
      vo[s + rank] = vi[a];
    }
  }
}

cudaError_t build_transpose(int64_t m, int64_t n, int64_t nnz, const int64_t* rp,
                            const int32_t* col, const float* val, int64_t* rowT, int32_t* colT,
                            float* valT, int32_t* scratch_i32_n, int32_t* scratch_col,
                            float* scratch_val, int64_t* scratch_blocks, cudaStream_t st) {
  cudaError_t e;
  const int grid = 148 * 8;
  if ((e = cudaMemsetAsync(scratch_i32_n, 0, sizeof(int32_t) * n, st)) != cudaSuccess) return e;
  if (nnz > 0) col_histogram_kernel<<<grid, 256, 0, st>>>(nnz, col, scratch_i32_n);
  const int64_t nb = (n + 1 + kScanBlock - 1) / kScanBlock;
  // scan over n+1 entries (count[n] treated as 0 gives rowT[n] = nnz)
  scan_blocks_kernel<<<(unsigned)nb, kScanBlock, 0, st>>>(n, scratch_i32_n, rowT, scratch_blocks);
  scan_totals_kernel<<<1, 32, 0, st>>>(nb, scratch_blocks, scratch_blocks + nb);
  scan_add_kernel<<<(unsigned)nb, kScanBlock, 0, st>>>(n, rowT, scratch_blocks);
  if ((e = cudaMemcpyAsync(rowT + n, scratch_blocks + nb, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                           st)) != cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(scratch_i32_n, 0, sizeof(int32_t) * n, st)) != cudaSuccess) return e;
  if (m > 0)
    scatter_kernel<<<grid, 256, 0, st>>>(m, rp, col, val, rowT, scratch_i32_n, scratch_col,
                                         scratch_val);
  if (n > 0) row_rank_sort_kernel<<<grid, 256, 0, st>>>(n, rowT, scratch_col, scratch_val, colT, valT);
  return cudaGetLastError();
}

}  // namespace tvr
