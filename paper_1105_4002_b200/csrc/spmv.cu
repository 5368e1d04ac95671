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
// Instruction budget per entry: predicate, select, swizzle, LDS, 2 conversions, 1 DFMA.
#include <climits>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace tvr {

// Shared-memory slot of window-local index c: one pad word per 32 (banks spread for the
// stride-4 lane pattern of the 128-bit loads; simulated on the c2 rows: ~1.7 wavefronts per
// gather vs ~2.7 for a per-image-row pitch).
__device__ __forceinline__ int swz(int c) { return c + (c >> 5); }

// Stage a slice window into shared memory (swizzled slots) with asynchronous 4-byte copies:
// every copy is in flight at once and the CTA waits one memory latency, instead of one per
// loop trip of a load -> store loop (the restage was ~10% of the A pass's stall samples).
// The caller brackets it with __syncthreads().
// The block size is a multiple of 32, so slot swz(i + blockDim) = swz(i) + blockDim * 33 / 32:
// both addresses advance by a constant (a few instructions per copy instead of a recomputed
// 64-bit address and swizzle).
template <bool WAIT = true>
__device__ __forceinline__ void stage_window(float* stage, const float* __restrict__ g, int len) {
  const int step = blockDim.x;
  uint32_t dst = (uint32_t)__cvta_generic_to_shared(stage + swz(threadIdx.x));
  const uint32_t dstep = (uint32_t)(step + (step >> 5)) * 4u;
  const float* src = g + threadIdx.x;
  int n = len > (int)threadIdx.x ? (len - (int)threadIdx.x + step - 1) / step : 0;
#pragma unroll 4
  for (; n > 0; --n, dst += dstep, src += step)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
  if constexpr (WAIT) asm volatile("cp.async.wait_all;" ::: "memory");
}

// Accumulate the (up to) 4 entries of one lane's 16-byte chunk that fall inside the row:
// entry q is in the row iff lo <= q < hi (lo, hi are 32-bit offsets of the row's ends from the
// chunk start).  Branch-free: masked entries gather slot 0 and multiply by 0.
template <bool STAGED>
__device__ __forceinline__ double chunk_dot(const int4 c, const float4 v, int lo, int hi,
                                            const float* __restrict__ sm, int wl,
                                            const float* __restrict__ src, double acc) {
  const int cc[4] = {c.x, c.y, c.z, c.w};
  const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool in = (q >= lo) & (q < hi);
    const float val = in ? vv[q] : 0.0f;
    float xv;
    if constexpr (STAGED) {
      xv = sm[swz(in ? cc[q] - wl : 0)];
    } else {
      xv = in ? __ldg(src + cc[q]) : 0.0f;
    }
    acc = fma((double)val, (double)xv, acc);
  }
  return acc;
}

// Groups of LPR lanes own one row at a time; each lane streams 16-byte chunks of col and val
// (two chunks in flight), gathers from the staged slice (or global memory), accumulates in
// fp64 and the group reduces with a fixed butterfly.  Row pointers of the next row are
// prefetched while the current row streams.
template <int LPR, bool STAGED, int UNR, int MINB>
__global__ void __launch_bounds__(512, MINB) spmv_kernel(SpmvArgs a) {
  extern __shared__ float stage[];
  const int lane = threadIdx.x & (LPR - 1);
  const int grp = threadIdx.x / LPR;
  const int ngrp = blockDim.x / LPR;
  const int64_t it0 = (a.nitems * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t it1 = (a.nitems * (int64_t)(blockIdx.x + 1)) / gridDim.x;
  int cur_slice = -1;
  int wl = 0;
  double sq = 0.0;
  // rows of one slice segment (the CTA's items of one slice) walked as one range (see spmv16p)
  for (int64_t it = it0; it < it1;) {
    const int z = a.item_slice[it];
    int64_t it_end = it + 1;
    while (it_end < it1 && a.item_slice[it_end] == z) ++it_end;
    if constexpr (STAGED) {
      if (z != cur_slice) {
        __syncthreads();
        const int64_t lo64 = a.win_lo[z];
        const int len = a.win_len[z];
        const float* src = a.src + lo64;
        for (int i = threadIdx.x; i < len; i += blockDim.x) stage[swz(i)] = __ldg(src + i);
        __syncthreads();
        cur_slice = z;
        wl = (int)lo64;
      }
    }
    const int64_t r0 = a.item_row[it], r1 = a.item_row[it_end];
    int64_t row = r0 + grp;
    int64_t s_n = 0, e_n = 0;
    float b_n = 0.0f;
    if (row < r1) {
      s_n = a.rp[row];
      e_n = a.rp[row + 1];
      if (a.b) b_n = __ldg(a.b + row);
    }
    for (int64_t base = r0; base < r1; base += ngrp) {
      const bool valid = row < r1;
      const int64_t s = s_n, e = e_n;
      const float bv = b_n;
      const int64_t nrow = row + ngrp;
      if (nrow < r1) {  // prefetch the next row's extent and data value
        s_n = a.rp[nrow];
        e_n = a.rp[nrow + 1];
        if (a.b) b_n = __ldg(a.b + nrow);
      }
      const int64_t kb = s & ~int64_t(3);
      const int span = (int)(e - kb);
      int lo = (int)(s - kb) - 4 * lane;
      int hi = span - 4 * lane;
      const int nch = valid ? (span + 4 * LPR - 1) / (4 * LPR) : 0;
      const int32_t* cp = a.col + kb + 4 * lane;
      const float* vp = a.val + kb + 4 * lane;
      double acc[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc[u] = 0.0;
      int ch = 0;
      for (; ch + UNR <= nch; ch += UNR) {  // UNR chunks in flight per lane
        int4 c[UNR];
        float4 v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = ld_stream_i4(cp + (ch + u) * 4 * LPR);
          v[u] = ld_stream_f4(vp + (ch + u) * 4 * LPR);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          acc[u] = chunk_dot<STAGED>(c[u], v[u], lo - 4 * LPR * u, hi - 4 * LPR * u, stage, wl,
                                     a.src, acc[u]);
        lo -= 4 * LPR * UNR;
        hi -= 4 * LPR * UNR;
      }
      for (; ch < nch; ++ch) {
        const int4 c0 = ld_stream_i4(cp + ch * 4 * LPR);
        const float4 v0 = ld_stream_f4(vp + ch * 4 * LPR);
        acc[0] = chunk_dot<STAGED>(c0, v0, lo, hi, stage, wl, a.src, acc[0]);
        lo -= 4 * LPR;
        hi -= 4 * LPR;
      }
#pragma unroll
      for (int u = 1; u < UNR; ++u) acc[0] += acc[u];
      const double accr = group_sum<LPR>(acc[0]);
      if (valid && lane == 0) {
        if (a.b) {
          const double r = accr - (double)bv;
          const float rh = (float)r;
          a.out[row] = rh;
          if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);  // hi + lo carries r to ~2^-48
          sq += r * r;
        } else {
          a.out[row] = (float)accr;
        }
      }
      row = nrow;
    }
    it = it_end;
  }
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// ---------------------------------------------------------------------------------------------
// 16-bit column variant for slice-staged matrices: every column is stored as its offset inside
// the slice window (< 65536), so one 16-byte load carries 8 columns and the entry costs 6 bytes
// of HBM instead of 8.  Chunks are 8 entries (one int4 of columns + two float4 of values).
// STAGED: gather from the shared-memory window; otherwise from global memory at gbase (the
// window start), for windows too large to stage (c3's 256 KB x-slice, mostly L1-resident).
template <bool STAGED>
__device__ __forceinline__ double chunk8_dot(const int4 c, const float4 v0, const float4 v1, int lo,
                                             int hi, const float* __restrict__ sm,
                                             const float* __restrict__ gbase, double acc) {
  const uint32_t cw[4] = {(uint32_t)c.x, (uint32_t)c.y, (uint32_t)c.z, (uint32_t)c.w};
  const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  double pr[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const bool in = (q >= lo) & (q < hi);
    const int cidx = (int)((cw[q >> 1] >> (16 * (q & 1))) & 0xffffu);  // little-endian halves
    const float val = in ? vv[q] : 0.0f;
    float xv;
    if constexpr (STAGED) xv = sm[swz(in ? cidx : 0)];
    else xv = in ? __ldg(gbase + cidx) : 0.0f;
    pr[q] = (double)val * (double)xv;  // exact: 24-bit x 24-bit significands fit fp64
  }
  // pairwise tree (depth 3) instead of an 8-deep fma chain: shorter dependency latency
  return acc + (((pr[0] + pr[1]) + (pr[2] + pr[3])) + ((pr[4] + pr[5]) + (pr[6] + pr[7])));
}

// Main 16-bit kernel: whole slice window staged in shared memory (STAGED) or gathered from
// global memory at the window start.  The CTA restages only when the slice changes.
template <int LPR, int UNR, int MINB, bool STAGED>
__global__ void __launch_bounds__(512, MINB) spmv16_kernel(SpmvArgs a) {
  extern __shared__ float stage[];
  const int lane = threadIdx.x & (LPR - 1);
  const int grp = threadIdx.x / LPR;
  const int ngrp = blockDim.x / LPR;
  const int64_t it0 = (a.nitems * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t it1 = (a.nitems * (int64_t)(blockIdx.x + 1)) / gridDim.x;
  int cur_slice = -1;
  const float* gbase = a.src;
  double sq = 0.0;
  // Rows of one slice segment (the CTA's items of one slice) are walked as one range: per-item
  // rounds left groups idle whenever an item had fewer rows than the CTA has groups.
  for (int64_t it = it0; it < it1;) {
    const int z = a.item_slice[it];
    int64_t it_end = it + 1;
    while (it_end < it1 && a.item_slice[it_end] == z) ++it_end;
    if (z != cur_slice) {
      const int64_t lo64 = a.win_lo[z];
      gbase = a.src + lo64;
      if constexpr (STAGED) {
        __syncthreads();
        const int len = a.win_len[z];
        stage_window(stage, gbase, len);
        __syncthreads();
      }
      cur_slice = z;
    }
    const int64_t r0 = a.item_row[it], r1 = a.item_row[it_end];
    int64_t row = r0 + grp;
    int64_t s_n = 0, e_n = 0;
    // b is prefetched with the next row's extent in the staged kernel (A pass -3% at c2); the
    // global-gather variant is register-bound and loads it at the end (prefetch cost 7% at c3).
    float b_n = 0.0f;
    if (row < r1) {
      s_n = a.rp[row];
      e_n = a.rp[row + 1];
      if (STAGED && a.b) b_n = __ldg(a.b + row);
    }
    for (int64_t base = r0; base < r1; base += ngrp) {
      const bool valid = row < r1;
      const int64_t s = s_n, e = e_n;
      const float bv = b_n;
      const int64_t nrow = row + ngrp;
      if (nrow < r1) {  // prefetch the next row's extent (and data value)
        s_n = a.rp[nrow];
        e_n = a.rp[nrow + 1];
        if (STAGED && a.b) b_n = __ldg(a.b + nrow);
      }
      const int64_t kb = s & ~int64_t(7);
      const int span = (int)(e - kb);
      int lo = (int)(s - kb) - 8 * lane;
      int hi = span - 8 * lane;
      const int nch = valid ? (span + 8 * LPR - 1) / (8 * LPR) : 0;
      const uint16_t* cp = a.col16 + kb + 8 * lane;
      const float* vp = a.val + kb + 8 * lane;
      double acc[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc[u] = 0.0;
      int ch = 0;
      for (; ch + UNR <= nch; ch += UNR) {
        int4 c[UNR];
        float4 va[UNR], vb[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + (ch + u) * 8 * LPR));
          va[u] = ld_stream_f4(vp + (ch + u) * 8 * LPR);
          vb[u] = ld_stream_f4(vp + (ch + u) * 8 * LPR + 4);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          acc[u] = chunk8_dot<STAGED>(c[u], va[u], vb[u], lo - 8 * LPR * u, hi - 8 * LPR * u, stage,
                                      gbase, acc[u]);
        lo -= 8 * LPR * UNR;
        hi -= 8 * LPR * UNR;
      }
      for (; ch < nch; ++ch) {
        const int4 c0 = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + ch * 8 * LPR));
        const float4 va0 = ld_stream_f4(vp + ch * 8 * LPR);
        const float4 vb0 = ld_stream_f4(vp + ch * 8 * LPR + 4);
        acc[0] = chunk8_dot<STAGED>(c0, va0, vb0, lo, hi, stage, gbase, acc[0]);
        lo -= 8 * LPR;
        hi -= 8 * LPR;
      }
#pragma unroll
      for (int u = 1; u < UNR; ++u) acc[0] += acc[u];
      const double accr = group_sum<LPR>(acc[0]);
      if (valid && lane == 0) {
        if (a.b) {
          const double r = accr - (double)(STAGED ? bv : __ldg(a.b + row));
          const float rh = (float)r;
          a.out[row] = rh;
          if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);
          sq += r * r;
        } else {
          a.out[row] = (float)accr;
        }
      }
      row = nrow;
    }
    it = it_end;
  }
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// Padded-row 16-bit kernel: the device copy starts every row on an 8-entry boundary and
// zero-pads it to a multiple of 8 entries (pad: value 0, offset 0).  A lane's 8-entry chunk is
// then entirely inside its row or entirely past it, so the per-entry range tests of
// spmv16_kernel (compare, select value, select gather index: ~5 instructions per entry) become
// one select per chunk.  Chunks past the row load whatever follows (valid memory: the arrays
// carry 8 LPR UNR entries of slack) and are discarded.
template <bool STAGED>
__device__ __forceinline__ double chunk8_sum(const int4 c, const float4 v0, const float4 v1,
                                             const float* __restrict__ sm,
                                             const float* __restrict__ gbase) {
  const uint32_t cw[4] = {(uint32_t)c.x, (uint32_t)c.y, (uint32_t)c.z, (uint32_t)c.w};
  const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  double pr[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cidx = (int)((cw[q >> 1] >> (16 * (q & 1))) & 0xffffu);
    float xv;
    if constexpr (STAGED) xv = sm[swz(cidx)];
    else xv = __ldg(gbase + cidx);
    pr[q] = (double)vv[q] * (double)xv;  // exact
  }
  return ((pr[0] + pr[1]) + (pr[2] + pr[3])) + ((pr[4] + pr[5]) + (pr[6] + pr[7]));
}

// The lo parts of an extended-precision source (global gathers through L1): sum of v * x_lo.
__device__ __forceinline__ double chunk8_sum_lo(const int4 c, const float4 v0, const float4 v1,
                                                const float* __restrict__ lbase) {
  const uint32_t cw[4] = {(uint32_t)c.x, (uint32_t)c.y, (uint32_t)c.z, (uint32_t)c.w};
  const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  double pr[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cidx = (int)((cw[q >> 1] >> (16 * (q & 1))) & 0xffffu);
    pr[q] = (double)vv[q] * (double)__ldg(lbase + cidx);
  }
  return ((pr[0] + pr[1]) + (pr[2] + pr[3])) + ((pr[4] + pr[5]) + (pr[6] + pr[7]));
}

// Partly staged window (HALF): offsets below h come from shared memory, the rest from global
// memory (L1) — for windows larger than shared memory (c3's 256 KB x-slice), so that part of the
// gathers leaves the L1 tag / data pipe that global gathers saturate.
__device__ __forceinline__ double chunk8_sum_part(const int4 c, const float4 v0, const float4 v1,
                                                  const float* __restrict__ sm,
                                                  const float* __restrict__ gbase, int h) {
  const uint32_t cw[4] = {(uint32_t)c.x, (uint32_t)c.y, (uint32_t)c.z, (uint32_t)c.w};
  const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  double pr[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cidx = (int)((cw[q >> 1] >> (16 * (q & 1))) & 0xffffu);
    const float xv = cidx < h ? sm[swz(cidx)] : __ldg(gbase + cidx);
    pr[q] = (double)vv[q] * (double)xv;  // exact
  }
  return ((pr[0] + pr[1]) + (pr[2] + pr[3])) + ((pr[4] + pr[5]) + (pr[6] + pr[7]));
}

template <int LPR, int UNR, bool STAGED, int NT = 512, bool HALF = false>
__global__ void __launch_bounds__(NT, 1024 / NT) spmv16p_kernel(SpmvArgs a) {
  extern __shared__ float stage[];
  const int lane = threadIdx.x & (LPR - 1);
  const int grp = threadIdx.x / LPR;
  const int ngrp = blockDim.x / LPR;
  const int64_t it0 = (a.nitems * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t it1 = (a.nitems * (int64_t)(blockIdx.x + 1)) / gridDim.x;
  int cur_slice = -1;
  const float* gbase = a.src;
  double sq = 0.0;
  // Rows of one slice segment (the CTA's items of one slice) are walked as one range: per-item
  // rounds left groups idle whenever an item had fewer rows than the CTA has groups.
  for (int64_t it = it0; it < it1;) {
    const int z = a.item_slice[it];
    int64_t it_end = it + 1;
    while (it_end < it1 && a.item_slice[it_end] == z) ++it_end;
    if (z != cur_slice) {
      gbase = a.src + a.win_lo[z];
      if constexpr (STAGED) {
        __syncthreads();
        const int len = HALF ? min(a.win_len[z], a.part_len) : a.win_len[z];
        stage_window(stage, gbase, len);
        __syncthreads();
      }
      cur_slice = z;
    }
    const int64_t r0 = a.item_row[it], r1 = a.item_row[it_end];
    int64_t row = r0 + grp;
    int64_t s_n = 0, e_n = 0;
    float b_n = 0.0f;
    if (row < r1) {
      s_n = a.rp[row];
      e_n = a.rp[row + 1];
      if (STAGED && a.b) b_n = __ldg(a.b + row);
    }
    for (int64_t base = r0; base < r1; base += ngrp) {
      const bool valid = row < r1;
      const int64_t s = s_n;
      const int span = (int)(e_n - s_n);  // padded: a multiple of 8
      const float bv = b_n;
      const int64_t nrow = row + ngrp;
      if (nrow < r1) {
        s_n = a.rp[nrow];
        e_n = a.rp[nrow + 1];
        if (STAGED && a.b) b_n = __ldg(a.b + nrow);
      }
      const int nch = valid ? (span + 8 * LPR - 1) / (8 * LPR) : 0;
      const int lim = span - 8 * lane;  // chunk k of this lane is in the row iff k 8 LPR < lim
      const uint16_t* cp = a.col16 + s + 8 * lane;
      const float* vp = a.val + s + 8 * lane;
      double acc[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc[u] = 0.0;
      int ch = 0;
      for (; ch + UNR <= nch; ch += UNR) {
        int4 c[UNR];
        float4 va[UNR], vb[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + (ch + u) * 8 * LPR));
          va[u] = ld_stream_f4(vp + (ch + u) * 8 * LPR);
          vb[u] = ld_stream_f4(vp + (ch + u) * 8 * LPR + 4);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const double t = HALF ? chunk8_sum_part(c[u], va[u], vb[u], stage, gbase, a.part_len)
                                : chunk8_sum<STAGED>(c[u], va[u], vb[u], stage, gbase);
          acc[u] += ((ch + u) * 8 * LPR < lim) ? t : 0.0;
        }
      }
      for (; ch < nch; ++ch) {
        const int4 c0 = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + ch * 8 * LPR));
        const float4 va0 = ld_stream_f4(vp + ch * 8 * LPR);
        const float4 vb0 = ld_stream_f4(vp + ch * 8 * LPR + 4);
        const double t = HALF ? chunk8_sum_part(c0, va0, vb0, stage, gbase, a.part_len)
                              : chunk8_sum<STAGED>(c0, va0, vb0, stage, gbase);
        acc[0] += (ch * 8 * LPR < lim) ? t : 0.0;
      }
#pragma unroll
      for (int u = 1; u < UNR; ++u) acc[0] += acc[u];
      const double accr = group_sum<LPR>(acc[0]);
      if (valid && lane == 0) {
        if (a.b) {
          const double r = accr - (double)(STAGED ? bv : __ldg(a.b + row));
          const float rh = (float)r;
          a.out[row] = rh;
          if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);
          sq += r * r;
        } else {
          a.out[row] = (float)accr;
        }
      }
      row = nrow;
    }
    it = it_end;
  }
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// Padded copy of a 16-bit CSR: row r's entries move from rp[r] to rpp[r] (an 8-entry boundary),
// pads to rpp[r+1] are zero.  One warp per row.
__global__ void pad_rows_kernel(int64_t m, const int64_t* rp, const int64_t* rpp,
                                const uint16_t* col16, const float* val, uint16_t* col16p,
                                float* valp) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    const int64_t s = rp[r], len = rp[r + 1] - s, d = rpp[r], plen = rpp[r + 1] - d;
    for (int64_t k = lane; k < plen; k += 32) {
      col16p[d + k] = k < len ? col16[s + k] : (uint16_t)0;
      valp[d + k] = k < len ? val[s + k] : 0.0f;
    }
  }
}

cudaError_t launch_pad_rows(int64_t m, const int64_t* rp, const int64_t* rpp, const uint16_t* col16,
                            const float* val, uint16_t* col16p, float* valp, cudaStream_t st) {
  pad_rows_kernel<<<1184, 256, 0, st>>>(m, rp, rpp, col16, val, col16p, valp);
  return cudaGetLastError();
}

// block 512 (default), or 1024 for a staged plan whose window leaves room for one CTA per SM
// only (c3 A^T: 131 KB), so 32 warps instead of 16 share the one window.
template <class F>
static cudaError_t dispatch16p(const SpmvVariant& v, int block, F&& f) {
  if (v.half) {  // partly staged window, one 1024-thread CTA per SM
    if (v.lpr == 4) return f(spmv16p_kernel<4, 2, true, 1024, true>);
    if (v.lpr == 8) return f(spmv16p_kernel<8, 2, true, 1024, true>);
    if (v.lpr == 16) return f(spmv16p_kernel<16, 2, true, 1024, true>);
    return cudaErrorInvalidValue;
  }
  if (block == 1024) {
    if (!v.staged) return cudaErrorInvalidValue;
    if (v.lpr == 4 && v.unroll == 2) return f(spmv16p_kernel<4, 2, true, 1024>);
    if (v.lpr == 8 && v.unroll == 2) return f(spmv16p_kernel<8, 2, true, 1024>);
    if (v.lpr == 16 && v.unroll == 2) return f(spmv16p_kernel<16, 2, true, 1024>);
    return cudaErrorInvalidValue;
  }
#define TVR_VP(L, U)                                                                   \
  if (v.lpr == L && v.unroll == U)                                                     \
    return v.staged ? f(spmv16p_kernel<L, U, true>) : f(spmv16p_kernel<L, U, false>);
  TVR_VP(4, 2) TVR_VP(4, 3) TVR_VP(4, 4) TVR_VP(8, 2) TVR_VP(8, 3) TVR_VP(16, 2)
#undef TVR_VP
  return cudaErrorInvalidValue;
}

cudaError_t launch_spmv16p(const SpmvArgs& a, const SpmvVariant& v, int grid, int block,
                           size_t smem, cudaStream_t st) {
  return dispatch16p(v, block, [&](auto k) -> cudaError_t {
    cudaError_t e = ensure_smem_attr((const void*)k, smem);
    if (e != cudaSuccess) return e;
    k<<<grid, block, smem, st>>>(a);
    return cudaGetLastError();
  });
}

int spmv16p_occupancy(const SpmvVariant& v, int block, size_t smem) {
  int occ = 0;
  dispatch16p(v, block, [&](auto k) -> cudaError_t {
    ensure_smem_attr((const void*)k, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, block, smem);
  });
  return occ > 0 ? occ : 1;
}

// Sliced-ELL kernel (SELL-32-sigma, sigma = one slice): inside each slice the rows are sorted by
// chunk count (descending, stable) and cut into blocks of 32 rows, one row per lane; a block's rows
// are padded with zero chunks to its longest row and stored chunk-interleaved
// ([block step][lane][8 entries]), so every warp load is 512 contiguous bytes, every lane walks
// its own row with no masking and no cross-lane reduction, and the sorted order keeps the zero
// padding to the rows that share a block with a longer one.  CTAs split the block range by
// work (a prefix sum of steps + 2 per block); warps take blocks round-robin.
__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* __restrict__ a, int64_t lo,
                                                   int64_t hi, int64_t key) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Work prefix of virtual block k (block k % nb of repetition k / nb; SellArgs) and the first
// virtual block in [lo, hi] whose prefix reaches t.
__device__ __forceinline__ int64_t sell_work(const SellArgs& a, int64_t k) {
  const int64_t z = k / a.nb;
  return z * a.cum[a.nb] + a.cum[k - z * a.nb];
}
__device__ __forceinline__ int64_t sell_lower(const SellArgs& a, int64_t lo, int64_t hi, int64_t t) {
  const int64_t ws = a.cum[a.nb];
  const int64_t z = ws > 0 ? t / ws : 0;
  const int64_t k = z >= a.rep ? (int64_t)a.rep * a.nb
                               : z * a.nb + lower_bound_i64(a.cum, 0, a.nb, t - z * ws);
  return min(max(k, lo), hi);
}

// First index in [lo, hi) with a[i] >= key (hi if none), a ascending, by a whole warp: 32 probes
// per round (log32 of the range dependent loads instead of log2: the CTA-range search of a c2
// pass is 2 x 16 dependent L2 loads with one thread, ~10 us before the CTA streams anything).
__device__ __forceinline__ int64_t warp_lower_bound_i64(const int64_t* __restrict__ a, int64_t lo,
                                                        int64_t hi, int64_t key) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const bool ge = p >= hi || __ldg(a + p) >= key;
    const unsigned m = __ballot_sync(0xffffffffu, ge);
    if (m == 0) {  // every probe below the key: the answer lies past the last one
      lo = lo + 31 * step + 1;
      continue;
    }
    const int f = __ffs(m) - 1;  // first probe at or past the answer
    if (f == 0) return lo;
    const int64_t pf = lo + f * step;
    lo = lo + (f - 1) * step + 1;
    hi = min(pf, hi);
  }
  return (hi - lo == 1 && __ldg(a + lo) >= key) ? lo : hi;
}
__device__ __forceinline__ int64_t sell_lower_warp(const SellArgs& a, int64_t lo, int64_t hi, int64_t t) {
  const int64_t ws = a.cum[a.nb];
  const int64_t z = ws > 0 ? t / ws : 0;
  const int64_t k = z >= a.rep ? (int64_t)a.rep * a.nb
                               : z * a.nb + warp_lower_bound_i64(a.cum, 0, a.nb, t - z * ws);
  return min(max(k, lo), hi);
}

// The CTA's virtual block range [b0, b1): warps 0 and 1 search its two ends concurrently,
// broadcast in shared memory (the same result as sell_lower).
template <bool USE_TAB = true>
__device__ __forceinline__ void sell_cta_range(const SellArgs& a, int64_t& b0, int64_t& b1) {
  // plan-time table of the same search (full-range launches): one load instead of the 2 x 4
  // dependent probe rounds before the CTA streams anything
  if (USE_TAB && a.cta_tab && a.cta_tab_grid == (int32_t)gridDim.x) {
    b0 = __ldg(a.cta_tab + blockIdx.x);
    b1 = __ldg(a.cta_tab + blockIdx.x + 1);
    return;
  }
  __shared__ int64_t s_rng[2];
  const int warp = threadIdx.x >> 5;
  if (warp < 2) {
    const int64_t w0 = sell_work(a, a.blk_lo), W = sell_work(a, a.blk_hi) - w0;
    const int64_t t = w0 + W * (blockIdx.x + warp) / gridDim.x;
    int64_t v;
    if (warp == 1 && blockIdx.x + 1 == gridDim.x) v = a.blk_hi;
    else v = sell_lower_warp(a, a.blk_lo, a.blk_hi, t);
    if ((threadIdx.x & 31) == 0) s_rng[warp] = v;
  }
  __syncthreads();
  b0 = s_rng[0];
  b1 = s_rng[1];
}

__global__ void sell_cta_table_kernel(SellArgs a, int grid, int64_t* tab) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // boundary, one per warp
  if (i > grid) return;
  const int64_t w0 = sell_work(a, a.blk_lo), W = sell_work(a, a.blk_hi) - w0;
  int64_t v;
  if (i == grid) v = a.blk_hi;
  else v = sell_lower_warp(a, a.blk_lo, a.blk_hi, w0 + W * i / grid);
  if ((threadIdx.x & 31) == 0) tab[i] = v;
}
cudaError_t launch_sell_cta_table(const SellArgs& a, int grid, int64_t* tab, cudaStream_t st) {
  SellArgs b = a;
  b.cta_tab = nullptr;
  sell_cta_table_kernel<<<(grid + 1 + 7) / 8, 256, 0, st>>>(b, grid, tab);
  return cudaGetLastError();
}

// LO: 0 = plain; 1 = + the lo parts gathered from global memory; 2 = + the lo window staged in
// shared memory after the hi one (a.lo_off floats on; when both fit: c2)
template <int UNR, bool STAGED, int NT = 512, bool HALF = false, bool DYN = true, int LO = 0>
__global__ void __launch_bounds__(NT, 1024 / NT) spmv16s_kernel(SellArgs a) {
  extern __shared__ float stage[];
  __shared__ int s_next;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = NT >> 5;
  pdl_trigger();  // the next kernel may take this SM as soon as this CTA leaves it
  int64_t b0, b1;
  sell_cta_range<LO != 2>(a, b0, b1);  // plan data only (LO == 2: no registers for the table path)
  pdl_wait();     // the gathered vector / partial sums are the previous kernel's
  if (LO == 0 && a.cta_prof && threadIdx.x == 0) {  // (the lo variants have no registers to spare)
    long long t;
    unsigned sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    a.cta_prof[3 * blockIdx.x] = t;
    a.cta_prof[3 * blockIdx.x + 2] = sm;
  }
  double sq = 0.0;  // static assignment: this thread's rows; DYN: the CTA's total (thread 0)
  for (int64_t it = b0; it < b1;) {
    const int64_t rz = it / a.nb, zb = rz * a.nb;  // repetition (slice-shared operator) and base
    const int z = a.blk_slice[it - zb];
    const int64_t it_end = min(b1, zb + a.zend[z]);
    const float* gbase = a.src + a.win_lo[z] + rz * a.rep_win;
    const float* lbase = LO != 0 ? a.src_lo + a.win_lo[z] + rz * a.rep_win : nullptr;
    const int64_t row_off = rz * a.rep_rows;
    if (STAGED || DYN) __syncthreads();  // previous segment done: window and counter reusable
    if (DYN && threadIdx.x == 0) s_next = nwarps;
    if constexpr (STAGED) stage_window(stage, gbase, HALF ? min(a.win_len[z], a.part_len) : a.win_len[z]);
    if constexpr (LO == 2) stage_window(stage + a.lo_off, lbase, a.win_len[z]);
    if (STAGED || DYN) __syncthreads();
    // DYN: warps take the segment's blocks from a shared counter (blocks are sorted by length
    // inside a slice, so this is longest-first list scheduling); the next block's descriptors are
    // loaded while the current block streams
    int64_t k = it + warp;
    int64_t off = 0;
    int K = 0, row = -1;
    if (k < it_end) {
      off = a.blk_off[k - zb];
      K = a.blk_k[k - zb];
      row = a.perm[(k - zb) * 32 + lane];
    }
    while (k < it_end) {
      int64_t kn;
      if constexpr (DYN) {
        int nx = 0;
        if (lane == 0) nx = atomicAdd(&s_next, 1);
        kn = it + __shfl_sync(0xffffffffu, nx, 0);
      } else {
        kn = k + nwarps;
      }
      int64_t off_n = 0;
      int K_n = 0, row_n = -1;
      if (kn < it_end) {
        off_n = a.blk_off[kn - zb];
        K_n = a.blk_k[kn - zb];
        row_n = a.perm[(kn - zb) * 32 + lane];
      }
      const uint16_t* cp = a.col16 + (off * 32 + lane) * 8;
      const float* vp = a.val + (off * 32 + lane) * 8;
      double acc = (a.acc_in && row >= 0) ? a.acc_in[row + row_off] : 0.0;
      int s = 0;
      for (; s + UNR <= K; s += UNR) {
        int4 c[UNR];
        float4 va[UNR], vb[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + (s + u) * 256));
          va[u] = ld_stream_f4(vp + (s + u) * 256);
          vb[u] = ld_stream_f4(vp + (s + u) * 256 + 4);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          acc += HALF ? chunk8_sum_part(c[u], va[u], vb[u], stage, gbase, a.part_len)
                      : chunk8_sum<STAGED>(c[u], va[u], vb[u], stage, gbase);
          if constexpr (LO == 1) acc += chunk8_sum_lo(c[u], va[u], vb[u], lbase);
          if constexpr (LO == 2) acc += chunk8_sum<true>(c[u], va[u], vb[u], stage + a.lo_off, lbase);
        }
      }
      for (; s < K; ++s) {
        const int4 c0 = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + s * 256));
        const float4 va0 = ld_stream_f4(vp + s * 256);
        const float4 vb0 = ld_stream_f4(vp + s * 256 + 4);
        acc += HALF ? chunk8_sum_part(c0, va0, vb0, stage, gbase, a.part_len)
                    : chunk8_sum<STAGED>(c0, va0, vb0, stage, gbase);
        if constexpr (LO == 1) acc += chunk8_sum_lo(c0, va0, vb0, lbase);
        if constexpr (LO == 2) acc += chunk8_sum<true>(c0, va0, vb0, stage + a.lo_off, lbase);
      }
      double q = 0.0;
      if (row >= 0 && a.acc_out) {
        a.acc_out[row + row_off] = acc;
      } else if (row >= 0) {
        const int64_t orow = row + row_off;
        if (a.b) {
          const double r = acc - (double)__ldg(a.b + orow);
          const float rh = (float)r;
          a.out[orow] = rh;
          if (a.out_lo) a.out_lo[orow] = (float)(r - (double)rh);
          q = r * r;
        } else {
          a.out[orow] = (float)acc;
        }
      }
      if (a.scal) {
        if constexpr (DYN) {  // per-block sum in a fixed lane order, summed in block order below
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) q += __shfl_xor_sync(0xffffffffu, q, d);
          if (lane == 0) a.blk_sq[k] = q;
        } else {
          sq += q;
        }
      }
      k = kn;
      off = off_n;
      K = K_n;
      row = row_n;
    }
    it = it_end;
  }
  if (LO == 0 && a.cta_prof) {
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.cta_prof[3 * blockIdx.x + 1] = t;
    }
  }
  if (a.scal) {
    if constexpr (DYN) {  // the CTA's blocks in block order: deterministic whatever warp ran them
      __syncthreads();
      if (warp == 0) {
        double t = 0.0;
        for (int64_t k = b0 + lane; k < b1; k += 32) t += a.blk_sq[k];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
        if (lane == 0) sq = t;
      }
    }
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// Slice-shared operator, Z slices per pass (the SpMM form of f4): a group of Z consecutive
// slices applies the same stored blocks, so the CTA stages the Z slices' windows side by side
// (a.wstride floats apart) and every lane loads each chunk of its row once and gathers it
// against the Z windows, accumulating Z rows (slice zs0 + zz, row row + (zs0 + zz) rep_rows).
// Per slice the chunk sums and their order are those of spmv16s_kernel (bitwise the same rows).
// Virtual block k: stored block k % nb of slice group k / nb (a.rep groups of a.zgroup slices,
// the last one possibly partial: a.rep_total slices).
template <int Z, int UNR, int NT = 1024>
__global__ void __launch_bounds__(NT, 1024 / NT) spmv16z_kernel(SellArgs a) {
  extern __shared__ float stage[];
  __shared__ int s_next;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = NT >> 5;
  pdl_trigger();  // launched through launch_pdl like spmv16s_kernel: the wait is mandatory
  int64_t b0, b1;
  sell_cta_range(a, b0, b1);
  pdl_wait();
  for (int64_t it = b0; it < b1;) {
    const int64_t rz = it / a.nb, zb = rz * a.nb;
    const int z = a.blk_slice[it - zb];
    const int64_t it_end = min(b1, zb + a.zend[z]);
    const int64_t zs0 = rz * Z;  // first slice of the group
    const int zc = (int)(a.rep_total - zs0 < Z ? a.rep_total - zs0 : Z);
    __syncthreads();
    if (threadIdx.x == 0) s_next = nwarps;
    {
      const int len = a.win_len[z];
      const uint32_t dstep = (uint32_t)(NT + NT / 32) * 4u;
      for (int zz = 0; zz < zc; ++zz) {
        const float* src = a.src + a.win_lo[z] + (zs0 + zz) * a.rep_win + threadIdx.x;
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(stage + zz * a.wstride + swz(threadIdx.x));
        int n = len > (int)threadIdx.x ? (len - (int)threadIdx.x + NT - 1) / NT : 0;
#pragma unroll 4
        for (; n > 0; --n, dst += dstep, src += NT)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    int64_t k = it + warp;
    int64_t off = 0;
    int K = 0, row = -1;
    if (k < it_end) {
      off = a.blk_off[k - zb];
      K = a.blk_k[k - zb];
      row = a.perm[(k - zb) * 32 + lane];
    }
    while (k < it_end) {
      int nx = 0;
      if (lane == 0) nx = atomicAdd(&s_next, 1);
      const int64_t kn = it + __shfl_sync(0xffffffffu, nx, 0);
      int64_t off_n = 0;
      int K_n = 0, row_n = -1;
      if (kn < it_end) {
        off_n = a.blk_off[kn - zb];
        K_n = a.blk_k[kn - zb];
        row_n = a.perm[(kn - zb) * 32 + lane];
      }
      const uint16_t* cp = a.col16 + (off * 32 + lane) * 8;
      const float* vp = a.val + (off * 32 + lane) * 8;
      double acc[Z];
#pragma unroll
      for (int zz = 0; zz < Z; ++zz) acc[zz] = 0.0;
      auto chunk = [&](const int4 c, const float4 v0, const float4 v1) {
#pragma unroll
        for (int zz = 0; zz < Z; ++zz)
          if (zz < zc) acc[zz] += chunk8_sum<true>(c, v0, v1, stage + zz * a.wstride, nullptr);
      };
      int s = 0;
      for (; s + UNR <= K; s += UNR) {
        int4 c[UNR];
        float4 va[UNR], vb[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + (s + u) * 256));
          va[u] = ld_stream_f4(vp + (s + u) * 256);
          vb[u] = ld_stream_f4(vp + (s + u) * 256 + 4);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) chunk(c[u], va[u], vb[u]);
      }
      for (; s < K; ++s) {
        const int4 c0 = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + s * 256));
        const float4 va0 = ld_stream_f4(vp + s * 256);
        const float4 vb0 = ld_stream_f4(vp + s * 256 + 4);
        chunk(c0, va0, vb0);
      }
      double q = 0.0;
      if (row >= 0) {
#pragma unroll
        for (int zz = 0; zz < Z; ++zz) {
          if (zz < zc) {
            const int64_t orow = row + (zs0 + zz) * a.rep_rows;
            if (a.b) {
              const double r = acc[zz] - (double)__ldg(a.b + orow);
              const float rh = (float)r;
              a.out[orow] = rh;
              if (a.out_lo) a.out_lo[orow] = (float)(r - (double)rh);
              q += r * r;
            } else {
              a.out[orow] = (float)acc[zz];
            }
          }
        }
      }
      if (a.scal) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) q += __shfl_xor_sync(0xffffffffu, q, d);
        if (lane == 0) a.blk_sq[k] = q;
      }
      k = kn;
      off = off_n;
      K = K_n;
      row = row_n;
    }
    it = it_end;
  }
  if (a.scal) {
    double sq = 0.0;
    __syncthreads();
    if (warp == 0) {
      double t = 0.0;
      for (int64_t k = b0 + lane; k < b1; k += 32) t += a.blk_sq[k];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
      if (lane == 0) sq = t;
    }
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// Sliced ELL over int32 global columns (non-separable geometry; spmv32s_kernel): blocks of 32
// consecutive rows (no sorting), two block modes chosen per block at create time by which
// gather order touches fewer cache lines:
//  * lane mode (blk_k >= 0): one row per lane, rows padded with zero 4-entry chunks to the
//    block's longest, stored [step][lane][4]: at each step the 32 lanes gather the s-th entries of
//    32 neighbouring rows (A^T: neighbouring voxels' rays, i.e. neighbouring ray ids; A: parallel
//    rays whose neighbours are along x);
//  * row mode (blk_k < 0, -blk_k chunks): the block's rows back to back (row starts in
//    a.row_start, in chunks), 8 lanes per row and 4 rows at a time, as the per-row kernel (rays
//    running along x: consecutive entries are neighbouring voxels).
// Offsets are in 4-entry chunks.  The gathers go through L1 (__ldg); warps take blocks from a
// shared counter; per-block sums as spmv16s_kernel (deterministic).
// L2 cache policies (L2H, spmv32s_kernel): bit 0 = the matrix stream is evict-first, bit 1 = the
// gathered vector is evict-last.  With z-ordered blocks (make_sell32) the gathered sub-volume in
// flight is a ~60-slice band (~16 MB at c5), but between two uses of an x line the grid streams
// ~5 GB of matrix through L2, which evicts it under plain LRU (profiles/r02: 25.0 GB of DRAM
// reads per c5 A pass against 21.4 GB algorithmic).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int4 ld_stream_i4_pol(const int32_t* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld_stream_f4_pol(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_gather_pol(const float* p, uint64_t pol) {
  float r;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return r;
}

template <int UNR, int NT = 512, int L2H = 0, bool LO = false>
__global__ void __launch_bounds__(NT, 1024 / NT) spmv32s_kernel(SellArgs a) {
  __shared__ int s_next;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = NT >> 5;
  uint64_t pol_s = 0, pol_g = 0;
  if constexpr (L2H & 1) pol_s = l2_policy_evict_first();
  if constexpr (L2H & 2) pol_g = l2_policy_evict_last();
  auto ldi = [&](const int32_t* p) {
    if constexpr (L2H & 1) return ld_stream_i4_pol(p, pol_s);
    else return ld_stream_i4(p);
  };
  auto ldf = [&](const float* p) {
    if constexpr (L2H & 1) return ld_stream_f4_pol(p, pol_s);
    else return ld_stream_f4(p);
  };
  auto ldg = [&](const float* p) {
    if constexpr (L2H & 2) return ld_gather_pol(p, pol_g);
    else return __ldg(p);
  };
  // The CTA's blocks as a sequence j = 0, 1, ..: contiguous (ilv = 0: [b0, b1)) or interleaved
  // (chunk q = blockIdx.x + (j / ilv) G of ilv blocks); blk(j) maps it to the stored block.
  int64_t b0, b1;
  const int64_t ilv = a.ilv;
  if (ilv > 0) {
    const int64_t nch = (a.blk_hi - a.blk_lo + ilv - 1) / ilv;  // chunks
    const int64_t mine = nch > blockIdx.x ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    b0 = 0;
    b1 = mine * ilv;  // an upper bound: the last chunk may be short (blk() >= blk_hi: skipped)
  } else {
    sell_cta_range(a, b0, b1);
  }
  auto blk = [&](int64_t j) -> int64_t {
    if (ilv <= 0) return j;
    const int64_t q = blockIdx.x + (j / ilv) * (int64_t)gridDim.x;
    return a.blk_lo + q * ilv + j % ilv;
  };
  if (threadIdx.x == 0) s_next = nwarps;
  __syncthreads();
  auto gather4 = [&](const int4 c, const float4 v) {
    const double p0 = (double)v.x * (double)ldg(a.src + c.x);
    const double p1 = (double)v.y * (double)ldg(a.src + c.y);
    const double p2 = (double)v.z * (double)ldg(a.src + c.z);
    const double p3 = (double)v.w * (double)ldg(a.src + c.w);
    double t = (p0 + p1) + (p2 + p3);
    if constexpr (LO) {  // extended-precision source: + the lo parts
      const double q0 = (double)v.x * (double)__ldg(a.src_lo + c.x);
      const double q1 = (double)v.y * (double)__ldg(a.src_lo + c.y);
      const double q2 = (double)v.z * (double)__ldg(a.src_lo + c.z);
      const double q3 = (double)v.w * (double)__ldg(a.src_lo + c.w);
      t += (q0 + q1) + (q2 + q3);
    }
    return t;
  };
  auto emit = [&](int64_t row, double acc) -> double {
    if (a.b) {
      const double r = acc - (double)__ldg(a.b + row);
      const float rh = (float)r;
      a.out[row] = rh;
      if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);
      return r * r;
    }
    if (a.out_peer) {  // fused reduce-scatter: straight into the owner's inbox (peer memory)
      int o = 0;
      while (o + 1 < a.n_out && row >= a.out_bounds[o + 1]) ++o;
      a.out_peer[o][row] = (float)acc;
      return 0.0;
    }
    a.out[row] = (float)acc;
    return 0.0;
  };
  // j: position in the CTA's sequence; k = blk(j) the stored block (k >= blk_hi: past the end)
  int64_t j = b0 + warp;
  int64_t k = blk(j);
  int64_t off = 0;
  int K = 0, row = -1;
  if (j < b1 && k < a.blk_hi) {
    off = a.blk_off[k];
    K = a.blk_k[k];
    row = a.perm[k * 32 + lane];
  }
  while (j < b1) {
    int nx = 0;
    if (lane == 0) nx = atomicAdd(&s_next, 1);
    const int64_t jn = b0 + __shfl_sync(0xffffffffu, nx, 0);
    const int64_t kn = blk(jn);
    int64_t off_n = 0;
    int K_n = 0, row_n = -1;
    if (jn < b1 && kn < a.blk_hi) {
      off_n = a.blk_off[kn];
      K_n = a.blk_k[kn];
      row_n = a.perm[kn * 32 + lane];
    }
    if (k >= a.blk_hi) {  // past the last (short) chunk: nothing to do
      j = jn;
      k = kn;
      off = off_n;
      K = K_n;
      row = row_n;
      continue;
    }
    double q = 0.0;
    if (K >= 0) {  // lane mode
      const int32_t* cp = a.col32 + (off + lane) * 4;
      const float* vp = a.val + (off + lane) * 4;
      double acc = 0.0;
      int s = 0;
      for (; s + UNR <= K; s += UNR) {
        int4 c[UNR];
        float4 v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = ldi(cp + (s + u) * 128);
          v[u] = ldf(vp + (s + u) * 128);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc += gather4(c[u], v[u]);
      }
      for (; s < K; ++s) acc += gather4(ldi(cp + s * 128), ldf(vp + s * 128));
      if (row >= 0) q = emit(row, acc);
    } else {  // row mode: 8 lanes per row, 4 rows at a time
      const int grp = lane >> 3, gl = lane & 7;
      const int64_t my_start = a.row_start[k * 32 + lane];  // chunks from the block start
      const int my_n = row >= 0 ? (int)((a.rp[row + 1] - a.rp[row] + 3) >> 2) : 0;
      for (int i0 = 0; i0 < 32; i0 += 4) {
        const int ri = __shfl_sync(0xffffffffu, row, i0 + grp);
        const int64_t si = off + __shfl_sync(0xffffffffu, my_start, i0 + grp);
        const int ni = __shfl_sync(0xffffffffu, my_n, i0 + grp);
        double acc = 0.0;
        int c = gl;
        for (; c + 8 < ni; c += 16) {
          const int4 c0 = ldi(a.col32 + (si + c) * 4);
          const float4 v0 = ldf(a.val + (si + c) * 4);
          const int4 c1 = ldi(a.col32 + (si + c + 8) * 4);
          const float4 v1 = ldf(a.val + (si + c + 8) * 4);
          acc += gather4(c0, v0);
          acc += gather4(c1, v1);
        }
        if (c < ni) acc += gather4(ldi(a.col32 + (si + c) * 4), ldf(a.val + (si + c) * 4));
        acc = group_sum<8>(acc);
        if (gl == 0 && ri >= 0) q += emit(ri, acc);
      }
    }
    if (a.scal) {
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) q += __shfl_xor_sync(0xffffffffu, q, d);
      if (lane == 0) a.blk_sq[k] = q;
    }
    j = jn;
    k = kn;
    off = off_n;
    K = K_n;
    row = row_n;
  }
  if (a.scal) {
    double sq = 0.0;
    __syncthreads();
    if (warp == 0) {  // the CTA's blocks in its sequence order: deterministic
      double t = 0.0;
      for (int64_t jj = b0 + lane; jj < b1; jj += 32) {
        const int64_t kk = blk(jj);
        if (kk < a.blk_hi) t += a.blk_sq[kk];
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
      if (lane == 0) sq = t;
    }
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// Block modes (one warp per block, lane = row): cache-line changes between the gathers a warp
// issues together, in lane mode (lane l vs l-1 at the same entry) and in row mode (entry e vs
// e-1 of one row); 1 = row mode when it changes lines less often.
__global__ void sell32_mode_kernel(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* col,
                                   uint8_t* mode, int bias_pct) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= nblk) return;
  const int64_t r = j * 32 + lane;
  const int64_t s = r < rows ? rp[r] : 0, len = r < rows ? rp[r + 1] - s : 0;
  int64_t mn = len;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
  int lane_chg = 0, row_chg = 0;
  int prev = mn > 0 ? (col[s] >> 5) : 0;
  for (int64_t e = 0; e < mn; ++e) {
    const int line = col[s + e] >> 5;  // 128-byte line of the gathered fp32 value
    const int up = __shfl_up_sync(0xffffffffu, line, 1);
    if (lane > 0 && up != line) ++lane_chg;
    if (e > 0 && line != prev) ++row_chg;
    prev = line;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    lane_chg += __shfl_xor_sync(0xffffffffu, lane_chg, d);
    row_chg += __shfl_xor_sync(0xffffffffu, row_chg, d);
  }
  if (lane == 0) mode[j] = (uint8_t)((int64_t)row_chg * 100 < (int64_t)lane_chg * bias_pct ? 1 : 0);
}

__global__ void sell32_zkey_kernel(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* col,
                                   int64_t plane, int32_t* key) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nblk) return;
  int32_t z = -1;
  const int64_t r_lo = j * 32, r_hi = min(rows, r_lo + 32);
  // the middle row, else the nearest nonempty one
  for (int64_t d = 0; d < 32 && z < 0; ++d) {
    for (int sgn = 0; sgn < 2 && z < 0; ++sgn) {
      const int64_t r = r_lo + 16 + (sgn ? -d - 1 : d);
      if (r < r_lo || r >= r_hi) continue;
      const int64_t s = rp[r], e = rp[r + 1];
      if (e > s) z = (int32_t)(col[s + (e - s) / 2] / plane);
    }
  }
  key[j] = z;
}

cudaError_t launch_sell32_zkey(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* col,
                               int64_t plane, int32_t* key, cudaStream_t st) {
  if (nblk <= 0) return cudaSuccess;
  sell32_zkey_kernel<<<(unsigned)((nblk + 255) / 256), 256, 0, st>>>(nblk, rows, rp, col, plane, key);
  return cudaGetLastError();
}

cudaError_t launch_sell32_mode(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* col,
                               uint8_t* mode, cudaStream_t st, int bias_pct) {
  if (nblk <= 0) return cudaSuccess;
  sell32_mode_kernel<<<(unsigned)((nblk * 32 + 255) / 256), 256, 0, st>>>(nblk, rows, rp, col, mode,
                                                                         bias_pct);
  return cudaGetLastError();
}

template <int L2H>
static const void* spmv32s_ptr_l2(int unroll, int block) {
  if (block == 1024)
    return unroll >= 3 ? (const void*)spmv32s_kernel<3, 1024, L2H>
                       : unroll == 2 ? (const void*)spmv32s_kernel<2, 1024, L2H>
                                     : (const void*)spmv32s_kernel<1, 1024, L2H>;
  return unroll >= 3 ? (const void*)spmv32s_kernel<3, 512, L2H>
                     : unroll == 2 ? (const void*)spmv32s_kernel<2, 512, L2H>
                                   : (const void*)spmv32s_kernel<1, 512, L2H>;
}
static const void* spmv32s_ptr(int unroll, int block, int l2 = 0, bool lo = false) {
  if (lo)  // extended-precision source (no L2 policies)
    return block == 1024 ? (unroll >= 3 ? (const void*)spmv32s_kernel<3, 1024, 0, true>
                                        : (const void*)spmv32s_kernel<2, 1024, 0, true>)
                         : (unroll >= 3 ? (const void*)spmv32s_kernel<3, 512, 0, true>
                                        : (const void*)spmv32s_kernel<2, 512, 0, true>);
  switch (l2) {
    case 1: return spmv32s_ptr_l2<1>(unroll, block);
    case 2: return spmv32s_ptr_l2<2>(unroll, block);
    case 3: return spmv32s_ptr_l2<3>(unroll, block);
    default: return spmv32s_ptr_l2<0>(unroll, block);
  }
}

cudaError_t launch_spmv32s(const SellArgs& a, int unroll, int grid, cudaStream_t st, int block) {
  if (a.blk_hi <= a.blk_lo) return cudaSuccess;
  void* args[] = {const_cast<SellArgs*>(&a)};
  return cudaLaunchKernel(spmv32s_ptr(unroll, block, a.l2hint, a.src_lo != nullptr), dim3(grid),
                          dim3(block == 1024 ? 1024 : 512),
                          args, 0, st);
}

int spmv32s_occupancy(int unroll, int block) {
  int occ = 0;
  const void* k = spmv32s_ptr(unroll, block);
  ensure_smem_attr(k, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, block == 1024 ? 1024 : 512, 0);
  return occ > 0 ? occ : 1;
}

__global__ void sell_fill32_kernel(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                                   const int32_t* blk_k, const int64_t* row_start,
                                   const int64_t* rp, const int32_t* col, const float* val,
                                   int32_t* cols, float* vals) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nslots) return;
  const int row = perm[t];
  if (row < 0) return;
  const int64_t j = t >> 5, l = t & 31, s = rp[row], len = rp[row + 1] - s;
  const int64_t base = blk_off[j];
  const bool lane_mode = blk_k[j] >= 0;
  for (int64_t e = 0; e < len; ++e) {
    const int64_t d = lane_mode ? (base + (e >> 2) * 32 + l) * 4 + (e & 3)
                                : (base + row_start[t]) * 4 + e;
    cols[d] = col[s + e];
    vals[d] = val[s + e];
  }
}

cudaError_t launch_sell_fill32(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                               const int32_t* blk_k, const int64_t* row_start, const int64_t* rp,
                               const int32_t* col, const float* val, int32_t* cols, float* vals,
                               cudaStream_t st) {
  if (nslots <= 0) return cudaSuccess;
  sell_fill32_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(
      nslots, perm, blk_off, blk_k, row_start, rp, col, val, cols, vals);
  return cudaGetLastError();
}

// ------------------------------------------------ gather layouts of the non-separable A pass
// (c5; profiles/r02/c5_raw.csv: the pass is bound by L1TEX wavefronts, 88 % of peak, one per
// distinct 128-byte line a 32-lane gather touches).  The gathered point is kept in three layouts
// side by side, xs = [x | x_yx | x_b], and every block of 32 rays gathers from the one in which
// its lanes' simultaneous accesses fall into the fewest lines (scripts/c5_lines.py: 17.1 ->
// 8.4 lines per gather instruction on c5's views):
//   0  row-major (z, y, x): rays along y, neighbouring rays at neighbouring x;
//   1  (z, x, y), x and y swapped: rays along x;
//   2  8x4 bricks in each xy plane (z, y/4, x/8, y%4, x%8): oblique rays.
// The block's columns are stored as indices into xs (layout * N + position), its entries sorted
// by them, so the kernel is unchanged; the point is re-laid out before each A pass.
__host__ __device__ __forceinline__ int64_t layout_index(int L, int64_t j, int nx, int ny, int64_t N) {
  if (L == 0) return j;
  const int64_t plane = (int64_t)nx * ny;
  const int64_t z = j / plane, r = j - z * plane;
  const int64_t y = r / nx, x = r - y * nx;
  if (L == 1) return N + (z * nx + x) * ny + y;
  return 2 * N + ((z * (ny >> 2) + (y >> 2)) * (nx >> 3) + (x >> 3)) * 32 + (y & 3) * 8 + (x & 7);
}

// The re-layout before each A pass (3N < 2^31: 32-bit indices).  x_yx: per z-slice a 32 x 32
// tiled transpose through shared memory (coalesced reads and writes); bricks: one warp per 8 x 4
// brick (a 128-byte line written whole, four 32-byte row pieces read).  Row-major: a copy.
__global__ void relayout_yx_kernel(const float* __restrict__ x, float* __restrict__ xt, int nx, int ny) {
  __shared__ float t[32][33];
  const int z = blockIdx.z;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const float* xz = x + (size_t)z * nx * ny;
  float* tz = xt + (size_t)z * nx * ny;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int y = by + i, xx = bx + threadIdx.x;
    if (y < ny && xx < nx) t[i][threadIdx.x] = __ldg(xz + y * nx + xx);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int xx = bx + i, y = by + threadIdx.x;
    if (y < ny && xx < nx) tz[xx * ny + y] = t[threadIdx.x][i];
  }
}
__global__ void relayout_brick_kernel(const float* __restrict__ x, float* __restrict__ xb, int nx, int ny,
                                      int nbricks) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nbricks) return;
  const int t = threadIdx.x & 31;
  const int nbx = nx >> 3, nby = ny >> 2;
  const int bx = b % nbx, by = (b / nbx) % nby, z = b / (nbx * nby);
  xb[(size_t)b * 32 + t] = __ldg(x + ((size_t)z * ny + by * 4 + (t >> 3)) * nx + bx * 8 + (t & 7));
}

cudaError_t launch_relayout(const float* x, float* xs, int nx, int ny, int64_t N, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(xs, x, sizeof(float) * N, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  const int nz = (int)(N / ((int64_t)nx * ny));
  relayout_yx_kernel<<<dim3((nx + 31) / 32, (ny + 31) / 32, nz), dim3(32, 8), 0, st>>>(x, xs + N, nx, ny);
  const int nbricks = (int)(N / 32);
  relayout_brick_kernel<<<(nbricks + 7) / 8, 256, 0, st>>>(x, xs + 2 * N, nx, ny, nbricks);
  return cudaGetLastError();
}

// Bitonic sort of n <= cap (key, payload) pairs in shared memory by one warp (padding: +inf keys)
template <bool PAY>
__device__ void warp_sort_pairs(int64_t* key, float* pay, int n, int lane) {
  int P = 32;
  while (P < n) P <<= 1;
  for (int i = n + lane; i < P; i += 32) key[i] = INT64_MAX;
  __syncwarp();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const int64_t a = key[i], b = key[l];
          if ((a > b) == up) {
            key[i] = b;
            key[l] = a;
            if constexpr (PAY) {
              const float t = pay[i];
              pay[i] = pay[l];
              pay[l] = t;
            }
          }
        }
      }
      __syncwarp();
    }
  }
}

constexpr int kLayoutCap = 1024;  // longest row the layout kernels sort (longer: layout 0)

// Phase 1: the rows' columns mapped to layout L and sorted, into scol (same row_ptr); rows longer
// than kLayoutCap are flagged in bad[row / 32].  One warp per row, 8 warps per CTA.
__global__ void __launch_bounds__(256) layout_sort_rows_kernel(int64_t rows, const int64_t* rp,
                                                               const int32_t* col, int L, int nx,
                                                               int ny, int64_t N, int32_t* scol,
                                                               uint8_t* bad) {
  extern __shared__ int64_t lsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t* key = lsm + warp * kLayoutCap;
  for (int64_t r = blockIdx.x * 8 + warp; r < rows; r += (int64_t)gridDim.x * 8) {
    const int64_t s = rp[r];
    const int n = (int)(rp[r + 1] - s);
    if (n > kLayoutCap) {
      if (lane == 0) bad[r >> 5] = 1;
      continue;
    }
    for (int e = lane; e < n; e += 32) key[e] = layout_index(L, col[s + e], nx, ny, N);
    __syncwarp();
    warp_sort_pairs<false>(key, nullptr, n, lane);
    for (int e = lane; e < n; e += 32) scol[s + e] = (int32_t)key[e];
    __syncwarp();
  }
}

// Distinct 128-byte lines per 32-lane gather of a block of 32 consecutive rows (lane = row) in
// spmv32s_kernel's two walks: lane mode (lane l at entry 4s + k of its row) and row mode (4 rows
// at a time, lane g of a row at entries 4 (g + 8 i) + k).  Pads are not counted.
__device__ __forceinline__ int distinct_lines(int64_t line, bool act) {
  // a lane leads its value when no lower active lane holds it (shuffles; __match_any_sync in this
  // loop hung on sm_100a)
  const int lane = threadIdx.x & 31;
  const unsigned am = __ballot_sync(0xffffffffu, act);
  const int32_t lo = (int32_t)line, hi = (int32_t)(line >> 32);
  bool leader = act;
  for (int d = 0; d < 31; ++d) {
    const int32_t vlo = __shfl_sync(0xffffffffu, lo, d), vhi = __shfl_sync(0xffffffffu, hi, d);
    if (d < lane && ((am >> d) & 1u) && vlo == lo && vhi == hi) leader = false;
  }
  return __popc(__ballot_sync(0xffffffffu, leader));
}
__global__ void layout_count_kernel(int64_t nblk, int64_t rows, const int64_t* rp,
                                    const int32_t* scol, int64_t* cnt_lane, int64_t* cnt_row) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= nblk) return;  // whole warps exit together
  const int64_t r = j * 32 + lane;
  const int64_t s = r < rows ? rp[r] : 0;
  const int n = r < rows ? (int)(rp[r + 1] - s) : 0;
  int mx = n;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  int64_t cl = 0, cr = 0;
  for (int e = 0; e < mx; ++e) {
    const bool act = e < n;
    cl += distinct_lines(act ? (int64_t)(scol[s + e] >> 5) : 0, act);
  }
  for (int i0 = 0; i0 < 32; i0 += 4) {
    const int ri = i0 + (lane >> 3), g = lane & 7;
    const int ni = __shfl_sync(0xffffffffu, n, ri);
    const int64_t si = __shfl_sync(0xffffffffu, s, ri);
    int mxi = ni;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mxi = max(mxi, __shfl_xor_sync(0xffffffffu, mxi, d));
    const int chunks = (mxi + 3) >> 2;
    for (int c0 = 0; c0 < chunks; c0 += 8) {
      const int c = c0 + g;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = 4 * c + k;
        const bool act = e < ni;
        cr += distinct_lines(act ? (int64_t)(scol[si + e] >> 5) : 0, act);
      }
    }
  }
  if (lane == 0) {
    cnt_lane[j] = cl;
    cnt_row[j] = cr;
  }
}

cudaError_t launch_layout_sort_rows(int64_t rows, const int64_t* rp, const int32_t* col, int L, int nx,
                                    int ny, int64_t N, int32_t* scol, uint8_t* bad, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const size_t smem = sizeof(int64_t) * kLayoutCap * 8;
  cudaError_t e = ensure_smem_attr((const void*)layout_sort_rows_kernel, smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)std::min<int64_t>((rows + 7) / 8, 148 * 8);
  layout_sort_rows_kernel<<<grid, 256, smem, st>>>(rows, rp, col, L, nx, ny, N, scol, bad);
  return cudaGetLastError();
}
cudaError_t launch_layout_count(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* scol,
                                int64_t* cnt_lane, int64_t* cnt_row, cudaStream_t st) {
  if (nblk <= 0) return cudaSuccess;
  layout_count_kernel<<<(unsigned)((nblk * 32 + 255) / 256), 256, 0, st>>>(nblk, rows, rp, scol,
                                                                          cnt_lane, cnt_row);
  return cudaGetLastError();
}

// Phase 3: sell_fill32 with each stored block's layout: one warp per slot (stored block j, lane
// l): its row's columns mapped to layout[j] and sorted with the values, written to the block's
// lane- or row-mode positions.
__global__ void __launch_bounds__(256) sell_fill32_layout_kernel(
    int64_t nslots, const int32_t* perm, const int64_t* blk_off, const int32_t* blk_k,
    const int64_t* row_start, const uint8_t* layout, const int64_t* rp, const int32_t* col,
    const float* val, int nx, int ny, int64_t N, int32_t* cols, float* vals) {
  extern __shared__ int64_t lsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t* key = lsm + warp * kLayoutCap;
  float* pay = reinterpret_cast<float*>(lsm + 8 * kLayoutCap) + warp * kLayoutCap;
  for (int64_t t = blockIdx.x * 8 + warp; t < nslots; t += (int64_t)gridDim.x * 8) {
    const int row = perm[t];
    if (row < 0) continue;
    const int64_t j = t >> 5, l = t & 31, s = rp[row];
    const int n = (int)(rp[row + 1] - s);
    const int64_t base = blk_off[j];
    const bool lane_mode = blk_k[j] >= 0;
    const int L = layout[j];
    auto dst = [&](int e) {
      return lane_mode ? (base + (e >> 2) * 32 + l) * 4 + (e & 3) : (base + row_start[t]) * 4 + e;
    };
    if (L == 0 || n > kLayoutCap) {  // the stored order (layout 0 sorts to itself)
      for (int e = lane; e < n; e += 32) {
        cols[dst(e)] = col[s + e];
        vals[dst(e)] = val[s + e];
      }
      continue;
    }
    for (int e = lane; e < n; e += 32) {
      key[e] = layout_index(L, col[s + e], nx, ny, N);
      pay[e] = val[s + e];
    }
    __syncwarp();
    warp_sort_pairs<true>(key, pay, n, lane);
    for (int e = lane; e < n; e += 32) {
      cols[dst(e)] = (int32_t)key[e];
      vals[dst(e)] = pay[e];
    }
    __syncwarp();
  }
}

cudaError_t launch_sell_fill32_layout(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                                      const int32_t* blk_k, const int64_t* row_start,
                                      const uint8_t* layout, const int64_t* rp, const int32_t* col,
                                      const float* val, int nx, int ny, int64_t N, int32_t* cols,
                                      float* vals, cudaStream_t st) {
  if (nslots <= 0) return cudaSuccess;
  const size_t smem = (sizeof(int64_t) + sizeof(float)) * kLayoutCap * 8;
  cudaError_t e = ensure_smem_attr((const void*)sell_fill32_layout_kernel, smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)std::min<int64_t>((nslots + 7) / 8, 148 * 8);
  sell_fill32_layout_kernel<<<grid, 256, smem, st>>>(nslots, perm, blk_off, blk_k, row_start, layout,
                                                     rp, col, val, nx, ny, N, cols, vals);
  return cudaGetLastError();
}

template <class F>
static cudaError_t dispatch16s(const SellVariant& v, F&& f) {
  if (v.zgroup == 2) return f(spmv16z_kernel<2, 1>);
  if (v.zgroup == 3) return f(spmv16z_kernel<3, 1>);
  if (v.zgroup == 4) return f(spmv16z_kernel<4, 1>);
  if (!v.dyn) {
    if (v.half) return f(spmv16s_kernel<2, true, 1024, true, false>);
    if (v.staged) return v.block == 1024 ? f(spmv16s_kernel<3, true, 1024, false, false>)
                                         : f(spmv16s_kernel<3, true, 512, false, false>);
    return f(spmv16s_kernel<3, false, 512, false, false>);
  }
  if (v.unroll == 3) {
    if (v.half) return f(spmv16s_kernel<3, true, 1024, true>);
    if (v.staged) return v.block == 1024 ? f(spmv16s_kernel<3, true, 1024>)
                                         : f(spmv16s_kernel<3, true, 512>);
    return v.block == 1024 ? f(spmv16s_kernel<3, false, 1024>) : f(spmv16s_kernel<3, false, 512>);
  }
  if (v.half) return v.block == 1024 ? f(spmv16s_kernel<2, true, 1024, true>)
                                     : f(spmv16s_kernel<2, true, 512, true>);
  if (v.staged) return v.block == 1024 ? f(spmv16s_kernel<2, true, 1024>)
                                       : f(spmv16s_kernel<2, true, 512>);
  return v.block == 1024 ? f(spmv16s_kernel<2, false, 1024>) : f(spmv16s_kernel<2, false, 512>);
}

// extended-precision source (a.src_lo): the default sliced-ELL configurations only (DYN, two
// steps in flight, one slice per pass); spmv16s_lo_ok() tells the planner
template <class F>
static cudaError_t dispatch16s_lo(const SellVariant& v, bool lo_staged, F&& f) {
  if (v.staged && lo_staged)
    return v.block == 1024 ? f(spmv16s_kernel<2, true, 1024, false, true, 2>)
                           : f(spmv16s_kernel<2, true, 512, false, true, 2>);
  if (v.staged) return v.block == 1024 ? f(spmv16s_kernel<2, true, 1024, false, true, 1>)
                                       : f(spmv16s_kernel<2, true, 512, false, true, 1>);
  return v.block == 1024 ? f(spmv16s_kernel<2, false, 1024, false, true, 1>)
                         : f(spmv16s_kernel<2, false, 512, false, true, 1>);
}
// (not the partly staged window: its lo instantiation spilled 312 bytes)
bool spmv16s_lo_ok(const SellVariant& v) {
  return v.zgroup == 1 && v.dyn && v.unroll == 2 && !v.half;
}

cudaError_t launch_spmv16s(const SellArgs& a, const SellVariant& v, int grid, size_t smem,
                           cudaStream_t st) {
  if (a.blk_hi <= a.blk_lo) return cudaSuccess;
  if (a.src_lo) {
    if (!spmv16s_lo_ok(v)) return cudaErrorNotSupported;
    // the lo window staged too when both windows fit (a.lo_off > 0 set by the caller)
    const size_t sm = a.lo_off > 0 ? smem + sizeof(float) * (size_t)a.lo_off : smem;
    return dispatch16s_lo(v, a.lo_off > 0, [&](auto k) -> cudaError_t {
      cudaError_t e = ensure_smem_attr((const void*)k, sm);
      if (e != cudaSuccess) return e;
      return launch_pdl(k, dim3(grid), dim3(v.block), sm, st, a);
    });
  }
  return dispatch16s(v, [&](auto k) -> cudaError_t {
    cudaError_t e = ensure_smem_attr((const void*)k, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(k, dim3(grid), dim3(v.block), smem, st, a);
  });
}

int spmv16s_occupancy(const SellVariant& v, size_t smem) {
  int occ = 0;
  dispatch16s(v, [&](auto k) -> cudaError_t {
    ensure_smem_attr((const void*)k, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, v.block, smem);
  });
  return occ > 0 ? occ : 1;
}

// Sliced-ELL copy: lane l of block j holds row perm[32 j + l]; its entry e goes to chunk step
// off_j + e / 8, lane l, position e % 8.  One thread per (block, lane); zero pads by memset.
// Column parts: lane l's row contributes its entries [lo_off[row], hi_off[row]) (null: 0 / the
// row's length) with the part's window start coff subtracted from the 16-bit offsets.
__global__ void sell_fill_kernel(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                                 const int64_t* rp, const int32_t* lo_off, const int32_t* hi_off,
                                 uint16_t coff, const uint16_t* col16, const float* val,
                                 uint16_t* col16s, float* vals) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nslots) return;
  const int row = perm[t];
  if (row < 0) return;
  const int64_t j = t >> 5, l = t & 31;
  const int64_t e0 = lo_off ? lo_off[row] : 0;
  const int64_t e1 = hi_off ? hi_off[row] : rp[row + 1] - rp[row];
  const int64_t s = rp[row] + e0, len = e1 - e0;
  const int64_t base = blk_off[j];
  for (int64_t e = 0; e < len; ++e) {
    const int64_t d = ((base + (e >> 3)) * 32 + l) * 8 + (e & 7);
    col16s[d] = (uint16_t)(col16[s + e] - coff);
    vals[d] = val[s + e];
  }
}

cudaError_t launch_sell_fill(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                             const int64_t* rp, const int32_t* lo_off, const int32_t* hi_off,
                             uint16_t coff, const uint16_t* col16, const float* val,
                             uint16_t* col16s, float* vals, cudaStream_t st) {
  if (nslots <= 0) return cudaSuccess;
  sell_fill_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(
      nslots, perm, blk_off, rp, lo_off, hi_off, coff, col16, val, col16s, vals);
  return cudaGetLastError();
}

__global__ void sell_split_kernel(int64_t rows, const int64_t* rp, const uint16_t* col16, int h,
                                  int32_t* split) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int64_t lo = rp[r], hi = rp[r + 1];
  const int64_t s = lo;
  while (lo < hi) {  // columns ascend within a row
    const int64_t mid = (lo + hi) >> 1;
    if ((int)col16[mid] < h) lo = mid + 1;
    else hi = mid;
  }
  split[r] = (int32_t)(lo - s);
}

cudaError_t launch_sell_split(int64_t rows, const int64_t* rp, const uint16_t* col16, int h,
                              int32_t* split, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  sell_split_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(rows, rp, col16, h, split);
  return cudaGetLastError();
}

// Padded-row int32 kernel (global columns: non-separable geometry or TVR_IDX16=0): rows start on
// 4-entry boundaries, zero-padded, one select per 4-entry chunk (as spmv16p_kernel); gathers
// from global memory (L1).
template <int LPR, int UNR>
__global__ void __launch_bounds__(512, 2) spmv32p_kernel(SpmvArgs a) {
  const int lane = threadIdx.x & (LPR - 1);
  const int grp = threadIdx.x / LPR;
  const int ngrp = blockDim.x / LPR;
  const int64_t it0 = (a.nitems * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t it1 = (a.nitems * (int64_t)(blockIdx.x + 1)) / gridDim.x;
  double sq = 0.0;
  // the CTA's whole item range is one row range (no slice windows in the global-gather kernel)
  const int64_t r0 = it0 < it1 ? a.item_row[it0] : 0, r1 = it0 < it1 ? a.item_row[it1] : 0;
  int64_t row = r0 + grp;
  int64_t s_n = 0, e_n = 0;
  if (row < r1) {
    s_n = a.rp[row];
    e_n = a.rp[row + 1];
  }
  for (int64_t base = r0; base < r1; base += ngrp) {
    const bool valid = row < r1;
    const int64_t s = s_n;
    const int span = (int)(e_n - s_n);  // padded: a multiple of 4
    const int64_t nrow = row + ngrp;
    if (nrow < r1) {
      s_n = a.rp[nrow];
      e_n = a.rp[nrow + 1];
    }
    const int nch = valid ? (span + 4 * LPR - 1) / (4 * LPR) : 0;
    const int lim = span - 4 * lane;
    const int32_t* cp = a.col + s + 4 * lane;
    const float* vp = a.val + s + 4 * lane;
    double acc[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc[u] = 0.0;
    int ch = 0;
    auto chunk = [&](const int4 c, const float4 v) {
      const double p0 = (double)v.x * (double)__ldg(a.src + c.x);
      const double p1 = (double)v.y * (double)__ldg(a.src + c.y);
      const double p2 = (double)v.z * (double)__ldg(a.src + c.z);
      const double p3 = (double)v.w * (double)__ldg(a.src + c.w);
      return (p0 + p1) + (p2 + p3);
    };
    for (; ch + UNR <= nch; ch += UNR) {
      int4 c[UNR];
      float4 v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        c[u] = ld_stream_i4(cp + (ch + u) * 4 * LPR);
        v[u] = ld_stream_f4(vp + (ch + u) * 4 * LPR);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const double t = chunk(c[u], v[u]);
        acc[u] += ((ch + u) * 4 * LPR < lim) ? t : 0.0;
      }
    }
    for (; ch < nch; ++ch) {
      const double t = chunk(ld_stream_i4(cp + ch * 4 * LPR), ld_stream_f4(vp + ch * 4 * LPR));
      acc[0] += (ch * 4 * LPR < lim) ? t : 0.0;
    }
#pragma unroll
    for (int u = 1; u < UNR; ++u) acc[0] += acc[u];
    const double accr = group_sum<LPR>(acc[0]);
    if (valid && lane == 0) {
      if (a.b) {
        const double r = accr - (double)__ldg(a.b + row);
        const float rh = (float)r;
        a.out[row] = rh;
        if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);
        sq += r * r;
      } else if (a.out_peer) {
        // fused reduce-scatter: store straight into the owner's inbox (NVLink peer memory)
        int o = 0;
        while (o + 1 < a.n_out && row >= a.out_bounds[o + 1]) ++o;
        a.out_peer[o][row] = (float)accr;
      } else {
        a.out[row] = (float)accr;
      }
    }
    row = nrow;
  }
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// Owner side of the fused reduce-scatter: out[i] = sum over ranks r (in rank order) of
// inbox[r stride + i].
__global__ void inbox_sum_kernel(int64_t n, const float* __restrict__ inbox, int64_t stride, int world,
                                 float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = inbox[i];
    for (int r = 1; r < world; ++r) acc += inbox[(int64_t)r * stride + i];
    out[i] = acc;
  }
}

cudaError_t launch_inbox_sum(int64_t n, const float* inbox, int64_t stride, int world, float* out,
                             cudaStream_t st) {
  inbox_sum_kernel<<<592, 256, 0, st>>>(n, inbox, stride, world, out);
  return cudaGetLastError();
}

__global__ void pad_rows32_kernel(int64_t m, const int64_t* rp, const int64_t* rpp, const int32_t* col,
                                  const float* val, int32_t* colp, float* valp) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    const int64_t s = rp[r], len = rp[r + 1] - s, d = rpp[r], plen = rpp[r + 1] - d;
    for (int64_t k = lane; k < plen; k += 32) {
      colp[d + k] = k < len ? col[s + k] : 0;
      valp[d + k] = k < len ? val[s + k] : 0.0f;
    }
  }
}

cudaError_t launch_pad_rows32(int64_t m, const int64_t* rp, const int64_t* rpp, const int32_t* col,
                              const float* val, int32_t* colp, float* valp, cudaStream_t st) {
  pad_rows32_kernel<<<1184, 256, 0, st>>>(m, rp, rpp, col, val, colp, valp);
  return cudaGetLastError();
}

template <class F>
static cudaError_t dispatch32p(const SpmvVariant& v, F&& f) {
  if (v.lpr == 4) return f(spmv32p_kernel<4, 2>);
  if (v.lpr == 8) return f(spmv32p_kernel<8, 2>);
  if (v.lpr == 16) return f(spmv32p_kernel<16, 2>);
  if (v.lpr == 32) return f(spmv32p_kernel<32, 2>);
  return cudaErrorInvalidValue;
}

cudaError_t launch_spmv32p(const SpmvArgs& a, const SpmvVariant& v, int grid, int block,
                           cudaStream_t st) {
  return dispatch32p(v, [&](auto k) -> cudaError_t {
    cudaError_t e = ensure_smem_attr((const void*)k, 0);
    if (e != cudaSuccess) return e;
    k<<<grid, block, 0, st>>>(a);
    return cudaGetLastError();
  });
}

int spmv32p_occupancy(const SpmvVariant& v, int block) {
  int occ = 0;
  dispatch32p(v, [&](auto k) -> cudaError_t {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, block, 0);
  });
  return occ > 0 ? occ : 1;
}

// Window parts (opt-in, TVR_PART_CAP): a slice window larger than the shared-memory budget is
// cut into `parts` pieces of part_len entries.  Columns ascend within a row, so each row's
// entries are contiguous per part; part_off[(p-1) nrows + row] is the row-relative start of
// part p.  The CTA stages part p and runs all rows of its slice segment on it, carrying the fp64
// partial sum of each row in part_acc (same thread every part, so no synchronisation needed);
// the last part finalises the row.  Measured slower than global gathers for c3's x-slice
// (every part re-walks each row with half-empty chunks), so not the default.
template <int LPR, int UNR, int MINB, bool STAGED>
__global__ void __launch_bounds__(512, MINB) spmv16_parts_kernel(SpmvArgs a) {
  extern __shared__ float stage[];
  const int lane = threadIdx.x & (LPR - 1);
  const int grp = threadIdx.x / LPR;
  const int ngrp = blockDim.x / LPR;
  const int64_t it0 = (a.nitems * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t it1 = (a.nitems * (int64_t)(blockIdx.x + 1)) / gridDim.x;
  const int P = a.parts;
  double sq = 0.0;
  for (int64_t sa = it0; sa < it1;) {
    const int z = a.item_slice[sa];
    const int64_t zend = a.slice_item_end[z];
    const int64_t sb = zend < it1 ? zend : it1;  // slice segment [sa, sb) of this CTA
    const int64_t wlo = a.win_lo[z];
    const int wlen = a.win_len[z];
  for (int p = 0; p < P; ++p) {
    const int plo = p * a.part_len;
    const float* gbase = a.src + wlo + plo;
    if constexpr (STAGED) {
      const int plen = min(a.part_len, wlen - plo);
      __syncthreads();
      stage_window(stage, gbase, plen);
      __syncthreads();
    }
  for (int64_t it = sa; it < sb; ++it) {
    const int64_t r0 = a.item_row[it], r1 = a.item_row[it + 1];
    // entry range of `row` inside part p
    auto extent = [&](int64_t rr, int64_t& s_, int64_t& e_) {
      const int64_t rs = a.rp[rr];
      s_ = rs + (p > 0 ? (int64_t)a.part_off[(int64_t)(p - 1) * a.nrows + rr] : 0);
      e_ = (p == P - 1) ? a.rp[rr + 1] : rs + (int64_t)a.part_off[(int64_t)p * a.nrows + rr];
    };
    int64_t row = r0 + grp;
    int64_t s_n = 0, e_n = 0;
    if (row < r1) extent(row, s_n, e_n);
    for (int64_t base = r0; base < r1; base += ngrp) {
      const bool valid = row < r1;
      const int64_t s = s_n, e = e_n;
      const int64_t nrow = row + ngrp;
      if (nrow < r1) extent(nrow, s_n, e_n);  // prefetch the next row's extent
      const int64_t kb = s & ~int64_t(7);
      const int span = (int)(e - kb);
      int lo = (int)(s - kb) - 8 * lane;
      int hi = span - 8 * lane;
      const int nch = valid ? (span + 8 * LPR - 1) / (8 * LPR) : 0;
      const uint16_t* cp = a.col16 + kb + 8 * lane;
      const float* vp = a.val + kb + 8 * lane;
      double acc[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc[u] = 0.0;
      int ch = 0;
      for (; ch + UNR <= nch; ch += UNR) {
        int4 c[UNR];
        float4 va[UNR], vb[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + (ch + u) * 8 * LPR));
          va[u] = ld_stream_f4(vp + (ch + u) * 8 * LPR);
          vb[u] = ld_stream_f4(vp + (ch + u) * 8 * LPR + 4);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          acc[u] = chunk8_dot<STAGED>(c[u], va[u], vb[u], lo - 8 * LPR * u, hi - 8 * LPR * u, stage,
                                      gbase, acc[u]);
        lo -= 8 * LPR * UNR;
        hi -= 8 * LPR * UNR;
      }
      for (; ch < nch; ++ch) {
        const int4 c0 = ld_stream_i4(reinterpret_cast<const int32_t*>(cp + ch * 8 * LPR));
        const float4 va0 = ld_stream_f4(vp + ch * 8 * LPR);
        const float4 vb0 = ld_stream_f4(vp + ch * 8 * LPR + 4);
        acc[0] = chunk8_dot<STAGED>(c0, va0, vb0, lo, hi, stage, gbase, acc[0]);
        lo -= 8 * LPR;
        hi -= 8 * LPR;
      }
#pragma unroll
      for (int u = 1; u < UNR; ++u) acc[0] += acc[u];
      double accr = group_sum<LPR>(acc[0]);
      if (valid && lane == 0) {
        if (p > 0) accr += a.part_acc[row];
        if (p < P - 1) {
          a.part_acc[row] = accr;
        } else if (a.b) {
          const double r = accr - (double)a.b[row];
          const float rh = (float)r;
          a.out[row] = rh;
          if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);
          sq += r * r;
        } else {
          a.out[row] = (float)accr;
        }
      }
      row = nrow;
    }
  }  // items
  }  // parts
    sa = sb;
  }  // slice segments
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

// Per row of a staged plan with window parts: part_off (row-relative start of parts 1..P-1) and
// col16[k] = (col[k] - win_lo) - part * part_len.  With expand, the inverse (canonical int32
// columns from col16 and part_off).
__global__ void parts_rows_kernel(int64_t nitems, const int64_t* __restrict__ item_row,
                                  const int32_t* __restrict__ item_slice,
                                  const int64_t* __restrict__ win_lo, const int64_t* __restrict__ rp,
                                  int parts, int part_len, int64_t nrows, bool expand,
                                  const int32_t* __restrict__ col, uint16_t* __restrict__ col16,
                                  uint16_t* __restrict__ part_off, int32_t* __restrict__ col_out) {
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int64_t base = win_lo[item_slice[it]];
    for (int64_t row = item_row[it] + threadIdx.x; row < item_row[it + 1]; row += blockDim.x) {
      const int64_t s = rp[row], e = rp[row + 1];
      int q = 1;  // next boundary to record
      for (int64_t k = s; k < e; ++k) {
        int pk;
        if (!expand) {
          const int64_t off = (int64_t)col[k] - base;
          pk = (int)(off / part_len);
          while (q <= pk && q < parts) part_off[(int64_t)(q - 1) * nrows + row] = (uint16_t)(k - s), ++q;
          col16[k] = (uint16_t)(off - (int64_t)pk * part_len);
        } else {
          pk = 0;
          while (pk + 1 < parts && (k - s) >= (int64_t)part_off[(int64_t)pk * nrows + row]) ++pk;
          col_out[k] = (int32_t)(base + (int64_t)pk * part_len + col16[k]);
        }
      }
      if (!expand)
        for (; q < parts; ++q) part_off[(int64_t)(q - 1) * nrows + row] = (uint16_t)(e - s);
    }
  }
}

cudaError_t launch_parts_rows(const SpmvArgs& a, bool expand, const int32_t* col, uint16_t* col16,
                              uint16_t* part_off, int32_t* col_out, cudaStream_t st) {
  const int grid = a.nitems < 148 * 16 ? (int)a.nitems : 148 * 16;
  if (grid <= 0) return cudaSuccess;
  parts_rows_kernel<<<grid, 128, 0, st>>>(a.nitems, a.item_row, a.item_slice, a.win_lo, a.rp, a.parts,
                                          a.part_len, a.nrows, expand, col, col16, part_off, col_out);
  return cudaGetLastError();
}

// col16[k] = col[k] - win_lo[slice of k's row]: the 16-bit window offsets of a staged plan.
__global__ void compress_cols_kernel(int64_t nitems, const int64_t* __restrict__ item_row,
                                     const int32_t* __restrict__ item_slice,
                                     const int64_t* __restrict__ win_lo,
                                     const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                     uint16_t* __restrict__ col16) {
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int64_t base = win_lo[item_slice[it]];
    const int64_t k0 = rp[item_row[it]], k1 = rp[item_row[it + 1]];
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) col16[k] = (uint16_t)(col[k] - base);
  }
}

// Inverse: the canonical int32 columns (for tvr_get_AT / inspection).
__global__ void expand_cols_kernel(int64_t nitems, const int64_t* __restrict__ item_row,
                                   const int32_t* __restrict__ item_slice,
                                   const int64_t* __restrict__ win_lo, const int64_t* __restrict__ rp,
                                   const uint16_t* __restrict__ col16, int32_t* __restrict__ col) {
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int64_t base = win_lo[item_slice[it]];
    const int64_t k0 = rp[item_row[it]], k1 = rp[item_row[it + 1]];
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) col[k] = (int32_t)(base + col16[k]);
  }
}

cudaError_t launch_compress_cols(const SpmvArgs& a, const int32_t* col, uint16_t* col16, bool expand,
                                 int32_t* col_out, cudaStream_t st) {
  const int grid = a.nitems < 148 * 16 ? (int)a.nitems : 148 * 16;
  if (grid <= 0) return cudaSuccess;
  if (expand)
    expand_cols_kernel<<<grid, 256, 0, st>>>(a.nitems, a.item_row, a.item_slice, a.win_lo, a.rp, col16,
                                             col_out);
  else
    compress_cols_kernel<<<grid, 256, 0, st>>>(a.nitems, a.item_row, a.item_slice, a.win_lo, a.rp, col,
                                               col16);
  return cudaGetLastError();
}

// a6: s = sum_i ((1+beta) r1_i - beta r0_i)^2 in fp64 (no vector written: only f(y) needs it).
// Residuals are carried as fp32 hi + lo pairs so that f(y) by linearity keeps fp64 accuracy
// (BT compares f values that differ by ~1e-14 relative near convergence).
__global__ void momentum_resid_kernel(int64_t m, const float* __restrict__ r1,
                                      const float* __restrict__ r1lo, const float* __restrict__ r0,
                                      const float* __restrict__ r0lo, double beta, double* partials,
                                      unsigned* counter, double* scal, const double* dbeta) {
  if (dbeta) beta = *dbeta;  // device-side control
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
    const double a1 = (double)r1[i] + (double)r1lo[i];
    const double a0 = (double)r0[i] + (double)r0lo[i];
    const double ry = (1.0 + beta) * a1 - beta * a0;
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
// Raise a kernel's dynamic shared-memory limit once per (function, device, size) instead of a
// driver call on every launch (host overhead of the synchronous per-call API).
cudaError_t ensure_smem_attr(const void* func, size_t smem) {
  if (smem == 0) {
    // global-gather kernels live on L1 hits: ask for the whole L1/shared array as L1 (c3 A pass
    // -1.6 %; the opposite carveout makes it 3.7x slower, measured)
    static std::mutex mu0;
    static std::map<const void*, bool> set0;
    std::lock_guard<std::mutex> lk(mu0);
    if (!set0[func]) {
      cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      set0[func] = true;
    }
    return cudaSuccess;
  }
  if (smem <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{func, dev}];
  if (have >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) have = smem;
  return e;
}

template <int LPR, bool STAGED, int UNR, int MINB>
static cudaError_t launch_spmv_t(const SpmvArgs& a, int grid, int block, size_t smem,
                                 cudaStream_t st) {
  auto k = spmv_kernel<LPR, STAGED, UNR, MINB>;
  cudaError_t e = ensure_smem_attr((const void*)k, smem);
  if (e != cudaSuccess) return e;
  k<<<grid, block, smem, st>>>(a);
  return cudaGetLastError();
}

template <int LPR, bool STAGED, int UNR, int MINB>
static int occupancy_t(int block, size_t smem) {
  auto k = spmv_kernel<LPR, STAGED, UNR, MINB>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, block, smem) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return n > 0 ? n : 1;
}

// Dispatch over the instantiated variants: lanes per row {4, 8, 16, 32}, staged or global
// gather, UNR chunks in flight {2 with min resident CTAs 1-3, 4 with 1}.
template <class F>
static auto dispatch(const SpmvVariant& v, F&& f) {
#define TVR_V(L, S, U, M)                                          \
  if (v.lpr == L && v.staged == S && v.unroll == U && v.minb == M) \
    return f(std::integral_constant<int, L>{}, std::integral_constant<bool, S>{}, \
             std::integral_constant<int, U>{}, std::integral_constant<int, M>{});
#define TVR_VL(L) TVR_V(L, true, 2, 1) TVR_V(L, false, 2, 1) TVR_V(L, true, 2, 2) TVR_V(L, false, 2, 2) \
  TVR_V(L, true, 2, 3) TVR_V(L, false, 2, 3) TVR_V(L, true, 4, 1) TVR_V(L, false, 4, 1)
  TVR_VL(4)
  TVR_VL(8)
  TVR_VL(16)
  TVR_VL(32)
#undef TVR_VL
#undef TVR_V
  return f(std::integral_constant<int, 8>{}, std::integral_constant<bool, false>{},
           std::integral_constant<int, 2>{}, std::integral_constant<int, 1>{});
}

// 16-bit variants: UNR 2, lanes per row {4, 8, 16}, min resident CTAs {1, 2, 3}, window staged
// in shared memory or gathered from global memory.
template <class F>
static auto dispatch16(const SpmvVariant& v, F&& f) {
#define TVR_V16(L, M)                                                                 \
  if (v.lpr == L && v.minb == M && v.unroll == 2)                                     \
    return v.parts ? f(spmv16_parts_kernel<L, 2, M, true>)                            \
                   : (v.staged ? f(spmv16_kernel<L, 2, M, true>) : f(spmv16_kernel<L, 2, M, false>));
  TVR_V16(4, 1) TVR_V16(4, 2) TVR_V16(4, 3)
  TVR_V16(8, 1) TVR_V16(8, 2) TVR_V16(8, 3)
  TVR_V16(16, 1) TVR_V16(16, 2) TVR_V16(16, 3)
#undef TVR_V16
  // deeper unrolling (staged, 2 CTAs/SM) for tuning sweeps
#define TVR_V16U(L, U) \
  if (v.lpr == L && v.minb == 2 && v.unroll == U && v.staged && !v.parts) return f(spmv16_kernel<L, U, 2, true>);
  TVR_V16U(4, 3) TVR_V16U(4, 4) TVR_V16U(8, 3) TVR_V16U(8, 4)
#undef TVR_V16U
  return f(spmv16_kernel<8, 2, 1, true>);
}

bool spmv_variant_exists(const SpmvVariant& v) {
  if (v.idx16) {
    if (v.unroll == 3 || v.unroll == 4)
      return (v.lpr == 4 || v.lpr == 8) && v.minb == 2 && v.staged && !v.parts;
    return v.unroll == 2 && (v.lpr == 4 || v.lpr == 8 || v.lpr == 16) && v.minb >= 1 && v.minb <= 3;
  }
  if (!(v.lpr == 4 || v.lpr == 8 || v.lpr == 16 || v.lpr == 32)) return false;
  if (v.unroll == 2) return v.minb >= 1 && v.minb <= 3;
  return v.unroll == 4 && v.minb == 1;
}

cudaError_t launch_spmv(const SpmvArgs& a, const SpmvVariant& v, int grid, int block, size_t smem,
                        cudaStream_t st) {
  if (!spmv_variant_exists(v)) return cudaErrorInvalidValue;
  if (v.idx16) {
    return dispatch16(v, [&](auto k) {
      cudaError_t e = ensure_smem_attr((const void*)k, smem);
      if (e != cudaSuccess) return e;
      k<<<grid, block, smem, st>>>(a);
      return cudaGetLastError();
    });
  }
  return dispatch(v, [&](auto L, auto S, auto U, auto M) {
    return launch_spmv_t<decltype(L)::value, decltype(S)::value, decltype(U)::value,
                         decltype(M)::value>(a, grid, block, S ? smem : 0, st);
  });
}

int spmv_occupancy(const SpmvVariant& v, int block, size_t smem) {
  if (!spmv_variant_exists(v)) return 1;
  if (v.idx16) {
    return dispatch16(v, [&](auto k) {
      if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int n = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, block, smem) != cudaSuccess) {
        cudaGetLastError();
        return 1;
      }
      return n > 0 ? n : 1;
    });
  }
  return dispatch(v, [&](auto L, auto S, auto U, auto M) {
    return occupancy_t<decltype(L)::value, decltype(S)::value, decltype(U)::value,
                       decltype(M)::value>(block, S ? smem : 0);
  });
}

cudaError_t launch_momentum_resid(int64_t m, const float* r1, const float* r1lo, const float* r0,
                                  const float* r0lo, double beta, double* partials,
                                  unsigned* counter, double* scal, int grid, cudaStream_t st,
                                  const double* dbeta) {
  momentum_resid_kernel<<<grid, 256, 0, st>>>(m, r1, r1lo, r0, r0lo, beta, partials, counter, scal,
                                              dbeta);
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
