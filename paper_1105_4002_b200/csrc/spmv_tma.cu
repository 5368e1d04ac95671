// TMA bulk-copy pipelined CSR SpMV for slice-separable matrices.
//
// The register-streaming kernel of spmv.cu tops out near 77% of HBM bandwidth because each
// group only has its own row's chunks in flight.  Here the streaming is decoupled from the
// arithmetic: one producer thread per CTA issues `cp.async.bulk` (TMA engine, SASS UBLKCP)
// copies of whole row tiles — col, val, the tile's row pointers and (A pass) b — into a ring of
// shared-memory stages guarded by mbarriers (full: transaction bytes; empty: one arrive per
// consumer warp).  Consumer warps own whole tiles round-robin (tile i -> warp i mod NC, stage
// i mod S), process them with LPR-lane groups per row reading 16-byte chunks from shared memory,
// gather x / r from the slice window staged in shared memory, accumulate in fp64 and reduce with
// a fixed butterfly, exactly as the register kernel (same per-row summation order, so results
// are bitwise identical).  Tiles never straddle a z-slice; on a slice change the consumer warps
// meet at a named barrier, restage the window and meet again.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace tvr {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ int swz(int c) { return c + (c >> 5); }

// Same masked 4-entry product as spmv.cu's staged chunk_dot (identical fma order).
__device__ __forceinline__ double tma_chunk_dot(const int4 c, const float4 v, int lo, int hi,
                                                const float* __restrict__ win, int wl, double acc) {
  const int cc[4] = {c.x, c.y, c.z, c.w};
  const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool in = (q >= lo) & (q < hi);
    const float val = in ? vv[q] : 0.0f;
    const float xv = win[swz(in ? cc[q] - wl : 0)];
    acc = fma((double)val, (double)xv, acc);
  }
  return acc;
}

// Carve the dynamic shared memory: window, then per stage col/val/rp/b, then the barriers.
struct Layout {
  float* win;
  int32_t* col;
  float* val;
  int64_t* rp;
  float* b;
  uint64_t* full;
  uint64_t* empty;
  int64_t* hdr;  // per stage: r0, r1, k0 of the tile it holds
  int* ticket;   // two per-segment tile counters of the consumer warps
};
__device__ __forceinline__ Layout carve(char* base, const TmaSpmvArgs& a) {
  Layout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base + off;
    off += (bytes + 127) & ~size_t(127);
    return p;
  };
  L.win = (float*)take(sizeof(float) * (size_t)a.win_cap);
  L.col = (int32_t*)take(sizeof(int32_t) * (size_t)a.tile_nnz * a.stages);
  L.val = (float*)take(sizeof(float) * (size_t)a.tile_nnz * a.stages);
  L.rp = (int64_t*)take(sizeof(int64_t) * (size_t)(a.tile_rows + 4) * a.stages);
  L.b = (float*)take(sizeof(float) * (size_t)(a.tile_rows + 8) * a.stages);
  L.full = (uint64_t*)take(sizeof(uint64_t) * a.stages);
  L.empty = (uint64_t*)take(sizeof(uint64_t) * a.stages);
  L.hdr = (int64_t*)take(sizeof(int64_t) * 4 * a.stages);
  L.ticket = (int*)take(sizeof(int) * 2);
  return L;
}

}  // namespace

size_t tma_spmv_smem_bytes(int win_cap, int tile_nnz, int tile_rows, int stages) {
  auto r = [](size_t b) { return (b + 127) & ~size_t(127); };
  return r(4ull * win_cap) + 2 * r(4ull * tile_nnz * stages) + r(8ull * (tile_rows + 4) * stages) +
         r(4ull * (tile_rows + 8) * stages) + 2 * r(8ull * stages) + r(32ull * stages) + r(8);
}

template <int LPR>
__global__ void __launch_bounds__((kTmaConsumerWarps + kTmaProducerWarps) * 32, 1)
    spmv_tma_kernel(TmaSpmvArgs a) {
  extern __shared__ __align__(128) char smem_raw[];
  const Layout L = carve(smem_raw, a);
  const int warp = threadIdx.x >> 5, lane32 = threadIdx.x & 31;
  const int S = a.stages;
  const int64_t t0 = (a.ntiles * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t t1 = (a.ntiles * (int64_t)(blockIdx.x + 1)) / gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&L.full[s], 1);
      mbar_init(&L.empty[s], 1);  // released by the one consumer warp that took the tile
    }
    L.ticket[0] = 0;
    L.ticket[1] = 0;
    for (int s = 0; s < S; ++s) L.hdr[4 * s + 3] = -1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double sq = 0.0;
  if (warp >= kTmaConsumerWarps) {
    // ---------------------------------------------------------------- producers
    // kTmaProducerWarps warps issue the copies of tiles i = p, p + NP, ... (a single issuing
    // thread serialised ~200 cycles per bulk copy, measured).  Each warp loads the metadata of
    // 32 of its tiles at once (one per lane) so the global round trips overlap; lane 0 then
    // issues each tile's copies and publishes (r0, r1, k0) in the stage header before arming
    // the stage's full barrier.  S is a multiple of NP, so tile i and i - S (the previous user
    // of the stage) belong to the same producer warp.
    const int pw = warp - kTmaConsumerWarps;
    for (int64_t tb = t0 + pw; tb < t1; tb += 32 * kTmaProducerWarps) {
      int64_t mk0 = 0, mk1 = 0, mr0 = 0, mr1 = 0;
      const int64_t tl = tb + (int64_t)lane32 * kTmaProducerWarps;
      if (tl < t1) {
        mk0 = a.tile_k0[tl];
        mk1 = a.tile_k1[tl];
        mr0 = a.tile_row[tl];
        mr1 = a.tile_row[tl + 1];
      }
      const int64_t rem = (t1 - tb + kTmaProducerWarps - 1) / kTmaProducerWarps;
      const int nt = rem < 32 ? (int)rem : 32;
      for (int j = 0; j < nt; ++j) {
        const int64_t k0 = __shfl_sync(0xffffffffu, mk0, j), k1 = __shfl_sync(0xffffffffu, mk1, j);
        const int64_t r0 = __shfl_sync(0xffffffffu, mr0, j), r1 = __shfl_sync(0xffffffffu, mr1, j);
        if (lane32 == 0) {
          const int64_t i = tb + (int64_t)j * kTmaProducerWarps - t0;
          const int s = (int)(i % S);
          const uint32_t ph = (uint32_t)((i / S) & 1);
          mbar_wait(&L.empty[s], ph ^ 1u);
          const int64_t ra = r0 & ~int64_t(1);
          const uint32_t rn = (uint32_t)(((r1 + 1 - ra) + 1) & ~int64_t(1));
          const int64_t ba = r0 & ~int64_t(3);
          const uint32_t bn = a.b ? (uint32_t)(((r1 - ba) + 3) & ~int64_t(3)) : 0u;
          const uint32_t nb = (uint32_t)(k1 - k0) * 4u;
          L.hdr[4 * s + 0] = r0;
          L.hdr[4 * s + 1] = r1;
          L.hdr[4 * s + 2] = k0;
          __threadfence_block();
          *((volatile int64_t*)&L.hdr[4 * s + 3]) = i;
          mbar_expect_tx(&L.full[s], 2u * nb + 8u * rn + 4u * bn);
          // col / val in pieces of a.piece bytes (several copies in flight per tile)
          for (uint32_t off = 0; off < nb; off += a.piece) {
            const uint32_t len = (nb - off) < a.piece ? (nb - off) : a.piece;
            bulk_g2s((char*)(L.col + (size_t)s * a.tile_nnz) + off, (const char*)(a.col + k0) + off, len, &L.full[s]);
            bulk_g2s((char*)(L.val + (size_t)s * a.tile_nnz) + off, (const char*)(a.val + k0) + off, len, &L.full[s]);
          }
          bulk_g2s(L.rp + (size_t)s * (a.tile_rows + 4), a.rp + ra, 8u * rn, &L.full[s]);
          if (bn) bulk_g2s(L.b + (size_t)s * (a.tile_rows + 8), a.b + ba, 4u * bn, &L.full[s]);
        }
      }
    }
  } else {
    // --------------------------------------------------------------- consumers
    const int lane = lane32 & (LPR - 1);
    const int grp = lane32 / LPR;
    constexpr int GPW = 32 / LPR;
    // slice segments of [t0, t1) from the list of tiles that start a new slice
    int64_t seg = 0;
    {
      int64_t lo = 0, hi = a.nbounds;  // last boundary <= t0
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (a.bounds[mid] <= t0) lo = mid;
        else hi = mid;
      }
      seg = lo;
    }
    int k = 0;  // segment parity: selects the ticket counter
    for (int64_t sa = t0; sa < t1; ++seg, ++k) {
      const int64_t nb_t = seg + 1 < a.nbounds ? a.bounds[seg + 1] : t1;
      const int64_t sb = nb_t < t1 ? nb_t : t1;
      const int z = a.tile_slice[sa];
      named_bar(1, kTmaConsumerWarps * 32);  // every consumer warp is done with the old window
      if (threadIdx.x == 0) L.ticket[(k + 1) & 1] = 0;  // next segment's counter (unused now)
      const int64_t lo64 = a.win_lo[z];
      const int len = a.win_len[z];
      const float* src = a.src + lo64;
      for (int q = threadIdx.x; q < len; q += kTmaConsumerWarps * 32) L.win[swz(q)] = __ldg(src + q);
      named_bar(1, kTmaConsumerWarps * 32);
      const int wl = (int)lo64;
    // Tiles are taken by whichever consumer warp is free (smem ticket), in order, so the S-deep
    // ring serves all warps.  Safe for S >= NC: a waiter can be at most one phase ahead of a
    // stage (the producer fills in order and blocks on the oldest unconsumed tile).
    for (;;) {
      int tk = 0;
      if (lane32 == 0) tk = atomicAdd(&L.ticket[k & 1], 1);
      tk = __shfl_sync(0xffffffffu, tk, 0);
      const int64_t t = sa + tk;
      if (t >= sb) break;
      const int64_t i = t - t0;
      const int s = (int)(i % S);
      // With several producers, stages fill out of global order and a taken tile can be two
      // phases ahead of its stage, which a parity wait cannot see.  The producer publishes the
      // tile id before arming the phase: once the header names this tile, the pending phase is
      // its phase and the parity wait is exact.
      while (*((volatile int64_t*)&L.hdr[4 * s + 3]) != i) __nanosleep(32);
      mbar_wait(&L.full[s], (uint32_t)((i / S) & 1));
      const int64_t r0 = L.hdr[4 * s + 0], r1 = L.hdr[4 * s + 1], k0 = L.hdr[4 * s + 2];
      const int64_t ra = r0 & ~int64_t(1), ba = r0 & ~int64_t(3);
      const int32_t* cs = L.col + (size_t)s * a.tile_nnz;
      const float* vs = L.val + (size_t)s * a.tile_nnz;
      const int64_t* rs = L.rp + (size_t)s * (a.tile_rows + 4);
      const float* bs = L.b + (size_t)s * (a.tile_rows + 8);
      for (int64_t base = r0; base < r1; base += GPW) {
        const int64_t row = base + grp;
        const bool valid = row < r1;
        int sl = 0, el = 0;
        if (valid) {
          sl = (int)(rs[row - ra] - k0);
          el = (int)(rs[row + 1 - ra] - k0);
        }
        const int kb = sl & ~3;
        int lo = sl - kb - 4 * lane, hi = el - kb - 4 * lane;
        const int nch = valid ? (el - kb + 4 * LPR - 1) / (4 * LPR) : 0;
        double acc0 = 0.0, acc1 = 0.0;
        int ch = 0;
        for (; ch + 2 <= nch; ch += 2) {
          const int4 c0 = *reinterpret_cast<const int4*>(cs + kb + 4 * lane + ch * 4 * LPR);
          const float4 v0 = *reinterpret_cast<const float4*>(vs + kb + 4 * lane + ch * 4 * LPR);
          const int4 c1 = *reinterpret_cast<const int4*>(cs + kb + 4 * lane + (ch + 1) * 4 * LPR);
          const float4 v1 = *reinterpret_cast<const float4*>(vs + kb + 4 * lane + (ch + 1) * 4 * LPR);
          acc0 = tma_chunk_dot(c0, v0, lo, hi, L.win, wl, acc0);
          acc1 = tma_chunk_dot(c1, v1, lo - 4 * LPR, hi - 4 * LPR, L.win, wl, acc1);
          lo -= 8 * LPR;
          hi -= 8 * LPR;
        }
        for (; ch < nch; ++ch) {
          const int4 c0 = *reinterpret_cast<const int4*>(cs + kb + 4 * lane + ch * 4 * LPR);
          const float4 v0 = *reinterpret_cast<const float4*>(vs + kb + 4 * lane + ch * 4 * LPR);
          acc0 = tma_chunk_dot(c0, v0, lo, hi, L.win, wl, acc0);
          lo -= 4 * LPR;
          hi -= 4 * LPR;
        }
        const double accr = group_sum<LPR>(acc0 + acc1);
        if (valid && lane == 0) {
          if (a.b) {
            const double r = accr - (double)bs[row - ba];
            const float rh = (float)r;
            a.out[row] = rh;
            if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);
            sq += r * r;
          } else {
            a.out[row] = (float)accr;
          }
        }
      }
      __syncwarp();
      if (lane32 == 0) mbar_arrive(&L.empty[s]);
    }  // tiles
      sa = sb;
    }  // segments
  }
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

cudaError_t launch_spmv_tma(const TmaSpmvArgs& a, int lpr, int grid, size_t smem, cudaStream_t st) {
  if (a.stages < kTmaConsumerWarps || a.stages % kTmaProducerWarps != 0) return cudaErrorInvalidValue;
  auto go = [&](auto kern) {
    cudaError_t e = ensure_smem_attr((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, (kTmaConsumerWarps + kTmaProducerWarps) * 32, smem, st>>>(a);
    return cudaGetLastError();
  };
  if (lpr == 4) return go(spmv_tma_kernel<4>);
  if (lpr == 8) return go(spmv_tma_kernel<8>);
  if (lpr == 16) return go(spmv_tma_kernel<16>);
  return cudaErrorInvalidValue;
}

}  // namespace tvr
