// Row-agnostic ("flat") CSR SpMV for the A and A^T passes.
//
// Why: the per-row kernel (spmv.cu) gives each row LPR lanes; rows of 76-115 entries leave lanes
// masked, let only one or two 16-byte chunks per lane be in flight and pay a butterfly, a
// row_ptr fetch and a store per row.  A stream of the same 6 bytes per entry with the same
// shared-memory gather but no row structure runs at 6.7 TB/s on c2's A shape
// (scripts/spmv_bounds.cu) against 4.3 TB/s for the per-row kernel.
//
// How: a warp owns an item (a contiguous row range, never straddling a slice window) and walks
// its entries as tiles of 32 consecutive 8-entry chunks, one chunk per lane, UNR tiles of loads
// in flight.  Row boundaries come from a precomputed head mask (bit q of byte c: entry 8c+q is
// the first entry of a nonempty row), so no lane ever searches row_ptr:
//   * heads before a lane: warp prefix sum of popc(mask);
//   * inside a lane: entries before its first head belong to the row entering the lane (A), rows
//     that start and end inside the lane are finished on the spot, entries after its last head
//     open a row (S);
//   * across lanes: a segmented inclusive scan of (H ? S : A) with head flags carries open rows
//     lane to lane; a head lane finishes the entering row as (scan of the previous lane) + A;
//   * across tiles: the open row's partial (lane 31's scan value) is carried in a register.
// Every sum runs in a fixed order that depends only on the item partition, so results are
// deterministic run to run; products are exact in fp64 (24-bit x 24-bit significands).
// Empty rows have no entries and are written by a grid-stride loop (r = -b, or 0 for A^T).
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace tvr {

__device__ __forceinline__ int swz_f(int c) { return c + (c >> 5); }  // as spmv.cu's window

__device__ __forceinline__ uint32_t ld_stream_u8(const uint8_t* p) {
  uint16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}

// One 8-entry chunk's loads: columns (16-bit window offsets or int32 global ids) and values.
template <bool IDX16>
struct Chunk {
  int4 c0, c1;  // c1 unused for 16-bit columns
  float4 v0, v1;
  uint32_t head;
};

// Item-relative stream pointers: chunk c of the item is entries 8(c0 + c) .. 8(c0 + c) + 7.
template <bool IDX16>
struct ItemPtrs {
  const void* col;
  const float* val;
  const uint8_t* head;
};

template <bool IDX16>
__device__ __forceinline__ void load_chunk(const ItemPtrs<IDX16>& ip, int c, Chunk<IDX16>& ch) {
  if constexpr (IDX16) {
    ch.c0 = ld_stream_i4(reinterpret_cast<const int32_t*>(static_cast<const uint16_t*>(ip.col) + c * 8));
  } else {
    const int32_t* cp = static_cast<const int32_t*>(ip.col) + c * 8;
    ch.c0 = ld_stream_i4(cp);
    ch.c1 = ld_stream_i4(cp + 4);
  }
  ch.v0 = ld_stream_f4(ip.val + c * 8);
  ch.v1 = ld_stream_f4(ip.val + c * 8 + 4);
  ch.head = ld_stream_u8(ip.head + c);
}

template <bool STAGED, bool IDX16>
__device__ __forceinline__ int chunk_col(const Chunk<IDX16>& ch, int q) {
  if constexpr (IDX16) {
    const uint32_t w[4] = {(uint32_t)ch.c0.x, (uint32_t)ch.c0.y, (uint32_t)ch.c0.z, (uint32_t)ch.c0.w};
    return (int)((w[q >> 1] >> (16 * (q & 1))) & 0xffffu);
  } else {
    const int w[8] = {ch.c0.x, ch.c0.y, ch.c0.z, ch.c0.w, ch.c1.x, ch.c1.y, ch.c1.z, ch.c1.w};
    return w[q];
  }
}

template <bool STAGED, bool IDX16, int UNR>
__device__ __forceinline__ void flat_item(const FlatArgs& a, int64_t k, const float* __restrict__ sm,
                                          const float* __restrict__ gbase, int lane, double& sq) {
  const int64_t r0 = a.item_row[k], r1 = a.item_row[k + 1];
  const int64_t e0 = a.rp[r0], e1 = a.rp[r1];
  if (e1 <= e0) return;  // only empty rows: written by the empty-row loop
  const int64_t c0 = e0 >> 3;
  // item-relative 32-bit coordinates: entries [elo, ehi) of chunks [0, nch)
  const int elo = (int)(e0 - c0 * 8), ehi = (int)(e1 - c0 * 8);
  const int nch = (ehi + 7) >> 3;
  ItemPtrs<IDX16> ip;
  if constexpr (IDX16) ip.col = a.col16 + c0 * 8;
  else ip.col = a.col + c0 * 8;
  ip.val = a.val + c0 * 8;
  ip.head = a.head + c0;
  const int32_t* nzr = a.nzr + a.item_nz[k];

  auto emit = [&](int nzi, double acc) {
    const int64_t row = nzr[nzi];
    if (a.b) {
      const double r = acc - (double)__ldg(a.b + row);
      const float rh = (float)r;
      a.out[row] = rh;
      if (a.out_lo) a.out_lo[row] = (float)(r - (double)rh);  // hi + lo carries r to ~2^-48
      sq += r * r;
    } else {
      a.out[row] = (float)acc;
    }
  };

  double carry = 0.0;  // partial of the row open at the start of the tile
  int heads = 0;       // heads of the item before the tile
  const unsigned lt_mask = (1u << lane) - 1u;

  // One tile: MASKED only for the item's first and last tiles (warp-uniform choice), so interior
  // tiles carry no per-entry range tests.
  auto tile = [&](const Chunk<IDX16>& ch, int cb, auto masked_tag) {
    constexpr bool MASKED = decltype(masked_tag)::value;
    uint32_t inmask = 0xffu;
    if constexpr (MASKED) {
      const int kb = (cb + lane) * 8;
      const int lo = min(max(elo - kb, 0), 8), hi = min(max(ehi - kb, 0), 8);
      inmask = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
    }
    const uint32_t h = ch.head & inmask;
    const float vv[8] = {ch.v0.x, ch.v0.y, ch.v0.z, ch.v0.w, ch.v1.x, ch.v1.y, ch.v1.z, ch.v1.w};
    double p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const bool in = !MASKED || ((inmask >> q) & 1u);
      const int col = chunk_col<STAGED, IDX16>(ch, q);
      float xv;
      if constexpr (STAGED) xv = sm[swz_f(MASKED ? (in ? col : 0) : col)];
      else xv = (!MASKED || in) ? __ldg(gbase + col) : 0.0f;
      p[q] = (double)(MASKED ? (in ? vv[q] : 0.0f) : vv[q]) * (double)xv;
    }
    // heads before this lane: ballots of (heads in lane >= k), k = 1, 2, ... while any lane has k
    const int nh = __popc(h);
    int before = 0, tile_heads = 0;
    for (int kk = 1;; ++kk) {
      const unsigned bal = __ballot_sync(0xffffffffu, nh >= kk);
      if (!bal) break;
      before += __popc(bal & lt_mask);
      tile_heads += __popc(bal);
    }
    const int hb = heads + before;  // item-level index of this lane's first head
    double A, S = 0.0;
    if (h == 0) {
      A = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
    } else {
      // lanes holding row starts (a few per tile at c2) walk their entries in order
      double acc = 0.0;
      int hh = hb;
      A = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if ((h >> q) & 1u) {
          if (hh == hb) A = acc;   // the row entering the lane stops here
          else emit(hh - 1, acc);  // a row that started and ended inside the lane
          acc = 0.0;
          ++hh;
        }
        acc += p[q];
      }
      S = acc;
    }
    // segmented inclusive scan of open-row partials across the warp
    double v = h ? S : A;
    bool f = h != 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double vu = __shfl_up_sync(0xffffffffu, v, d);
      const bool fu = __shfl_up_sync(0xffffffffu, f, d);
      if (lane >= d) {
        if (!f) v += vu;
        f = f || fu;
      }
    }
    if (!f) v += carry;  // no head in lanes 0..lane: the row open before the tile continues
    double vin = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane == 0) vin = carry;
    if (h && hb > 0) emit(hb - 1, vin + A);  // the row entering this head lane ends here
    carry = __shfl_sync(0xffffffffu, v, 31);
    heads += tile_heads;
  };

  Chunk<IDX16> nxt[UNR];
#pragma unroll
  for (int u = 0; u < UNR; ++u) load_chunk<IDX16>(ip, min(32 * u + lane, nch - 1), nxt[u]);
  for (int cb = 0; cb < nch; cb += 32) {
    // rotate the ring of UNR tiles in flight: take the oldest, issue the load UNR tiles ahead
    const Chunk<IDX16> cur = nxt[0];
#pragma unroll
    for (int u = 0; u + 1 < UNR; ++u) nxt[u] = nxt[u + 1];
    load_chunk<IDX16>(ip, min(cb + 32 * UNR + lane, nch - 1), nxt[UNR - 1]);
    const bool interior = cb * 8 >= elo && (cb + 32) * 8 <= ehi;
    if (interior) tile(cur, cb, std::false_type{});
    else tile(cur, cb, std::true_type{});
  }
  if (lane == 0) emit(heads - 1, carry);  // the item's last row
}

template <bool STAGED, bool IDX16, int UNR>
#ifndef TVR_FLAT_BLOCK
#define TVR_FLAT_BLOCK 512
#define TVR_FLAT_MINB 2
#endif
__global__ void __launch_bounds__(TVR_FLAT_BLOCK, TVR_FLAT_MINB) spmv_flat_kernel(FlatArgs a) {
  extern __shared__ float stage[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double sq = 0.0;
  // empty rows: r = -b (A pass) or 0 (A^T pass)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_empty;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = a.empty_rows[i];
    if (a.b) {
      const double r = -(double)a.b[row];
      a.out[row] = (float)r;
      if (a.out_lo) a.out_lo[row] = 0.0f;
      sq += r * r;
    } else {
      a.out[row] = 0.0f;
    }
  }
  const int64_t it0 = (a.nitems * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t it1 = (a.nitems * (int64_t)(blockIdx.x + 1)) / gridDim.x;
  for (int64_t it = it0; it < it1;) {
    const int z = a.item_slice[it];
    const int64_t pend = min(it1, a.slice_item_end[z]);
    const float* gbase = a.src + a.win_lo[z];
    if constexpr (STAGED) {
      __syncthreads();
      const int len = a.win_len[z];
      for (int i = threadIdx.x; i < len; i += blockDim.x) stage[swz_f(i)] = __ldg(gbase + i);
      __syncthreads();
    }
    for (int64_t k = it + warp; k < pend; k += nwarps)
      flat_item<STAGED, IDX16, UNR>(a, k, stage, gbase, lane, sq);
    it = pend;
  }
  if (a.scal) {
    double v[1] = {sq};
    reduce_to_scalars<1>(v, a.partials, a.counter, a.scal);
  }
}

template <class F>
static cudaError_t with_flat(const FlatVariant& v, F&& f) {
  if (v.idx16) {
    if (v.staged) return v.unroll == 1 ? f(spmv_flat_kernel<true, true, 1>) : f(spmv_flat_kernel<true, true, 2>);
    return v.unroll == 1 ? f(spmv_flat_kernel<false, true, 1>) : f(spmv_flat_kernel<false, true, 2>);
  }
  return v.unroll == 1 ? f(spmv_flat_kernel<false, false, 1>) : f(spmv_flat_kernel<false, false, 2>);
}

cudaError_t launch_spmv_flat(const FlatArgs& a, const FlatVariant& v, int grid, int block,
                             size_t smem, cudaStream_t st) {
  return with_flat(v, [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) {
      cudaError_t e = ensure_smem_attr((const void*)kern, smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, block, smem, st>>>(a);
    return cudaGetLastError();
  });
}

int spmv_flat_occupancy(const FlatVariant& v, int block, size_t smem) {
  int occ = 0;
  with_flat(v, [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) ensure_smem_attr((const void*)kern, smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
  });
  return occ > 0 ? occ : 1;
}

}  // namespace tvr
