// Device helpers shared by the libtvreg kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

namespace tvr {

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may become resident
// while its predecessor in the stream drains (after every predecessor CTA has issued pdl_trigger
// or exited); it must call pdl_wait() before touching anything a predecessor writes -- the wait
// returns once the predecessor grid has completed and its writes are visible.  Both are no-ops
// in a launch without the attribute.  Eager launches only: under stream capture (solver and
// pipeline graphs) the attribute is left off.  TVR_PDL=0 turns it off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TVR_PDL");
    return !(e && *e == '0');
  }();
  return on;
}
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (pdl_enabled() && cudaStreamIsCapturing(st, &cs) == cudaSuccess &&
      cs == cudaStreamCaptureStatusNone) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr int kMaxScalars = 8;  // fp64 scalars one reduction launch may produce

// 128-bit streaming loads through the non-coherent path, no L1 allocation: the CSR arrays
// are read exactly once per pass (SURVEY §8(a) a1/a2 "vectorised 128-bit loads").
__device__ __forceinline__ int4 ld_stream_i4(const int32_t* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// 256-bit streaming load (sm_100: LDG.E.256): a lane's 8 consecutive fp32 values in one
// request, so the 32-byte sectors of the value stream are fetched once (two 128-bit loads at a
// 32-byte lane stride each touch every sector half-used, and without L1 allocation the sector
// comes from L2 twice).
struct f8 {
  float4 lo, hi;
};
__device__ __forceinline__ f8 ld_stream_f8(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x),
                 "=f"(r.hi.y), "=f"(r.hi.z), "=f"(r.hi.w)
               : "l"(p));
  return r;
}

// Fixed-order butterfly reduction inside a group of G lanes (G power of two <= 32):
// deterministic for a fixed launch configuration.
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}

// Block reduction of NS fp64 scalars (fixed order); result valid in thread 0.
template <int NS>
__device__ __forceinline__ void block_sum(double (&v)[NS], double* smem /* >= 32*NS */) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nthreads + 31) >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) v[s] = group_sum<32>(v[s]);
  if (lane == 0)
#pragma unroll
    for (int s = 0; s < NS; ++s) smem[warp * NS + s] = v[s];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      double t = (lane < nwarps) ? smem[lane * NS + s] : 0.0;
      v[s] = group_sum<32>(t);
    }
  }
  __syncthreads();
}

// Per-block partials + "last block finalises" in a fixed order, so the NS scalars land in
// out[0..NS) deterministically with a single launch.  partials: >= gridSize*NS doubles;
// counter: one unsigned that is 0 before the launch (the last block resets it).
template <int NS>
__device__ void reduce_to_scalars(double (&v)[NS], double* partials, unsigned* counter,
                                  double* out) {
  __shared__ double red_smem[32 * NS];
  __shared__ bool am_last;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
  block_sum<NS>(v, red_smem);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) partials[(size_t)bid * NS + s] = v[s];
    __threadfence();
    const unsigned ticket = atomicAdd(counter, 1u);
    am_last = (ticket == nblocks - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double acc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) acc[s] = 0.0;
  for (unsigned b = tid; b < nblocks; b += nthreads)
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] += __ldcg(&partials[(size_t)b * NS + s]);
  block_sum<NS>(acc, red_smem);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) out[s] = acc[s];
    *counter = 0u;
  }
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return fmin(fmax(v, lo), hi);
}

}  // namespace tvr
