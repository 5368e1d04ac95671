// Ceilings for the staged 16-bit SpMV (c2 A pass shape): how fast can a kernel stream the
// entry arrays (16-bit column + fp32 value = 6 B per entry) with and without the shared-memory
// gather, ignoring row structure?  Standalone: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// scripts/spmv_bounds.cu -o /tmp/spmv_bounds && /tmp/spmv_bounds
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ int4 ldi4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldf4(const void* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// MODE 0: stream only (sum of values); MODE 1: + gather x from a staged shared window
template <int MODE, int UNR>
__global__ void __launch_bounds__(512, 2) stream_kernel(const uint16_t* col, const float* val, int64_t nchunks,
                                                        const float* x, int wlen, double* out) {
  extern __shared__ float win[];
  if (MODE == 1) {
    for (int i = threadIdx.x; i < wlen; i += blockDim.x) win[i + (i >> 5)] = x[i];
    __syncthreads();
  }
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  int64_t c = tid;
  for (; c + (UNR - 1) * nth < nchunks; c += UNR * nth) {
    int4 ci[UNR];
    float4 va[UNR], vb[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      ci[u] = ldi4(col + (c + u * nth) * 8);
      va[u] = ldf4(val + (c + u * nth) * 8);
      vb[u] = ldf4(val + (c + u * nth) * 8 + 4);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint32_t cw[4] = {(uint32_t)ci[u].x, (uint32_t)ci[u].y, (uint32_t)ci[u].z, (uint32_t)ci[u].w};
      const float vv[8] = {va[u].x, va[u].y, va[u].z, va[u].w, vb[u].x, vb[u].y, vb[u].z, vb[u].w};
      double p[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float xv = 1.0f;
        if (MODE == 1) {
          const int ci16 = (cw[q >> 1] >> (16 * (q & 1))) & 0xffff;
          xv = win[ci16 + (ci16 >> 5)];
        } else {
          xv = __int_as_float(cw[q >> 1] | 0x3f800000);
        }
        p[q] = (double)vv[q] * (double)xv;
      }
      acc += ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int64_t nnz = 160079872, nch = nnz / 8;
  const int wlen = 16384;
  uint16_t* col; float* val; float* x; double* out;
  CK(cudaMalloc(&col, nnz * 2)); CK(cudaMalloc(&val, nnz * 4)); CK(cudaMalloc(&x, wlen * 4)); CK(cudaMalloc(&out, 8));
  // pseudo-random columns with ray-like locality: runs of +1 / +128 steps
  uint16_t* hc = (uint16_t*)malloc(nnz * 2);
  uint32_t s = 12345, c = 0;
  for (int64_t i = 0; i < nnz; ++i) {
    s = s * 1664525u + 1013904223u;
    if ((i % 115) == 0) c = s % wlen;
    c = (c + (((s >> 16) & 1) ? 1 : 128)) % wlen;
    hc[i] = (uint16_t)c;
  }
  CK(cudaMemcpy(col, hc, nnz * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(val, 0, nnz * 4)); CK(cudaMemset(x, 0, wlen * 4));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (wlen + wlen / 32 + 1) * 4;
  CK(cudaFuncSetAttribute(stream_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(stream_kernel<1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(stream_kernel<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, size_t sm) {
    for (int w = 0; w < 3; ++w) kern<<<nsm * 2, 512, sm>>>(col, val, nch, x, wlen, out);
    cudaEventRecord(a);
    const int R = 20;
    for (int r = 0; r < R; ++r) kern<<<nsm * 2, 512, sm>>>(col, val, nch, x, wlen, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= R;
    printf("%-28s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, nnz * 6.0 / (ms * 1e-3) / 1e9);
  };
  run("stream only, unr 2", stream_kernel<0, 2>, 0);
  run("stream only, unr 3", stream_kernel<0, 3>, 0);
  run("stream + smem gather, unr 2", stream_kernel<1, 2>, smem);
  run("stream + smem gather, unr 3", stream_kernel<1, 3>, smem);
  run("stream + smem gather, unr 4", stream_kernel<1, 4>, smem);
  CK(cudaGetLastError());
  return 0;
}
