// Device-side solver control: the scalar logic of GPBB (Alg. 1) and UPN
// (Alg. 3 with BT, Alg. 2) as single-thread kernels that read the fused passes' fp64 reductions
// from device memory, decide, write the next pass parameters and set CUDA-graph conditional
// handles.  A whole solve is one graph launch: while-loops over iterations and line-search /
// BT trials run on the device, the host waits once.  The arithmetic is the host controller's,
// operation for operation, so both controllers take identical decisions (tested bitwise).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/libtvreg.h"

namespace tvr {

struct GpbbDev {
  // options and constants
  double eps, sigma, beta0, beta_min, gref, N, alpha;
  int64_t max_iters;
  int32_t K, stop_mode;
  // state
  double f, theta, beta, fhat, f_bar, gn;
  double bb_dd, bb_dg;  // ||x_k - x_{k-1}||^2, <x_k - x_{k-1}, g_k - g_{k-1}>
  double fhist[64];  // accepted objective values, ring (P:147 uses the last K+1, K < 64)
  int64_t nh;        // values pushed so far
  int64_t k, n_f, n_g, n_ls, ls_execs;
  int32_t trials, conv, status;
  double dparam[3];  // trial pass parameters: s = beta theta, stop_step, (unused)
  // history
  tvr_record* rec;
  int64_t rec_cap, n_rec;
};

struct GpbbHandles {
  cudaGraphConditionalHandle outer, ls, acc;
};

struct UpnDev {
  double eps, gref, N, alpha, rho_L;
  int64_t max_iters;
  int32_t bt_max, stop_mode;
  // state (names as upn_impl)
  double L, mu, theta, theta_n, beta, fxk, fy, gn;
  double bt_f, bt_L, mu_gd, mu_dd;
  int64_t k, n_f, n_g, n_ls, bt_execs;
  int32_t bt_trials, conv, status, first;  // first: y_k = x_k (no mu_k update, C9)
  double dp_trial[3];  // BT trial: s = 1/L~
  double dp_stop[3];   // stop-test stencil at x_{k+1}: stop_step = 1/L_k
  double dp_mom[3];    // momentum point: beta (source and w blend)
  tvr_record* rec;
  int64_t rec_cap, n_rec;
};

struct UpnHandles {
  cudaGraphConditionalHandle outer, bt, rest;
};

cudaError_t launch_upn_bt_begin(UpnDev* d, UpnHandles h, cudaStream_t st);
cudaError_t launch_upn_bt(UpnDev* d, const double* scal, UpnHandles h, cudaStream_t st);
cudaError_t launch_upn_mid(UpnDev* d, UpnHandles h, cudaStream_t st);
cudaError_t launch_upn_end(UpnDev* d, const double* scal, UpnHandles h, cudaStream_t st);

cudaError_t launch_gpbb_begin(GpbbDev* d, GpbbHandles h, cudaStream_t st);
cudaError_t launch_gpbb_ls(GpbbDev* d, const double* scal, GpbbHandles h, cudaStream_t st);
cudaError_t launch_gpbb_accept(GpbbDev* d, const double* scal, cudaStream_t st);

}  // namespace tvr
