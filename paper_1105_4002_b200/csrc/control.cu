// Device-side GPBB control; see control.h.  Each kernel is one thread and
// mirrors a block of gpbb_impl (solvers.cu) operation for operation, so the device and host
// controllers take the same decisions on the same reductions.  Products and sums are written
// with the _rn intrinsics so nvcc does not contract them into FMAs the host code does not use.
#include <cmath>

#include "control.h"
#include "solver_slots.h"

namespace tvr {

__device__ __forceinline__ bool dev_stop_test(double gn, double gref, double N, double eps, int mode) {
  if (mode == TVR_STOP_ABS_PER_N) return gn / N <= eps;
  return gn <= __dmul_rn(eps, gref);
}

// history record of iteration k, written when its line search ends (as gpbb_impl)
__device__ void gpbb_record(GpbbDev* d) {
  if (d->n_rec < d->rec_cap) {
    tvr_record r{};
    r.iter = d->k;
    r.f = d->f;
    r.gmap_rel = d->gref > 0 ? d->gn / d->gref : 0.0;
    r.gmap_abs_per_n = d->gn / d->N;
    r.step_or_inv_L = d->theta;
    r.ls_trials = d->trials;
    d->rec[d->n_rec] = r;
  }
  ++d->n_rec;
  d->n_ls += d->trials;
}

// Top of iteration k: BB step (C6: keep theta_{k-1} on a non-positive or non-finite
// denominator), beta = beta_0, f_hat = max of the last K+1 accepted values (C21).
__global__ void gpbb_begin_kernel(GpbbDev* d, GpbbHandles h) {
  if (d->k > 0 && d->bb_dg > 0.0 && isfinite(d->bb_dg) && isfinite(d->bb_dd))
    d->theta = d->bb_dd / d->bb_dg;
  d->beta = d->beta0;
  double fhat = -INFINITY;
  const int64_t first = d->nh > d->K + 1 ? d->nh - d->K - 1 : 0;
  for (int64_t i = first; i < d->nh; ++i) fhat = fmax(fhat, d->fhist[i % 64]);
  d->fhat = fhat;
  d->trials = 0;
  d->dparam[0] = __dmul_rn(d->beta, d->theta);
  d->dparam[1] = d->theta;  // stop-test reduction at nu = 1/theta_k on the first trial (C11)
  d->dparam[2] = 0.0;
  cudaGraphSetConditional(h.ls, 1);
  cudaGraphSetConditional(h.acc, 0);
}

// After a trial's stencil and A passes.
__global__ void gpbb_ls_kernel(GpbbDev* d, const double* sc, GpbbHandles h) {
  ++d->ls_execs;
  auto finish = [&](bool accept, bool stop) {
    gpbb_record(d);
    cudaGraphSetConditional(h.ls, 0);
    cudaGraphSetConditional(h.acc, accept ? 1 : 0);
    if (stop) cudaGraphSetConditional(h.outer, 0);
  };
  if (d->trials == 0) {
    d->gn = sqrt(sc[S_TV + 3]) / d->theta;
    d->conv = dev_stop_test(d->gn, d->gref, d->N, d->eps, d->stop_mode) ? 1 : 0;
    if (d->conv || d->k >= d->max_iters) { finish(false, true); return; }
  }
  d->f_bar = __dadd_rn(__dmul_rn(0.5, sc[S_RSQ]), __dmul_rn(d->alpha, sc[S_TV]));
  const double gdx = sc[S_TV + 1];  // g_k^T (x_k - x_bar)
  ++d->trials;
  ++d->n_f;
  if (!isfinite(d->f_bar)) { d->status = TVR_E_NONFINITE; finish(false, true); return; }
  if (!(d->f_bar >= __dsub_rn(d->fhat, __dmul_rn(d->sigma, gdx)))) { finish(true, false); return; }
  d->beta = __dmul_rn(d->beta, d->beta);
  if (d->beta < d->beta_min) { d->status = TVR_E_LINESEARCH; finish(false, true); return; }
  d->dparam[0] = __dmul_rn(d->beta, d->theta);
  d->dparam[1] = 0.0;
  cudaGraphSetConditional(h.ls, 1);
}

// After x_{k+1} = x_bar and its gradient pass: BB reductions, f, history of f.
__global__ void gpbb_accept_kernel(GpbbDev* d, const double* sc) {
  d->bb_dd = sc[S_TV + 1];
  d->bb_dg = sc[S_TV + 2];
  ++d->n_g;
  d->f = d->f_bar;
  d->fhist[d->nh % 64] = d->f;
  ++d->nh;
  ++d->k;
}

cudaError_t launch_gpbb_begin(GpbbDev* d, GpbbHandles h, cudaStream_t st) {
  gpbb_begin_kernel<<<1, 1, 0, st>>>(d, h);
  return cudaGetLastError();
}
cudaError_t launch_gpbb_ls(GpbbDev* d, const double* scal, GpbbHandles h, cudaStream_t st) {
  gpbb_ls_kernel<<<1, 1, 0, st>>>(d, scal, h);
  return cudaGetLastError();
}
cudaError_t launch_gpbb_accept(GpbbDev* d, const double* scal, cudaStream_t st) {
  gpbb_accept_kernel<<<1, 1, 0, st>>>(d, scal);
  return cudaGetLastError();
}

}  // namespace tvr
