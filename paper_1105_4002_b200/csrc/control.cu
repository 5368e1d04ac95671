// Device-side GPBB and UPN control; see control.h.  Each kernel is one thread and
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

// ------------------------------------------------------------------------ UPN
// Positive root of theta^2 = (1 - theta) theta_k^2 + q theta, C10: solvers.cu's
// theta_root with the host's evaluation order.
__device__ double dev_theta_root(double tk, double q) {
  const double tk2 = __dmul_rn(tk, tk);
  const double a = __dsub_rn(tk2, q);
  const double s = sqrt(__dadd_rn(__dmul_rn(a, a), __dmul_rn(__dmul_rn(4.0, tk), tk)));
  return a >= 0.0 ? __dmul_rn(2.0, tk) * tk / __dadd_rn(a, s) : __dmul_rn(0.5, __dadd_rn(-a, s));
}

// BT (Alg. 2) start: L~ = L_{k-1}
__global__ void upn_bt_begin_kernel(UpnDev* d, UpnHandles h) {
  d->bt_trials = 0;
  d->bt_L = d->L;
  d->mu_gd = d->mu_dd = 0.0;
  d->dp_trial[0] = 1.0 / d->bt_L;
  d->dp_trial[1] = 0.0;
  d->dp_trial[2] = 0.0;
  cudaGraphSetConditional(h.bt, 1);
  cudaGraphSetConditional(h.rest, 0);
}

// After a BT trial's stencil and A passes: accept on f(x) <= f(y) + g^T(x - y) + L~/2 ||x - y||^2
// (C7), else L~ <- rho L~.
__global__ void upn_bt_kernel(UpnDev* d, const double* sc, UpnHandles h) {
  ++d->bt_execs;
  const double fx = __dadd_rn(__dmul_rn(0.5, sc[S_RSQ]), __dmul_rn(d->alpha, sc[S_TV]));
  const double gd = -sc[S_TV + 1];  // g_y^T (x - y)
  const double dd = sc[S_TV + 2];   // ||x - y||^2
  if (d->bt_trials == 0) {
    d->mu_gd = sc[S_TV + 4];
    d->mu_dd = sc[S_TV + 5];
  }
  ++d->bt_trials;
  auto stop = [&](int status) {
    d->status = status;
    cudaGraphSetConditional(h.bt, 0);
    cudaGraphSetConditional(h.rest, 0);
    cudaGraphSetConditional(h.outer, 0);
  };
  if (!isfinite(fx)) { stop(TVR_E_NONFINITE); return; }
  const double rhs = __dadd_rn(__dadd_rn(d->fy, gd), __dmul_rn(__dmul_rn(0.5, d->bt_L), dd));
  if (!(fx > rhs)) {
    d->bt_f = fx;
    cudaGraphSetConditional(h.bt, 0);
    cudaGraphSetConditional(h.rest, 1);
    return;
  }
  if (d->bt_trials >= d->bt_max) { stop(TVR_E_LINESEARCH); return; }
  d->bt_L = __dmul_rn(d->bt_L, d->rho_L);
  d->dp_trial[0] = 1.0 / d->bt_L;
  cudaGraphSetConditional(h.bt, 1);
}

// After BT: L_k, mu_k (Eq. (9), C9), theta_{k+1}, beta_k; parameters of the stop
// stencil (nu = L_k, C11) and of the momentum point.
__global__ void upn_mid_kernel(UpnDev* d, UpnHandles h) {
  if (!d->status) {
    d->n_f += d->bt_trials;
    d->n_ls += d->bt_trials;
    d->L = d->bt_L;
    if (!d->first && d->mu_dd > 0.0) {
      const double M = __dsub_rn(__dsub_rn(d->fxk, d->fy), d->mu_gd) / __dmul_rn(0.5, d->mu_dd);
      if (M > 0.0 && isfinite(M)) d->mu = fmin(d->mu, M);
    }
    d->theta_n = dev_theta_root(d->theta, d->mu / d->L);
    if (!(d->theta_n > 0.0 && d->theta_n <= 1.0) || !isfinite(d->theta_n)) {
      d->status = TVR_E_THETA;
      cudaGraphSetConditional(h.rest, 0);
      cudaGraphSetConditional(h.outer, 0);
      return;
    }
    d->beta = __dmul_rn(d->theta, 1.0 - d->theta) /
              __dadd_rn(__dmul_rn(d->theta, d->theta), d->theta_n);
    d->dp_stop[0] = 0.0;
    d->dp_stop[1] = 1.0 / d->L;
    d->dp_stop[2] = 0.0;
    d->dp_mom[0] = d->beta;
    d->dp_mom[1] = 0.0;
    d->dp_mom[2] = d->beta;
  }
}

// End of iteration: stop test at x_{k+1}, f(y_{k+1}) by linearity (a6), record.
__global__ void upn_end_kernel(UpnDev* d, const double* sc, UpnHandles h) {
  ++d->n_g;
  d->gn = __dmul_rn(d->L, sqrt(sc[S_TV + 3]));
  ++d->k;
  d->fxk = d->bt_f;
  d->fy = __dadd_rn(__dmul_rn(0.5, sc[S_MOM]), __dmul_rn(d->alpha, sc[S_TV2]));
  d->theta = d->theta_n;
  d->first = 0;
  d->conv = dev_stop_test(d->gn, d->gref, d->N, d->eps, d->stop_mode) ? 1 : 0;
  if (d->n_rec < d->rec_cap) {
    tvr_record r{};
    r.iter = d->k;
    r.f = d->fxk;
    r.gmap_rel = d->gref > 0 ? d->gn / d->gref : 0.0;
    r.gmap_abs_per_n = d->gn / d->N;
    r.step_or_inv_L = 1.0 / d->L;
    r.mu = d->mu;
    r.L = d->L;
    r.ls_trials = d->bt_trials;
    d->rec[d->n_rec] = r;
  }
  ++d->n_rec;
  if (!isfinite(d->fy)) d->status = TVR_E_NONFINITE;
  cudaGraphSetConditional(h.outer, (!d->status && !d->conv && d->k < d->max_iters) ? 1 : 0);
}

cudaError_t launch_upn_bt_begin(UpnDev* d, UpnHandles h, cudaStream_t st) {
  upn_bt_begin_kernel<<<1, 1, 0, st>>>(d, h);
  return cudaGetLastError();
}
cudaError_t launch_upn_bt(UpnDev* d, const double* scal, UpnHandles h, cudaStream_t st) {
  upn_bt_kernel<<<1, 1, 0, st>>>(d, scal, h);
  return cudaGetLastError();
}
cudaError_t launch_upn_mid(UpnDev* d, UpnHandles h, cudaStream_t st) {
  upn_mid_kernel<<<1, 1, 0, st>>>(d, h);
  return cudaGetLastError();
}
cudaError_t launch_upn_end(UpnDev* d, const double* scal, UpnHandles h, cudaStream_t st) {
  upn_end_kernel<<<1, 1, 0, st>>>(d, scal, h);
  return cudaGetLastError();
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
