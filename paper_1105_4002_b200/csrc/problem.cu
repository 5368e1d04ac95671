// libtvreg: problem creation, device memory, SpMV plans, pass functions and the C ABI
// entry points other than the solvers (solvers.cu) and NCCL plumbing (dist.cu).
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <numeric>
#include <vector>

#include "problem.h"

namespace tvr {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

const char* kKernelNames[K_COUNT] = {"spmv_A", "spmv_AT", "tv_grad", "tv_trial",
                                     "momentum", "project", "gmap"};

static tvr_alloc_fn g_alloc = nullptr;
static tvr_free_fn g_free = nullptr;
static void* g_alloc_ctx = nullptr;

int dev_alloc(tvr_problem* p, void** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* q = nullptr;
  if (g_alloc) {
    q = g_alloc(bytes, p->device, (void*)p->stream, g_alloc_ctx);
  } else if (cudaMalloc(&q, bytes) != cudaSuccess) {
    cudaGetLastError();
    q = nullptr;
  }
  if (!q) {
    set_error("device allocation of " + std::to_string(bytes) + " bytes failed");
    return TVR_E_OOM;
  }
  p->allocs.push_back(q);
  p->device_bytes += (int64_t)bytes;
  *ptr = q;
  return TVR_OK;
}

void dev_free(tvr_problem* p, void* q) {
  for (size_t i = 0; i < p->allocs.size(); ++i)
    if (p->allocs[i] == q) {
      if (g_free) g_free(q, p->device, (void*)p->stream, g_alloc_ctx);
      else cudaFree(q);
      p->allocs.erase(p->allocs.begin() + i);
      return;
    }
}

static void dev_free_all(tvr_problem* p) {
  for (void* q : p->allocs) {
    if (g_free) g_free(q, p->device, (void*)p->stream, g_alloc_ctx);
    else cudaFree(q);
  }
  p->allocs.clear();
}

int64_t n_local(const tvr_problem* p) { return p->plane * p->nzl; }
float* volvec(tvr_problem* p, int i) { return p->vol[i]; }
// first element and length of the allocation behind volume vector v (halo planes, or in VIEWS_REP
// the whole replicated volume)
void vol_extent(const tvr_problem* p, float* v, float** first, int64_t* count) {
  if (rep_dist(p)) {
    *first = v - (int64_t)p->z0 * p->plane;
    *count = (int64_t)p->nz * p->plane;
  } else {
    *first = v - p->plane;
    *count = (int64_t)(p->nzl + 2) * p->plane;
  }
}
float* datvec(tvr_problem* p, int i) { return p->dat[i]; }

// --------------------------------------------------------------- timing
static cudaEvent_t get_event(tvr_problem* p) {
  if (!p->event_pool.empty()) {
    cudaEvent_t e = p->event_pool.back();
    p->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

static void resolve_timings(tvr_problem* p) {
  for (auto& t : p->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
      p->kt_ms[t.kid] += ms;
      p->kt_bytes[t.kid] += t.bytes;
      p->kt_launches[t.kid] += 1;
    }
    p->event_pool.push_back(t.a);
    p->event_pool.push_back(t.b);
  }
  p->pending.clear();
}

template <class F>
static int launch(tvr_problem* p, int kid, double bytes, F&& f) {
  NvtxRange nv(kKernelNames[kid]);
  cudaEvent_t a = nullptr, b = nullptr;
  if (p->prof) {
    a = get_event(p);
    b = get_event(p);
    cudaEventRecord(a, p->stream);
  }
  cudaError_t e = f();
  if (e != cudaSuccess) {
    set_error(std::string("kernel ") + kKernelNames[kid] + ": " + cudaGetErrorString(e));
    return TVR_E_CUDA;
  }
  if (p->prof) {
    cudaEventRecord(b, p->stream);
    p->pending.push_back({kid, a, b, bytes});
  }
  p->launches++;
  p->bytes_total += bytes;
  return TVR_OK;
}

static int elem_grid(tvr_problem* p, int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)p->num_sms * 8));
}

// ----------------------------------------------------------------- passes
static SpmvArgs spmv_args(tvr_problem* p, const SpmvPlan& pl, bool transposed, const float* src,
                          const float* b, float* out, double* scal) {
  SpmvArgs a{};
  a.out_lo = nullptr;
  a.out_peer = nullptr;
  a.out_bounds = nullptr;
  a.n_out = 0;
  a.rp = transposed ? p->rpT : p->rp;
  a.col = transposed ? p->colT : p->col;
  a.col16 = transposed ? p->colT16 : p->col16;
  a.val = transposed ? p->valT : p->val;
  a.src = src;
  a.b = b;
  a.out = out;
  a.item_row = pl.item_row;
  a.item_slice = pl.item_slice;
  a.slice_item_end = pl.slice_item_end;
  a.nitems = pl.nitems;
  a.win_lo = pl.win_lo;
  a.win_len = pl.win_len;
  a.parts = pl.parts;
  a.part_len = pl.part_len > 0 ? pl.part_len : (1 << 30);
  a.nrows = pl.nrows;
  a.part_off = pl.part_off;
  a.part_acc = pl.part_acc;
  a.partials = p->partials;
  a.counter = p->counter;
  a.scal = scal;
  return a;
}

// Launch one SpMV pass with the plan's kernel: sliced ELL (16-bit or int32), else the padded or
// plain per-row kernel.
static cudaError_t run_spmv(tvr_problem* p, const SpmvPlan& pl, bool transposed, const float* src,
                            const float* b, float* out, float* out_lo, double* scal,
                            int z_lo = 0, int z_hi = -1, const float* src_lo = nullptr) {
  // src_lo (extended-precision solver iterates): the sliced-ELL kernels only (p->ext_eval)
  if (src_lo && !(pl.sell32 || pl.sell)) return cudaErrorNotSupported;
  if (pl.sell32) {  // int32 sliced ELL (non-separable: no slice ranges)
    const SellData& d = pl.sd[0];
    SellArgs s{};
    s.blk_off = d.off;
    s.blk_k = d.k;
    s.blk_slice = d.slice;
    s.zend = d.zend;
    s.blk_sq = d.sq;
    s.cum = d.cum;
    s.perm = d.perm;
    s.col32 = d.col32;
    s.row_start = d.row_start;
    s.rp = transposed ? p->rpT : p->rp;
    s.val = d.val;
    s.src = src;
    s.src_lo = src_lo;
    if (pl.sell32_layouts) {  // the point in the three gather layouts (columns index into them)
      cudaError_t e = launch_relayout(src, p->xs, p->nx, p->ny, p->ncol, p->stream);
      if (e != cudaSuccess) return e;
      s.src = p->xs;
      if (src_lo) {
        e = launch_relayout(src_lo, p->xs_lo, p->nx, p->ny, p->ncol, p->stream);
        if (e != cudaSuccess) return e;
        s.src_lo = p->xs_lo;
      }
    }
    s.b = b;
    s.out = out;
    s.out_lo = out_lo;
    s.blk_lo = 0;
    s.blk_hi = d.nblk;
    s.nb = d.nblk;
    s.rep = 1;
    s.ilv = pl.sell32_ilv;
    s.l2hint = pl.sell32_l2;
    s.partials = p->partials;
    s.counter = p->counter;
    s.scal = scal;
    if (transposed && p->fused_rs) {  // VIEWS A^T: rows stored into their owners' inboxes
      s.out_peer = p->out_peer_dev;
      s.out_bounds = p->out_bounds_dev;
      s.n_out = p->world;
    }
    if (d.nblk == 0) return scal ? cudaMemsetAsync(scal, 0, sizeof(double), p->stream) : cudaSuccess;
    return launch_spmv32s(s, pl.sv.unroll, (int)std::min<int64_t>(pl.pad_grid, d.nblk), p->stream,
                          pl.sv.block);
  }
  if (pl.sell) {  // slices [z_lo, z_hi) (the e2e pipeline's chunks) or all; column parts in order
    const int P = (int)pl.sd.size();
    for (int q = 0; q < P; ++q) {
      const SellData& d = pl.sd[q];
      SellArgs s{};
      s.blk_off = d.off;
      s.blk_k = d.k;
      s.blk_slice = d.slice;
      s.zend = d.zend;
      s.blk_sq = d.sq;
      s.cum = d.cum;
      s.perm = d.perm;
      s.col16 = d.col16;
      s.val = d.val;
      s.src = src;
      s.src_lo = src_lo;
      // stage the lo window too when both fit (c2: 2 x 66 KB): the hi window occupies
      // pl.smem bytes, the lo one the same amount after it
      if (src_lo && pl.staged && !pl.sv.half && 2 * pl.smem + 2048 <= (size_t)p->max_smem_optin)
        s.lo_off = (int32_t)(pl.smem / sizeof(float));
      s.b = q == P - 1 ? b : nullptr;
      s.out = out;
      s.out_lo = q == P - 1 ? out_lo : nullptr;
      s.acc_in = q > 0 ? pl.sell_acc : nullptr;
      s.acc_out = q < P - 1 ? pl.sell_acc : nullptr;
      s.blk_lo = z_hi >= 0 ? (z_lo > 0 ? d.h_slice_end[z_lo - 1] : 0) : 0;
      s.blk_hi = z_hi >= 0 ? d.h_slice_end[z_hi - 1] : d.nblk * pl.rep;
      s.nb = d.nblk;
      s.rep = pl.rep;
      s.rep_rows = pl.rep_rows;
      s.rep_win = pl.rep_win;
      s.rep_total = pl.rep_total;
      s.wstride = pl.wstride;
      s.win_lo = d.win_lo;
      s.win_len = d.win_len;
      s.part_len = pl.part_len;
      s.partials = p->partials;
      s.counter = p->counter;
      s.scal = q == P - 1 ? scal : nullptr;
      if (s.blk_hi <= s.blk_lo) {
        if (s.scal) {  // nothing to sum: the pass still defines its scalar
          cudaError_t e = cudaMemsetAsync(s.scal, 0, sizeof(double), p->stream);
          if (e != cudaSuccess) return e;
        }
        continue;
      }
      const int g = (int)std::min<int64_t>(pl.pad_grid, std::max<int64_t>(1, s.blk_hi - s.blk_lo));
      if (z_hi < 0 && d.cta_tab && d.cta_tab_grid == g) {  // full range: plan-time CTA ranges
        s.cta_tab = d.cta_tab;
        s.cta_tab_grid = g;
      }
      // diagnostic: per-CTA start / end times and SM ids of every full-range launch on stderr
      static const bool cta_prof = [] { const char* v = std::getenv("TVR_SELL_PROF"); return v && *v == '1'; }();
      static long long* prof_buf = nullptr;
      if (cta_prof && z_hi < 0) {
        if (!prof_buf) cudaMalloc(&prof_buf, sizeof(long long) * 3 * 1024);
        s.cta_prof = prof_buf;
      }
      cudaError_t e = launch_spmv16s(s, pl.sv, g, pl.smem, p->stream);
      if (e != cudaSuccess) return e;
      if (s.cta_prof) {
        std::vector<long long> hb(3 * 1024);
        cudaMemcpyAsync(hb.data(), prof_buf, sizeof(long long) * 3 * g, cudaMemcpyDeviceToHost, p->stream);
        cudaStreamSynchronize(p->stream);
        const long long* prof_buf = hb.data();
        long long t0 = prof_buf[0], t1 = 0;
        for (int i = 0; i < g; ++i) { t0 = std::min(t0, prof_buf[3 * i]); t1 = std::max(t1, prof_buf[3 * i + 1]); }
        std::fprintf(stderr, "SELLPROF %s part %d grid %d span_ns %lld :", transposed ? "AT" : "A", q, g, t1 - t0);
        for (int i = 0; i < g; ++i)
          std::fprintf(stderr, " %lld,%lld,%lld", prof_buf[3 * i] - t0, prof_buf[3 * i + 1] - t0, prof_buf[3 * i + 2]);
        std::fprintf(stderr, "\n");
      }
    }
    return cudaSuccess;
  }
  int64_t it_lo = 0, it_hi = -1;  // per-row kernels: the items of slices [z_lo, z_hi)
  if (z_hi >= 0) {
    it_lo = z_lo > 0 ? pl.h_slice_item_end[z_lo - 1] : 0;
    it_hi = pl.h_slice_item_end[z_hi - 1];
  }
  if (it_hi >= 0) {  // items [it_lo, it_hi) only (per-row kernels; the e2e pipeline's chunks)
    SpmvArgs a = spmv_args(p, pl, transposed, src, b, out, scal);
    a.out_lo = out_lo;
    a.item_row += it_lo;
    a.item_slice += it_lo;
    a.nitems = it_hi - it_lo;
    if (pl.pad) {
      a.rp = pl.rpp;
      a.col16 = pl.col16p;
      a.col = pl.col32p;
      a.val = pl.valp;
      const int g = (int)std::min<int64_t>(pl.pad_grid, std::max<int64_t>(1, a.nitems));
      return pl.v.idx16 ? launch_spmv16p(a, pl.v, g, pl.block, pl.smem, p->stream)
                        : launch_spmv32p(a, pl.v, g, pl.block, p->stream);
    }
    return launch_spmv(a, pl.v, (int)std::min<int64_t>(pl.grid, std::max<int64_t>(1, a.nitems)),
                       pl.block, pl.smem, p->stream);
  }
  SpmvArgs a = spmv_args(p, pl, transposed, src, b, out, scal);
  a.out_lo = out_lo;
  if (transposed && p->fused_rs) {  // VIEWS A^T: rows stored into their owners' inboxes
    a.out_peer = p->out_peer_dev;
    a.out_bounds = p->out_bounds_dev;
    a.n_out = p->world;
  }
  if (pl.pad) {
    a.rp = pl.rpp;
    a.col16 = pl.col16p;
    a.col = pl.col32p;
    a.val = pl.valp;
    return pl.v.idx16 ? launch_spmv16p(a, pl.v, pl.pad_grid, pl.block, pl.smem, p->stream)
                      : launch_spmv32p(a, pl.v, pl.pad_grid, pl.block, p->stream);
  }
  return launch_spmv(a, pl.v, pl.grid, pl.block, pl.smem, p->stream);
}

// Algorithmic bytes per entry: fp32 value + int32 column, or + 16-bit column offset.
static double entry_bytes(const SpmvPlan& pl) { return pl.v.idx16 ? 6.0 : 8.0; }

// x: a slab volume vector.  VIEWS mode gathers the whole point first (gather_volume).
int pass_residual(tvr_problem* p, const float* x, float* r, int slot, float* r_lo,
                  const float* x_lo) {
  const float* src = x;
  TVR_TRY(gather_volume(p, x, &src));
  if (x_lo) {  // A (x + x_lo): extended-precision iterate evaluated whole (p->ext_eval)
    const double nnz_hbm = p->sliced ? (double)p->nnz_s : (double)p->nnz;
    const double bytes = entry_bytes(p->planA) * nnz_hbm + 8.0 * ((p->sliced ? p->m_s : p->m) + 1.0) +
                         8.0 * p->ncol + 8.0 * p->m + (r_lo ? 4.0 * p->m : 0.0);
    return launch(p, K_SPMV_A, bytes, [&] {
      return run_spmv(p, p->planA, false, src, p->b, r, r_lo, p->dscal + slot, 0, -1, x_lo);
    });
  }
  // slice-shared operator: the one stored slice matrix is read from HBM once (L2 after that)
  const double nnz_hbm = p->sliced ? (double)p->nnz_s : (double)p->nnz;
  const double rows_hbm = p->sliced ? (double)p->m_s : (double)p->m;
  const double bytes = entry_bytes(p->planA) * nnz_hbm + 8.0 * (rows_hbm + 1) + 4.0 * p->ncol +
                       8.0 * p->m + (r_lo ? 4.0 * p->m : 0.0);
  return launch(p, K_SPMV_A, bytes, [&] {
    return run_spmv(p, p->planA, false, src, p->b, r, r_lo, p->dscal + slot);
  });
}

// w: a slab volume vector.  VIEWS mode computes the full-volume partial A_p^T r_p and
// reduce-scatters it to the slabs.
// w: a slab volume vector.  VIEWS mode computes the full-volume partial A_p^T r_p and
// reduce-scatters it to the slabs: fused (the A^T kernel stores every row straight into its
// owner's inbox over peer memory, the owner sums the inboxes in rank order) or through NCCL.
int pass_AT(tvr_problem* p, const float* r, float* w) {
  float* dst = views_dist(p) ? p->wfull : w;
  const double bytes = entry_bytes(p->planT) * (p->sliced ? (double)p->nnz_s : (double)p->nnz) +
                       8.0 * ((p->sliced ? (double)p->plane : (double)p->ncol) + 1) + 4.0 * p->m +
                       4.0 * p->ncol;
  if (p->fused_rs) TVR_TRY(dist_barrier(p));  // every owner has consumed the previous inbox
  TVR_TRY(launch(p, K_SPMV_AT, bytes, [&] {
    return run_spmv(p, p->planT, true, r, nullptr, dst, nullptr, nullptr);
  }));
  if (p->fused_rs) {
    TVR_TRY(dist_barrier(p));  // every rank's stores into this rank's inbox are complete
    TVR_CUDA(launch_inbox_sum(p->slab_cnt[p->rank], p->inbox, p->inbox_stride, p->world, w,
                              p->stream));
    return TVR_OK;
  }
  if (views_dist(p)) TVR_TRY(reduce_scatter_volume(p, dst, w));
  return TVR_OK;
}

static TVArgs tv_args(tvr_problem* p, int slot) {
  TVArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nx = p->nx;
  a.ny = p->ny;
  a.nzl = p->nzl;
  a.plane = p->plane;
  a.zg0 = p->z0;
  a.nzg = p->nz;
  a.tau = p->tau;
  a.alpha = p->alpha;
  a.lo = p->lo;
  a.hi = p->hi;
  a.partials = p->partials;
  a.counter = p->counter;
  a.scal = p->dscal + slot;
  return a;
}

int pass_tv_grad(tvr_problem* p, const float* x, const float* x0, double beta, const float* w1,
                 const float* w0, double wbeta, float* g, float* v_out, const float* xp,
                 const float* gp, double stop_step, int slot, double alpha, const double* dparam) {
  TVArgs a = tv_args(p, slot);
  a.dparam = dparam;
  a.alpha = alpha;
  a.w1 = w1;
  a.w0 = w0;
  a.wbeta = wbeta;
  a.g_out = g;
  a.v_out = v_out;
  a.xp = xp;
  a.gp = gp;
  a.stop_step = stop_step;
  const double N = (double)n_local(p);
  const double bytes = N * (4.0 * (x0 ? 2 : 1) + (w1 ? 4.0 : 0.0) + (w0 ? 4.0 : 0.0) +
                            (g ? 4.0 : 0.0) + (v_out ? 4.0 : 0.0) + (xp ? 8.0 : 0.0));
  return launch(p, K_TV_GRAD, bytes, [&] {
    return x0 ? launch_tv_grad_momentum(a, x, x0, beta, p->stream)
              : launch_tv_grad_plain(a, x, p->stream);
  });
}

int pass_tv_grad(tvr_problem* p, const float* x, const float* x0, double beta, const float* w1,
                 const float* w0, double wbeta, float* g, float* v_out, const float* xp,
                 const float* gp, double stop_step, int slot) {
  return pass_tv_grad(p, x, x0, beta, w1, w0, wbeta, g, v_out, xp, gp, stop_step, slot, p->alpha);
}

int pass_tv_trial(tvr_problem* p, const float* x, const float* g, double s, float* v,
                  double stop_step, const float* xo, int slot, const double* dparam) {
  TVArgs a = tv_args(p, slot);
  a.dparam = dparam;
  a.v_out = v;
  a.tx = x;
  a.tg = g;
  a.xo = xo;
  a.stop_step = stop_step;
  const double N = (double)n_local(p);
  const double bytes = N * (12.0 + (xo ? 4.0 : 0.0));
  return launch(p, K_TV_TRIAL, bytes, [&] { return launch_tv_trial(a, x, g, s, p->stream); });
}

int pass_tv_grad_x(tvr_problem* p, const float* x, const float* x_lo, const float* w1, float* g,
                   double stop_step, int slot, const double* dparam) {
  TVArgs a = tv_args(p, slot);
  a.dparam = dparam;
  a.w1 = w1;
  a.g_out = g;
  a.stop_step = stop_step;
  const double N = (double)n_local(p);
  return launch(p, K_TV_GRAD, N * (12.0 + (g ? 4.0 : 0.0)),
                [&] { return launch_tv_grad_plain_x(a, x, x_lo, p->stream); });
}

int pass_tv_trial_x(tvr_problem* p, const float* x, const float* x_lo, const float* g, double s,
                    float* v, float* v_lo, const float* xo, const float* xo_lo, int slot,
                    const double* dparam) {
  TVArgs a = tv_args(p, slot);
  a.dparam = dparam;
  a.v_out = v;
  a.v_lo_out = v_lo;
  a.tx = x;
  a.tg = g;
  a.xo = xo;
  a.xo_lo = xo_lo;
  a.stop_step = 0.0;
  const double N = (double)n_local(p);
  const double bytes = N * (20.0 + (xo ? 8.0 : 0.0));
  return launch(p, K_TV_TRIAL, bytes,
                [&] { return launch_tv_trial_x(a, x, x_lo, g, s, p->stream, p->ext_on); });
}

int pass_tv_momentum_x(tvr_problem* p, const float* x1, const float* x1_lo, const float* x0,
                       const float* x0_lo, double beta, const float* w1, const float* w0,
                       float* g, float* y, float* y_lo, int slot, const double* dparam) {
  TVArgs a = tv_args(p, slot);
  a.dparam = dparam;
  a.w1 = w1;
  a.w0 = w0;
  a.wbeta = beta;
  a.g_out = g;
  a.v_out = y;
  a.v_lo_out = y_lo;
  const double N = (double)n_local(p);
  return launch(p, K_TV_GRAD, N * 36.0, [&] {
    return launch_tv_grad_momentum_x(a, x1, x1_lo, x0, x0_lo, beta, p->stream, p->ext_on);
  });
}

int pass_momentum(tvr_problem* p, const float* r1, const float* r1lo, const float* r0,
                  const float* r0lo, double beta, int slot, const double* dbeta) {
  const int grid = elem_grid(p, p->m);
  return launch(p, K_MOMENTUM, 16.0 * p->m, [&] {
    return launch_momentum_resid(p->m, r1, r1lo, r0, r0lo, beta, p->partials, p->counter,
                                 p->dscal + slot, grid, p->stream, dbeta);
  });
}

int pass_project(tvr_problem* p, float* x) {
  const int64_t n = n_local(p);
  const int grid = elem_grid(p, n);
  return launch(p, K_PROJECT, 8.0 * n,
                [&] { return launch_project(n, x, p->lo, p->hi, grid, p->stream); });
}

int pass_gmap(tvr_problem* p, const float* x, const float* g, double nu, float* G, int slot) {
  const int64_t n = n_local(p);
  const int grid = elem_grid(p, n);
  return launch(p, K_GMAP, (G ? 12.0 : 8.0) * n, [&] {
    return launch_gradient_map(n, x, g, nu, p->lo, p->hi, G, p->partials, p->counter,
                               p->dscal + slot, grid, p->stream);
  });
}

int fetch_scalars(tvr_problem* p, int nslots) {
  if (p->world > 1) return dist_sum_scalars(p, p->hscal, nslots);
  TVR_CUDA(cudaMemcpyAsync(p->hscal, p->dscal, sizeof(double) * nslots, cudaMemcpyDeviceToHost,
                           p->stream));
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  if (p->prof) resolve_timings(p);
  return TVR_OK;
}

void resolve_pending_timings(tvr_problem* p) {
  if (p->prof) resolve_timings(p);
}

// ------------------------------------------------------------------ plans
// Split rows [r0, r1) into items of about `target` nonzeros (at least one row each).
static void split_rows(const int64_t* rp, int64_t r0, int64_t r1, int64_t target, int32_t slice,
                       std::vector<int64_t>& rows, std::vector<int32_t>& slices) {
  int64_t start = r0;
  while (start < r1) {
    int64_t end = start + 1;
    const int64_t lim = rp[start] + target;
    // binary search the first row boundary reaching lim
    int64_t lo = start + 1, hi = r1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (rp[mid] >= lim) hi = mid;
      else lo = mid + 1;
    }
    end = std::max(end, lo);
    rows.push_back(start);
    slices.push_back(slice);
    start = end;
  }
}

// Lanes per row from the mean row length: 16-byte chunks of 4 entries, about one to two
// chunk pairs per row.
// Measured at c2 (scripts/sweep_spmv.py): 4-entry chunks: LPR 8 for rows of 76 and 115;
// 8-entry chunks (16-bit columns): LPR 8 for 115, LPR 4 for 76.
static int lpr_for(double mean_len, int chunk) {
  const double per_chunk_rows = mean_len / chunk;  // chunks per row
  return per_chunk_rows > 40 ? 16 : (per_chunk_rows > 12 ? 8 : 4);
}

// Tuning overrides (TVR_LPR_A, TVR_LPR_AT, TVR_SPMV_BLOCK, TVR_SPMV_STAGE=0); unset in production.
static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

static int upload(tvr_problem* p, void** dst, const void* src, size_t bytes) {
  TVR_TRY(dev_alloc(p, dst, bytes));
  if (src && bytes) TVR_CUDA(cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, p->stream));
  return TVR_OK;
}

// CTA block ranges by SIMULATED MAKESPAN (round 2).  The sliced-ELL kernel walks a CTA's range
// slice segment by slice segment (barrier, window restage), and inside a segment its warps take
// blocks from a counter in stored order (longest rows of the slice first).  Equal work sums do
// not finish together: a range that ends a few blocks into the next slice leaves most warps idle
// while a handful run that slice's longest blocks (c2 A pass: CTA times 128-150 us around a
// 139 us mean, the slow ones exactly those ranges, scripts/sell_prof.py).  So the ranges are cut
// where the kernel's own schedule -- list scheduling of block costs (steps + blk_cost) on
// `nwarps` warps per segment, seg_cost per segment -- reaches a common makespan T, the smallest
// T (bisection) that needs no more than `grid` CTAs.  tab[i] = first block of CTA i, tab[grid] =
// nblk.
static std::vector<int64_t> makespan_partition(const std::vector<int32_t>& k,
                                               const std::vector<int32_t>& slice, int nwarps,
                                               int grid, double blk_cost, double seg_cost,
                                               double lambda) {
  const int64_t nb = (int64_t)k.size();
  std::vector<double> heap((size_t)nwarps);
  // Incremental cost of a range that grows block by block: lambda x simulated makespan +
  // (1 - lambda) x work sum per warp (the pass is bandwidth-bound, so a CTA's idle warps are
  // partly made up by the other SMs: measured CTA times lie between the two models).
  struct Sim {
    double seg_base, seg_max, work;
    int cur_slice;
    int64_t taken;
  };
  auto reset = [&](Sim& m, int sl) {
    m.seg_base = seg_cost;
    m.seg_max = 0.0;
    m.work = seg_cost * nwarps;
    m.cur_slice = sl;
    m.taken = 0;
    std::fill(heap.begin(), heap.end(), 0.0);
  };
  // cost if block i were added (does not modify); commit = true adds it
  auto add = [&](Sim& m, int64_t i, bool commit) -> double {
    double sb = m.seg_base, sm = m.seg_max, wk = m.work;
    const bool new_seg = slice[i] != m.cur_slice;
    if (new_seg) {  // barrier: the next segment starts when the current one has drained
      sb = m.seg_base + m.seg_max + seg_cost;
      sm = 0.0;
      wk += seg_cost * nwarps;
    }
    const double c = (double)k[i] + blk_cost;
    const double fin = (new_seg ? 0.0 : heap.front()) + c;  // earliest-free warp takes the block
    wk += c;
    const double cost = lambda * (sb + std::max(sm, fin)) + (1.0 - lambda) * wk / nwarps;
    if (commit) {
      if (new_seg) {
        std::fill(heap.begin(), heap.end(), 0.0);
        m.cur_slice = slice[i];
      }
      std::pop_heap(heap.begin(), heap.end(), std::greater<double>());
      heap.back() = fin;
      std::push_heap(heap.begin(), heap.end(), std::greater<double>());
      m.seg_base = sb;
      m.seg_max = std::max(sm, fin);
      m.work = wk;
      ++m.taken;
    }
    return cost;
  };
  auto range_cost = [&](int64_t b0, int64_t b1) -> double {
    if (b1 <= b0) return 0.0;
    Sim m;
    reset(m, slice[b0]);
    double c = 0.0;
    for (int64_t i = b0; i < b1; ++i) c = add(m, i, true);
    return c;
  };
  auto cut = [&](double T, std::vector<int64_t>* out) -> int64_t {
    // greedy: extend the current CTA block by block while its cost stays <= T
    int64_t ctas = 0, i = 0;
    if (out) out->assign(1, 0);
    Sim m;
    while (i < nb) {
      ++ctas;
      reset(m, slice[i]);
      while (i < nb) {
        if (m.taken > 0 && add(m, i, false) > T) break;
        add(m, i, true);
        ++i;
      }
      if (out) out->push_back(i);
    }
    return ctas;
  };
  double total = 0.0, longest = 0.0;
  for (int64_t i = 0; i < nb; ++i) {
    total += k[i] + blk_cost;
    longest = std::max(longest, (double)k[i] + blk_cost);
  }
  double lo = total / ((double)grid * nwarps), hi = 2.0 * lo + 4.0 * (longest + seg_cost) + 1.0;
  while (cut(hi, nullptr) > grid) hi *= 2.0;
  for (int it = 0; it < 40 && hi - lo > 1e-3 * hi; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (cut(mid, nullptr) <= grid) hi = mid;
    else lo = mid;
  }
  std::vector<int64_t> tab;
  cut(hi, &tab);
  // the greedy cut may need fewer CTAs than the grid has (its count jumps with T): halve the
  // costliest ranges until every CTA has one
  while ((int64_t)tab.size() - 1 < grid) {
    size_t worst = 0;
    double wc = -1.0;
    for (size_t c = 0; c + 1 < tab.size(); ++c) {
      if (tab[c + 1] - tab[c] < 2) continue;
      const double rc = range_cost(tab[c], tab[c + 1]);
      if (rc > wc) { wc = rc; worst = c; }
    }
    if (wc < 0.0) break;  // nothing left to split
    const int64_t b0 = tab[worst], b1 = tab[worst + 1];
    int64_t best = b0 + 1;
    double bc = 1e300;
    int64_t lo_b = b0 + 1, hi_b = b1 - 1;  // the cut where both halves cost the same (bisection)
    while (lo_b <= hi_b) {
      const int64_t mid = (lo_b + hi_b) / 2;
      const double c0 = range_cost(b0, mid), c1 = range_cost(mid, b1);
      if (std::max(c0, c1) < bc) { bc = std::max(c0, c1); best = mid; }
      if (c0 < c1) lo_b = mid + 1;
      else hi_b = mid - 1;
    }
    tab.insert(tab.begin() + (std::ptrdiff_t)worst + 1, best);
  }
  tab.resize((size_t)grid + 1, nb);
  tab[(size_t)grid] = nb;
  return tab;
}

// One sliced-ELL structure: per slice (prow / psl: the per-row plan's items), rows stably sorted
// by 8-entry chunk count of `lens` (descending) in blocks of 32; entries [lo_off, hi_off) of each
// row with coff subtracted from the offsets; the windows shifted by coff and clipped to part_h
// (0: whole).  ok = false when it does not fit in free device memory.
static int build_sell_data(tvr_problem* p, SpmvPlan& pl, bool transposed,
                           const std::vector<int64_t>& prow, const std::vector<int32_t>& psl,
                           const std::vector<int64_t>& lens, const int32_t* lo_off,
                           const int32_t* hi_off, int coff, int part_h,
                           const std::vector<int64_t>& wlo, const std::vector<int32_t>& wlen,
                           SellData& d, bool& ok) {
  ok = false;
  const int64_t nitems = (int64_t)psl.size();
  std::vector<int64_t> off, cum(1, 0), zend(pl.h_slice_item_end.size(), 0);
  std::vector<int32_t> kk, sl, perm, idx;
  int64_t steps = 0;
  const int64_t wcost = env_int("TVR_SELL_BLKCOST", 2);
  for (int64_t i = 0; i < nitems;) {
    int64_t e = i + 1;
    while (e < nitems && psl[e] == psl[i]) ++e;
    const int64_t R0 = prow[i], R1 = prow[e];
    idx.resize(R1 - R0);
    for (int64_t r = R0; r < R1; ++r) idx[r - R0] = (int32_t)r;
    auto nch = [&](int32_t r) { return (lens[r] + 7) / 8; };
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t x, int32_t y) { return nch(x) > nch(y); });
    for (size_t j = 0; j < idx.size(); j += 32) {
      const int64_t K = nch(idx[j]);
      off.push_back(steps);
      kk.push_back((int32_t)K);
      sl.push_back(psl[i]);
      cum.push_back(cum.back() + K + wcost);
      for (size_t l = 0; l < 32; ++l) perm.push_back(j + l < idx.size() ? idx[j + l] : -1);
      steps += K;
    }
    if ((size_t)psl[i] < zend.size()) zend[psl[i]] = (int64_t)kk.size();
    i = e;
  }
  for (size_t z = 1; z < zend.size(); ++z) zend[z] = std::max(zend[z], zend[z - 1]);
  const int64_t nblk = (int64_t)kk.size();
  const size_t cap = (size_t)steps * 256 + 8;
  const size_t need = cap * 6 + (size_t)nblk * (8 + 4 + 4 + 8 + 128);
  size_t fr = 0, tot = 0;
  TVR_CUDA(cudaMemGetInfo(&fr, &tot));
  if (need + ((size_t)1 << 30) > fr) return TVR_OK;  // keep 1 GB of headroom
  std::vector<int64_t> wl(wlo.size());
  std::vector<int32_t> wn(wlen.size());
  for (size_t z = 0; z < wlo.size(); ++z) {
    wl[z] = wlo[z] + coff;
    const int32_t rest = std::max<int32_t>(0, wlen[z] - coff);
    wn[z] = part_h > 0 ? std::min<int32_t>(rest, part_h) : rest;
  }
  TVR_TRY(upload(p, (void**)&d.off, off.data(), sizeof(int64_t) * off.size()));
  TVR_TRY(upload(p, (void**)&d.k, kk.data(), sizeof(int32_t) * kk.size()));
  TVR_TRY(upload(p, (void**)&d.slice, sl.data(), sizeof(int32_t) * sl.size()));
  d.h_k = kk;
  d.h_slice = sl;
  TVR_TRY(upload(p, (void**)&d.cum, cum.data(), sizeof(int64_t) * cum.size()));
  TVR_TRY(upload(p, (void**)&d.zend, zend.data(), sizeof(int64_t) * zend.size()));
  TVR_TRY(upload(p, (void**)&d.win_lo, wl.data(), sizeof(int64_t) * wl.size()));
  TVR_TRY(upload(p, (void**)&d.win_len, wn.data(), sizeof(int32_t) * wn.size()));
  TVR_TRY(dev_alloc(p, (void**)&d.sq, sizeof(double) * std::max<int64_t>(1, nblk * pl.rep)));
  TVR_TRY(upload(p, (void**)&d.perm, perm.data(), sizeof(int32_t) * perm.size()));
  TVR_TRY(dev_alloc(p, (void**)&d.val, sizeof(float) * cap));
  TVR_CUDA(cudaMemsetAsync(d.val, 0, sizeof(float) * cap, p->stream));
  TVR_TRY(dev_alloc(p, (void**)&d.col16, sizeof(uint16_t) * cap));
  TVR_CUDA(cudaMemsetAsync(d.col16, 0, sizeof(uint16_t) * cap, p->stream));
  TVR_CUDA(launch_sell_fill(nblk * 32, d.perm, d.off, transposed ? p->rpT : p->rp, lo_off, hi_off,
                            (uint16_t)coff, transposed ? p->colT16 : p->col16,
                            transposed ? p->valT : p->val, d.col16, d.val, p->stream));
  TVR_CUDA(cudaStreamSynchronize(p->stream));  // host vectors die here
  d.nblk = nblk;
  d.h_slice_end = zend;
  ok = true;
  return TVR_OK;
}

// Sliced-ELL copy (spmv16s_kernel, TVR_SPMV_SELL): replaces the padded copy.  A slice window too
// large for shared memory is cut into P column parts of h entries (TVR_SELL_PARTS=1, default),
// each staged whole in its own pass; else its first part is staged and the rest gathered from
// global memory (HALF).  Returns TVR_OK with pl.sell unset when not applicable (no slice
// windows, too many rows, not enough device memory).
static int make_sell(tvr_problem* p, SpmvPlan& pl, bool transposed, const std::vector<int64_t>& rph,
                     int64_t rows) {
  pl.sell = false;
  if (!pl.v.idx16 || rows >= ((int64_t)1 << 31) || pl.nitems == 0) return TVR_OK;
  std::vector<int64_t> prow(pl.nitems + 1);
  std::vector<int32_t> psl(pl.nitems);
  TVR_CUDA(cudaMemcpy(prow.data(), pl.item_row, sizeof(int64_t) * (pl.nitems + 1), cudaMemcpyDeviceToHost));
  TVR_CUDA(cudaMemcpy(psl.data(), pl.item_slice, sizeof(int32_t) * pl.nitems, cudaMemcpyDeviceToHost));
  const size_t nsl = pl.h_slice_item_end.size();
  std::vector<int64_t> wlo(nsl);
  std::vector<int32_t> wlen(nsl);
  TVR_CUDA(cudaMemcpy(wlo.data(), pl.win_lo, sizeof(int64_t) * nsl, cudaMemcpyDeviceToHost));
  TVR_CUDA(cudaMemcpy(wlen.data(), pl.win_len, sizeof(int32_t) * nsl, cudaMemcpyDeviceToHost));
  SellVariant v;
  v.staged = pl.staged;
  v.block = env_int("TVR_SELL_BLOCK", 1024);  // 512: c2 A 166.9 -> 171.5 us, A^T 161.1 -> 167.1
  v.dyn = env_int("TVR_SELL_DYN", 1) != 0;
  v.unroll = env_int("TVR_SELL_UNROLL", 2);
  size_t smem = pl.staged ? pl.smem : 0;
  // column parts for windows larger than shared memory
  int P = 1, h = 0;
  if (!pl.staged && p->separable && env_int("TVR_SELL_PARTS", 1)) {
    int maxsm = 0;
    TVR_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device));
    int capf = (int)(((size_t)(maxsm - 4096) / 4) * 32 / 33) / 32 * 32;  // floats per part
    capf = std::min(capf, std::max(32, env_int("TVR_SELL_PART_FLOATS", capf)));  // tests
    if (capf > 0) {
      P = (pl.max_win + capf - 1) / capf;
      h = ((pl.max_win + P - 1) / P + 31) / 32 * 32;
    }
    if (P < 2) P = 1;
  }
  std::vector<int32_t> split_h;  // P = 2: per row, the first entry of part 1
  int32_t* split_d = nullptr;
  if (P > 1) {
    // (P - 1) split arrays, one per inner part boundary
    TVR_TRY(dev_alloc(p, (void**)&split_d, sizeof(int32_t) * (size_t)rows * (P - 1)));
    for (int q = 1; q < P; ++q)
      TVR_CUDA(launch_sell_split(rows, transposed ? p->rpT : p->rp, transposed ? p->colT16 : p->col16,
                                 q * h, split_d + (size_t)rows * (q - 1), p->stream));
    split_h.resize((size_t)rows * (P - 1));
    TVR_CUDA(cudaMemcpyAsync(split_h.data(), split_d, sizeof(int32_t) * split_h.size(),
                             cudaMemcpyDeviceToHost, p->stream));
    TVR_CUDA(cudaStreamSynchronize(p->stream));
  }
  pl.sd.assign(P, SellData());
  for (int q = 0; q < P; ++q) {
    std::vector<int64_t> lens(rows);
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t len = rph[r + 1] - rph[r];
      const int64_t e0 = q == 0 ? 0 : split_h[(size_t)rows * (q - 1) + r];
      const int64_t e1 = q == P - 1 ? len : split_h[(size_t)rows * q + r];
      lens[r] = e1 - e0;
    }
    bool ok = false;
    TVR_TRY(build_sell_data(p, pl, transposed, prow, psl, lens,
                            q == 0 ? nullptr : split_d + (size_t)rows * (q - 1),
                            q == P - 1 ? nullptr : split_d + (size_t)rows * q, q * h,
                            P > 1 ? h : 0, wlo, wlen, pl.sd[q], ok));
    if (!ok) { pl.sd.clear(); return TVR_OK; }
  }
  if (P > 1) {
    TVR_TRY(dev_alloc(p, (void**)&pl.sell_acc, sizeof(double) * std::max<int64_t>(1, rows * pl.rep)));
    v.staged = true;
    smem = sizeof(float) * ((size_t)h + (size_t)h / 32 + 1);
  } else if (!pl.staged && env_int("TVR_SPMV_HALF", 1)) {
    // a window too large for shared memory: its first part staged, the rest from global memory
    const int budget = env_int("TVR_SPMV_HALF_KB", 148) * 1024;
    const int hh = std::min<int>(pl.max_win, (int)((budget / 4) * 32 / 33) / 32 * 32);
    if (hh > 0 && pl.max_win > hh) {
      v.staged = v.half = true;
      v.unroll = env_int("TVR_SELL_HALF_UNROLL", 2);
      v.block = v.unroll == 3 ? 1024 : env_int("TVR_SELL_HALF_BLOCK", 1024);
      smem = sizeof(float) * ((size_t)hh + (size_t)hh / 32 + 1);
      pl.part_len = hh;
    }
  }
  // a staged window that fits one 512-thread CTA per SM: one 1024-thread CTA instead
  if (v.staged && !v.half && spmv16s_occupancy(v, smem) == 1 && env_int("TVR_SPMV_WIDE", 1)) {
    SellVariant w = v;
    w.block = 1024;
    if (spmv16s_occupancy(w, smem) >= 1) v = w;
  }
  const int64_t nblk = pl.sd[0].nblk;
  pl.h_slice_item_end = pl.sd[0].h_slice_end;
  // slice-shared operator: Z consecutive slices per pass (spmv16z_kernel), as many staged
  // windows as fit one 1024-thread CTA's shared memory (TVR_SLICE_Z caps Z; 1 disables)
  pl.rep_total = pl.rep;
  if (pl.rep > 1 && v.staged && !v.half && P == 1) {
    const int32_t ws = (int32_t)(((size_t)pl.max_win + pl.max_win / 32 + 1 + 3) / 4 * 4);
    int maxsm = 0;
    TVR_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device));
    const int zcap = std::min(4, std::max(1, env_int("TVR_SLICE_Z", 2)));
    for (int Z = zcap; Z >= 2; --Z) {
      const size_t sz = sizeof(float) * (size_t)ws * Z;
      if (Z > pl.rep || sz + 2048 > (size_t)maxsm) continue;
      SellVariant w = v;
      w.zgroup = Z;
      w.block = 1024;
      if (spmv16s_occupancy(w, sz) < 1) continue;
      v = w;
      smem = sz;
      pl.wstride = ws;
      pl.rep = (int32_t)((pl.rep_total + Z - 1) / Z);
      break;
    }
  }
  if (pl.rep_total > 1) {  // per slice: one past the last block of the groups ending by it
    const int Z = v.zgroup;
    for (auto& d : pl.sd) {
      d.h_slice_end.resize(pl.rep_total);
      for (int64_t z = 0; z < pl.rep_total; ++z)
        d.h_slice_end[z] = (z == pl.rep_total - 1 ? (int64_t)pl.rep : (z + 1) / Z) * d.nblk;
    }
    pl.h_slice_item_end = pl.sd[0].h_slice_end;
  }
  pl.sv = v;
  pl.smem = smem;
  pl.pad_grid = (int)std::min<int64_t>((int64_t)p->num_sms * spmv16s_occupancy(v, smem),
                                       std::max<int64_t>(1, nblk * pl.rep));
  // the CTA ranges of the full-range launch, searched once here instead of by every CTA of
  // every launch (TVR_SELL_CTA_TAB=0: off)
  const char* ct = std::getenv("TVR_SELL_CTA_TAB");
  if (!(ct && *ct == '0')) {
    for (auto& d : pl.sd) {
      const int64_t hi = d.nblk * pl.rep;
      if (hi <= 0) continue;
      const int g = (int)std::min<int64_t>(pl.pad_grid, hi);
      TVR_TRY(dev_alloc(p, (void**)&d.cta_tab, sizeof(int64_t) * (g + 1)));
      // one repetition, counter-scheduled warps: ranges of equal simulated makespan
      // (TVR_SELL_MAKESPAN=0: the work-sum split); else the kernels' own search, tabulated
      // -- where a CTA has few enough blocks for its schedule's tails to matter (c2: 290-440 per
      // CTA, A 165.5 -> 162.1 us, A^T 160.2 -> 158.6 us; c3's 1,800-3,500 per CTA: work sums, the
      // model's error there cost the A pass 1.7 %)
      const int mk = env_int("TVR_SELL_MAKESPAN", 1);
      if (pl.rep == 1 && v.dyn && mk != 0 && (int64_t)d.h_k.size() == d.nblk &&
          (mk == 2 || d.nblk < (int64_t)1024 * g)) {
        const std::vector<int64_t> tab = makespan_partition(
            d.h_k, d.h_slice, v.block / 32, g,
            (double)env_int("TVR_SELL_MK_BLKCOST", 4),  // c2 A 160.2 -> 158.9 us against 2 (6: 159.8)
            (double)env_int("TVR_SELL_SEGCOST", 3), 0.01 * env_int("TVR_SELL_MK_LAMBDA", 50));
        TVR_CUDA(cudaMemcpyAsync(d.cta_tab, tab.data(), sizeof(int64_t) * (g + 1),
                                 cudaMemcpyHostToDevice, p->stream));
        TVR_CUDA(cudaStreamSynchronize(p->stream));  // tab is a local
      } else {
        SellArgs s{};
        s.cum = d.cum;
        s.nb = d.nblk;
        s.rep = pl.rep;
        s.blk_lo = 0;
        s.blk_hi = hi;
        TVR_CUDA(launch_sell_cta_table(s, g, d.cta_tab, p->stream));
      }
      d.cta_tab_grid = g;
    }
  }
  pl.sell = true;
  return TVR_OK;
}

// Int32 sliced ELL (spmv32s_kernel, TVR_SPMV_SELL32, non-separable plans): blocks of 32
// consecutive rows; per block lane mode (padded to the longest row, one row per lane) or, with
// `modes`, row mode (rows back to back, 8 lanes per row) when its gathers change cache lines less
// often.  Replaces the padded copy.
static int make_sell32(tvr_problem* p, SpmvPlan& pl, bool transposed, const std::vector<int64_t>& rph,
                       int64_t rows, bool modes) {
  pl.sell32 = false;
  if (rows >= ((int64_t)1 << 31) || rows == 0) return TVR_OK;
  const int64_t nblk = (rows + 31) / 32;
  std::vector<uint8_t> mode(nblk, 0);
  if (modes) {
    uint8_t* md = nullptr;
    TVR_CUDA(cudaMalloc(&md, nblk));
    cudaError_t e = launch_sell32_mode(nblk, rows, transposed ? p->rpT : p->rp,
                                       transposed ? p->colT : p->col, md, p->stream,
                                       env_int("TVR_SELL32_BIAS", 40));
    if (e == cudaSuccess) e = cudaMemcpyAsync(mode.data(), md, nblk, cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    cudaFree(md);
    TVR_CUDA(e);
  }
  // Block order.  The A pass of a large non-separable volume (c5: 67 MB of x, ~100 x refetched
  // from DRAM when the grid works on rays spread over every view, profiles/r01m) stores its
  // blocks in z order of the voxels they gather (the z of each block's middle entry; rays tilted
  // by <= 10 deg span a band of ~60 slices) and the grid sweeps that order together (interleaved
  // CTA chunks), so the x sub-volume in flight stays in L2.  TVR_SELL32_ZORDER=0: row order.
  // Gather layouts (A pass with modes: c5): per block the layout of the point (row-major, x / y
  // swapped, 8x4 bricks; spmv.cu layout_index) and the walk (lane / row mode) whose gathers touch
  // the fewest 128-byte lines, counted exactly on the device (TVR_SELL32_LAYOUTS=0: row-major).
  std::vector<uint8_t> layout(nblk, 0);
  bool layouts = false;
  const int64_t Nl = p->ncol;
  const int lmask = env_int("TVR_SELL32_LAYOUTS", 7);  // bit L: layout L may be chosen
  if (!transposed && modes && (lmask & 6) != 0 && p->nx % 8 == 0 &&
      p->ny % 4 == 0 && 3 * Nl < ((int64_t)1 << 31)) {
    size_t fr = 0, tot_mem = 0;
    TVR_CUDA(cudaMemGetInfo(&fr, &tot_mem));
    const int64_t nnz_rows = rph[rows];
    const size_t scratch = sizeof(int32_t) * (size_t)nnz_rows + (size_t)nblk * (16 + 1);
    // the scratch, the two 3N layout buffers, and the sliced-ELL copy built below
    if (scratch + sizeof(float) * 6 * (size_t)Nl + (size_t)nnz_rows * 9 + ((size_t)2 << 30) < fr) {
      layouts = true;
      const double bias = env_int("TVR_SELL32_ROWBIAS", 100) / 100.0;  // row-mode overheads
      // the matrix stream too: lane mode pads every row to its block's longest (c5: +14.6 %
      // bytes, row mode +0.6 %); a stored 4-entry chunk (32 B) costs ~1.4 L1 wavefronts of time
      // at the measured HBM rate (6.5 TB/s against 148 SMs x 1 wavefront per cycle)
      const double bw = env_int("TVR_SELL32_BYTEW", 140) / 100.0;
      std::vector<int64_t> ch_lane(nblk, 0), ch_row(nblk, 0);
      for (int64_t j = 0; j < nblk; ++j) {
        int64_t K = 0, tot = 0;
        for (int64_t r = j * 32; r < std::min(rows, j * 32 + 32); ++r) {
          const int64_t c = (rph[r + 1] - rph[r] + 3) / 4;
          K = std::max(K, c);
          tot += c;
        }
        ch_lane[j] = 32 * K;
        ch_row[j] = tot;
      }
      int32_t* scol = nullptr;
      int64_t *cl = nullptr, *cr = nullptr;
      uint8_t* bad = nullptr;
      TVR_CUDA(cudaMalloc(&scol, sizeof(int32_t) * std::max<int64_t>(nnz_rows, 1)));
      TVR_CUDA(cudaMalloc(&cl, sizeof(int64_t) * nblk));
      TVR_CUDA(cudaMalloc(&cr, sizeof(int64_t) * nblk));
      TVR_CUDA(cudaMalloc(&bad, nblk));
      TVR_CUDA(cudaMemsetAsync(bad, 0, nblk, p->stream));
      std::vector<int64_t> hl(nblk), hr(nblk), best(nblk, INT64_MAX);
      std::vector<uint8_t> hbad(nblk);
      cudaError_t e = cudaSuccess;
      for (int L = 0; L < 3 && e == cudaSuccess; ++L) {
        if (L > 0 && !((lmask >> L) & 1)) continue;
        const int32_t* c = p->col;
        if (L > 0) {
          e = launch_layout_sort_rows(rows, p->rp, p->col, L, p->nx, p->ny, Nl, scol, bad, p->stream);
          c = scol;
        }
        if (e == cudaSuccess) e = launch_layout_count(nblk, rows, p->rp, c, cl, cr, p->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hl.data(), cl, sizeof(int64_t) * nblk, cudaMemcpyDeviceToHost, p->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hr.data(), cr, sizeof(int64_t) * nblk, cudaMemcpyDeviceToHost, p->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hbad.data(), bad, nblk, cudaMemcpyDeviceToHost, p->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
        if (e != cudaSuccess) break;
        for (int64_t j = 0; j < nblk; ++j) {
          if (L > 0 && hbad[j]) continue;  // a row too long to sort: row-major
          if (L == 0 && !(lmask & 1)) continue;  // row-major only as the fallback (rows > cap)
          const int64_t cost_lane = hl[j] + (int64_t)(bw * (double)ch_lane[j]);
          const int64_t cost_row = (int64_t)(bias * (double)hr[j] + bw * (double)ch_row[j]);
          const int64_t c_best = std::min(cost_lane, cost_row);
          if (c_best < best[j]) {
            best[j] = c_best;
            layout[j] = (uint8_t)L;
            mode[j] = cost_row < cost_lane ? 1 : 0;
          }
        }
      }
      cudaFree(scol);
      cudaFree(cl);
      cudaFree(cr);
      cudaFree(bad);
      TVR_CUDA(e);
    }
  }
  std::vector<int64_t> ord(nblk);
  for (int64_t j = 0; j < nblk; ++j) ord[j] = j;
  const bool zorder = !transposed && modes && env_int("TVR_SELL32_ZORDER", 1) != 0;
  if (zorder) {
    int32_t* kd = nullptr;
    std::vector<int32_t> key(nblk);
    TVR_CUDA(cudaMalloc(&kd, sizeof(int32_t) * nblk));
    cudaError_t e = launch_sell32_zkey(nblk, rows, p->rp, p->col, p->plane, kd, p->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(key.data(), kd, sizeof(int32_t) * nblk, cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    cudaFree(kd);
    TVR_CUDA(e);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  }
  std::vector<int64_t> off(nblk), cum(nblk + 1, 0), rstart((size_t)nblk * 32, 0);
  std::vector<int32_t> kk(nblk), sl(nblk, 0), perm((size_t)nblk * 32);
  int64_t chunks = 0, n_row_mode = 0;
  for (int64_t j = 0; j < nblk; ++j) {
    int64_t K = 0, tot = 0;
    for (int64_t l = 0; l < 32; ++l) {
      const int64_t r = ord[j] * 32 + l;
      perm[(size_t)j * 32 + l] = r < rows ? (int32_t)r : -1;
      const int64_t n = r < rows ? (rph[r + 1] - rph[r] + 3) / 4 : 0;
      rstart[(size_t)j * 32 + l] = tot;
      tot += n;
      K = std::max(K, n);
    }
    off[j] = chunks;
    if (mode[ord[j]]) {
      kk[j] = (int32_t)-tot;
      chunks += tot;
      cum[j + 1] = cum[j] + (tot + 31) / 32 + 2;
      ++n_row_mode;
    } else {
      kk[j] = (int32_t)K;
      chunks += K * 32;
      cum[j + 1] = cum[j] + K + 2;
    }
  }
  const size_t cap = (size_t)chunks * 4 + 8;
  const size_t need = cap * 8 + (size_t)nblk * (8 + 4 + 4 + 8 + 128 + 8 + 256);
  size_t fr = 0, tot_mem = 0;
  TVR_CUDA(cudaMemGetInfo(&fr, &tot_mem));
  if (need + ((size_t)1 << 30) > fr) return TVR_OK;  // keep 1 GB of headroom
  SellData d;
  std::vector<int64_t> zend(1, nblk), wl(1, 0);
  std::vector<int32_t> wn(1, 0);
  TVR_TRY(upload(p, (void**)&d.off, off.data(), sizeof(int64_t) * off.size()));
  TVR_TRY(upload(p, (void**)&d.k, kk.data(), sizeof(int32_t) * kk.size()));
  TVR_TRY(upload(p, (void**)&d.slice, sl.data(), sizeof(int32_t) * sl.size()));
  TVR_TRY(upload(p, (void**)&d.cum, cum.data(), sizeof(int64_t) * cum.size()));
  TVR_TRY(upload(p, (void**)&d.zend, zend.data(), sizeof(int64_t)));
  TVR_TRY(upload(p, (void**)&d.win_lo, wl.data(), sizeof(int64_t)));
  TVR_TRY(upload(p, (void**)&d.win_len, wn.data(), sizeof(int32_t)));
  TVR_TRY(upload(p, (void**)&d.row_start, rstart.data(), sizeof(int64_t) * rstart.size()));
  TVR_TRY(dev_alloc(p, (void**)&d.sq, sizeof(double) * std::max<int64_t>(1, nblk)));
  TVR_TRY(upload(p, (void**)&d.perm, perm.data(), sizeof(int32_t) * perm.size()));
  TVR_TRY(dev_alloc(p, (void**)&d.val, sizeof(float) * cap));
  TVR_CUDA(cudaMemsetAsync(d.val, 0, sizeof(float) * cap, p->stream));
  TVR_TRY(dev_alloc(p, (void**)&d.col32, sizeof(int32_t) * cap));
  TVR_CUDA(cudaMemsetAsync(d.col32, 0, sizeof(int32_t) * cap, p->stream));
  if (layouts) {
    std::vector<uint8_t> lst(nblk);
    for (int64_t j = 0; j < nblk; ++j) lst[j] = layout[ord[j]];
    uint8_t* dl = nullptr;
    TVR_CUDA(cudaMalloc(&dl, nblk));
    cudaError_t e = cudaMemcpyAsync(dl, lst.data(), nblk, cudaMemcpyHostToDevice, p->stream);
    if (e == cudaSuccess)
      e = launch_sell_fill32_layout(nblk * 32, d.perm, d.off, d.k, d.row_start, dl, p->rp, p->col,
                                    p->val, p->nx, p->ny, Nl, d.col32, d.val, p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    cudaFree(dl);
    TVR_CUDA(e);
    int64_t per[3] = {0, 0, 0};
    for (int64_t j = 0; j < nblk; ++j) ++per[lst[j]];
    pl.sell32_layout_blocks[0] = per[0];
    pl.sell32_layout_blocks[1] = per[1];
    pl.sell32_layout_blocks[2] = per[2];
    if (!p->xs) TVR_TRY(dev_alloc(p, (void**)&p->xs, sizeof(float) * 3 * Nl));
    if (!p->xs_lo) TVR_TRY(dev_alloc(p, (void**)&p->xs_lo, sizeof(float) * 3 * Nl));
  } else {
    TVR_CUDA(launch_sell_fill32(nblk * 32, d.perm, d.off, d.k, d.row_start,
                                transposed ? p->rpT : p->rp, transposed ? p->colT : p->col,
                                transposed ? p->valT : p->val, d.col32, d.val, p->stream));
  }
  TVR_CUDA(cudaStreamSynchronize(p->stream));  // host vectors die here
  pl.sell32_layouts = layouts;
  d.nblk = nblk;
  d.h_slice_end = zend;
  pl.sd.assign(1, d);
  pl.sv = SellVariant();
  // steps in flight: 3 for A^T (c5 3.85 -> 3.69 ms); for A 2 with row-ordered blocks (3: 5.21 ->
  // 5.29 ms), 3 with the z order (4.72 -> 4.50 ms: the gathers now hit L2, latency-bound)
  pl.sv.unroll = env_int("TVR_SELL32_UNROLL", transposed || zorder ? 3 : 2);
  // 1024-thread CTAs (one per SM: 32 warps share the block counter) for a gathered volume larger
  // than 32 MB (c5 A^T 3.80 -> 3.68 ms, A 4.72 -> 4.65 ms); 512 on small volumes (f2: slower)
  pl.sv.block = env_int("TVR_SELL32_BLOCK", (double)p->ncol * 4.0 > 32.0 * (1 << 20) ? 1024 : 512);
  pl.pad_grid = (int)std::min<int64_t>((int64_t)p->num_sms * spmv32s_occupancy(pl.sv.unroll, pl.sv.block),
                                       std::max<int64_t>(1, nblk));
  pl.sell32 = true;
  pl.sell32_row_blocks = n_row_mode;
  pl.sell32_zorder = zorder;
  // interleaved chunks of TVR_SELL32_ILV blocks (default 4 with the z order, else ranges)
  pl.sell32_ilv = env_int("TVR_SELL32_ILV", zorder ? 4 : 0);
  pl.sell32_l2 = env_int("TVR_SELL32_L2", 0);
  return TVR_OK;
}

// rp: host row pointer of the operator (n_rows+1); slices: n_slices+1 row boundaries when
// separable; windows: per slice gather window (lo, len); pitch padding for the A pass.
static int make_plan(tvr_problem* p, SpmvPlan& pl, const std::vector<int64_t>& rp, int64_t n_rows,
                     bool separable, const std::vector<int64_t>& slice_rows,
                     const std::vector<int64_t>& win_lo, const std::vector<int32_t>& win_len,
                     double mean_len, const char* lpr_env, bool pad) {
  pl.v.unroll = env_int("TVR_SPMV_UNROLL", 2);
  pl.v.minb = 0;  // chosen below from the shared-memory footprint
  pl.block = env_int("TVR_SPMV_BLOCK", 512);
  // Slice-structured matrices (every row inside one slice window) admit:
  //  * 16-bit column offsets inside the window: 6 instead of 8 HBM bytes per entry (any window of
  //    <= 65536 entries: c2 and c3);
  //  * staging the window in shared memory when it fits (c2 both passes, c3 A^T); a larger
  //    window (c3's 256 KB x-slice) is gathered from global memory (mostly L1 hits), or, with
  //    TVR_PART_CAP set, cut into parts staged one after another (measured slower at c3).
  // TVR_IDX16=0 uses int32 columns with whole staged windows only.
  size_t smem = 0;
  bool staged = separable && env_int("TVR_SPMV_STAGE", 1) != 0;
  pl.parts = 1;
  pl.part_len = 0;
  int32_t maxlen = 0;
  for (int32_t l : win_len) maxlen = std::max(maxlen, l);
  pl.max_win = maxlen;
  const bool want16 = separable && maxlen <= 65536 && env_int("TVR_IDX16", 1) != 0;
  if (staged) {
    int32_t wlen = maxlen;
    const int32_t cap = want16 ? std::min(65536, std::max(1024, env_int("TVR_PART_CAP", 65536))) : maxlen;
    if (want16 && maxlen > cap) {
      pl.parts = (maxlen + cap - 1) / cap;
      pl.part_len = ((maxlen + pl.parts - 1) / pl.parts + 31) / 32 * 32;
      wlen = pl.part_len;
    } else if (want16) {
      pl.part_len = (maxlen + 31) / 32 * 32;
    }
    smem = sizeof(float) * ((size_t)wlen + ((size_t)wlen >> 5) + 1);  // swz(c) = c + c/32
    int maxsmem = 0;
    cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
    // leave room for the reduction scratch of the kernel
    if (smem + 2048 > (size_t)maxsmem) {
      staged = false;
      pl.parts = 1;
    }
  }
  if (want16 && !staged) pl.part_len = (maxlen + 31) / 32 * 32;
  (void)pad;
  pl.staged = staged;
  pl.v.staged = staged;
  pl.smem = staged ? smem : 0;
  pl.v.idx16 = want16;
  pl.v.parts = want16 && staged && pl.parts > 1;
  pl.v.lpr = env_int(lpr_env, lpr_for(mean_len, pl.v.idx16 ? 8 : 4));
  // Resident CTAs per SM: as many 512-thread CTAs as fit while leaving >= 80 KB of the 228 KB
  // L1/smem for L1 (the in-flight 128-bit streaming loads are staged in L1; with ~25 KB left the
  // A pass at c2 loses half its bandwidth, measured).  The 16-bit kernel spills at the 40
  // registers of 3 CTAs and is faster with 2 (scripts/sweep_spmv.py).
  {
    int minb = 1;
    for (int m = pl.v.idx16 ? 2 : 3; m >= 1; --m)
      if ((double)m * (pl.smem + 1024) <= (228.0 - 80.0) * 1024) { minb = m; break; }
    pl.v.minb = env_int("TVR_SPMV_MINB", minb);
  }
  // 3 chunks in flight for the staged 16-bit kernel at 2 CTAs/SM (1-3% faster than 2 at c2)
  if (pl.v.idx16 && staged && !pl.v.parts && pl.v.minb == 2) pl.v.unroll = env_int("TVR_SPMV_UNROLL", 3);
  if (!spmv_variant_exists(pl.v)) {
    set_error("no SpMV kernel variant for lpr=" + std::to_string(pl.v.lpr));
    return TVR_E_ARG;
  }

  // occupancy-sized persistent grid: exactly one wave of resident CTAs
  const int occ = spmv_occupancy(pl.v, pl.block, pl.smem);
  pl.grid = p->num_sms * occ;

  const int64_t nnz = rp[n_rows];
  std::vector<int64_t> rows;
  std::vector<int32_t> slices;
  const int64_t target = std::max<int64_t>(2048, nnz / ((int64_t)pl.grid * 16) + 1);
  if (separable) {
    for (size_t z = 0; z + 1 < slice_rows.size(); ++z)
      split_rows(rp.data(), slice_rows[z], slice_rows[z + 1], target, (int32_t)z, rows, slices);
  } else {
    split_rows(rp.data(), 0, n_rows, target, 0, rows, slices);
  }
  rows.push_back(n_rows);
  pl.nitems = (int64_t)slices.size();
  if (pl.grid > pl.nitems) pl.grid = (int)std::max<int64_t>(1, pl.nitems);
  TVR_TRY(upload(p, (void**)&pl.item_row, rows.data(), sizeof(int64_t) * rows.size()));
  TVR_TRY(upload(p, (void**)&pl.item_slice, slices.data(), sizeof(int32_t) * std::max<size_t>(1, slices.size())));
  if (separable) {
    TVR_TRY(upload(p, (void**)&pl.win_lo, win_lo.data(), sizeof(int64_t) * win_lo.size()));
    TVR_TRY(upload(p, (void**)&pl.win_len, win_len.data(), sizeof(int32_t) * win_len.size()));
    std::vector<int64_t> zend(win_lo.size(), 0);
    for (size_t i = 0; i < slices.size(); ++i) zend[slices[i]] = (int64_t)i + 1;
    for (size_t z = 1; z < zend.size(); ++z) zend[z] = std::max(zend[z], zend[z - 1]);
    TVR_TRY(upload(p, (void**)&pl.slice_item_end, zend.data(), sizeof(int64_t) * std::max<size_t>(1, zend.size())));
    pl.h_slice_item_end = zend;
  }

  return TVR_OK;
}

}  // namespace tvr

using namespace tvr;

// ===================================================================== C ABI
extern "C" {

const char* tvr_last_error(void) { return g_err.c_str(); }
int tvr_abi_version(void) { return TVR_ABI_VERSION; }

int tvr_set_allocator(tvr_alloc_fn a, tvr_free_fn f, void* ctx) {
  if ((a == nullptr) != (f == nullptr)) {
    set_error("tvr_set_allocator: alloc and free must both be set or both NULL");
    return TVR_E_ARG;
  }
  g_alloc = a;
  g_free = f;
  g_alloc_ctx = ctx;
  return TVR_OK;
}

void tvr_gpbb_default(tvr_gpbb_opts* o) {
  if (!o) return;
  o->max_iters = 10000;
  o->eps = 1e-6;
  o->stop_mode = TVR_STOP_REL;
  o->K = 2;
  o->sigma = 0.1;
  o->beta0 = 0.95;
  o->beta_min = 1e-10;
}

void tvr_gp_default(tvr_gp_opts* o) {
  if (!o) return;
  o->max_iters = 10000;
  o->eps = 1e-6;
  o->stop_mode = TVR_STOP_REL;
  o->L0 = 1.0;
  o->rho_L = 1.3;
  o->bt_max = 200;
}

void tvr_upn_default(tvr_upn_opts* o) {
  if (!o) return;
  o->max_iters = 10000;
  o->eps = 1e-6;
  o->stop_mode = TVR_STOP_REL;
  o->L0 = 1.0;
  o->mu0 = 1.0;
  o->rho_L = 1.3;
  o->bt_max = 200;
}

// sliced: A is one slice's matrix (n_cols = nx*ny) applied to every slice (tvr_create_sliced).
static int create_impl(tvr_problem* p, const tvr_csr* A, const float* b_host, tvr_grid grid,
                       double alpha, double tau, double lo, double hi, const tvr_dist* dist,
                       bool sliced) {
  if (!A || !b_host) { set_error("tvr_create: NULL argument"); return TVR_E_ARG; }
  if (grid.nx <= 0 || grid.ny <= 0 || grid.nz <= 0) { set_error("tvr_create: bad grid"); return TVR_E_ARG; }
  if (!(tau > 0.0) || !std::isfinite(tau)) { set_error("tvr_create: tau must be > 0"); return TVR_E_ARG; }
  if (!(alpha >= 0.0) || !std::isfinite(alpha)) { set_error("tvr_create: alpha must be >= 0"); return TVR_E_ARG; }
  if (!(lo < hi) || std::isnan(lo) || std::isnan(hi)) { set_error("tvr_create: need lo < hi"); return TVR_E_ARG; }
  p->nx = grid.nx; p->ny = grid.ny; p->nz = grid.nz;
  p->plane = (int64_t)grid.nx * grid.ny;
  const int64_t Nglob = sliced ? p->plane : p->plane * grid.nz;  // column range of the given A
  if (A->n_cols != Nglob) {
    set_error(sliced ? "tvr_create_sliced: A_slice.n_cols != nx*ny" : "tvr_create: A.n_cols != nx*ny*nz");
    return TVR_E_ARG;
  }
  if (A->n_rows < 0 || A->nnz < 0 || (A->nnz > 0 && (!A->col_idx || !A->val)) || !A->row_ptr) {
    set_error("tvr_create: bad CSR sizes/pointers");
    return TVR_E_ARG;
  }
  p->alpha = alpha; p->tau = tau; p->lo = lo; p->hi = hi;
  p->z0 = 0; p->z1 = grid.nz; p->device = -1;
  cudaStream_t user_stream = nullptr;
  if (dist) {
    p->world = dist->world < 1 ? 1 : dist->world;
    p->rank = dist->rank;
    p->mode = dist->mode;
    p->comm = dist->nccl_comm;
    p->device = dist->device;
    user_stream = (cudaStream_t)dist->cuda_stream;
    if (p->mode == TVR_SHARD_ZSLAB || p->mode == TVR_SHARD_VIEWS || p->mode == TVR_SHARD_VIEWS_REP) {
      p->z0 = dist->z0; p->z1 = dist->z1;
      if (p->z0 < 0 || p->z1 > grid.nz || p->z0 >= p->z1) { set_error("tvr_create: bad slab"); return TVR_E_ARG; }
    } else if (p->mode != TVR_SHARD_NONE) {
      set_error("tvr_create: unknown shard mode");
      return TVR_E_ARG;
    }
    if (p->rank < 0 || p->rank >= p->world) { set_error("tvr_create: bad rank"); return TVR_E_ARG; }
    if (p->world > 1 && (p->mode == TVR_SHARD_NONE || !valid_comm(p->comm))) {
      set_error("tvr_create: world > 1 needs ZSLAB or VIEWS mode and a communicator "
                "(tvr_nccl_comm_init or tvr_local_comm_create)");
      return TVR_E_ARG;
    }
    if (p->world == 1 && p->comm && !valid_comm(p->comm)) {
      set_error("tvr_create: nccl_comm is not a libtvreg communicator handle");
      return TVR_E_ARG;
    }
    if (p->world == 1 && (p->z0 != 0 || p->z1 != grid.nz)) {
      // one rank owns every slice: no neighbour would fill the halo planes of a partial slab
      set_error("tvr_create: a single rank (world == 1) must own every slice (z0 = 0, z1 = nz)");
      return TVR_E_ARG;
    }
  }
  p->nzl = p->z1 - p->z0;
  const bool views = p->mode == TVR_SHARD_VIEWS || p->mode == TVR_SHARD_VIEWS_REP;
  if (sliced && views) {
    set_error("tvr_create_sliced: VIEWS mode is not supported (use ZSLAB)");
    return TVR_E_ARG;
  }
  p->sliced = sliced;
  p->zA0 = views ? 0 : p->z0;
  p->nzA = views ? grid.nz : p->nzl;

  // ---- validate the CSR (host) ----
  // m, nnz: rows and entries of the matrix stored on the device (the slice matrix when sliced);
  // m_full: rows of the operator (and of b, r)
  const int64_t m = A->n_rows, nnz = A->nnz;
  const int64_t m_full = sliced ? m * p->nzA : m;
  const int64_t* rp = A->row_ptr;
  if (rp[0] != 0 || rp[m] != nnz) { set_error("CSR: row_ptr[0] != 0 or row_ptr[m] != nnz"); return TVR_E_CSR; }
  const int64_t colmin = sliced ? 0 : p->zA0 * p->plane;
  const int64_t colmax = sliced ? p->plane : (p->zA0 + p->nzA) * p->plane;
  p->separable = true;
  std::vector<int32_t> row_slice(m, -1);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t s = rp[i], e = rp[i + 1];
    if (e < s) { set_error("CSR: row_ptr not non-decreasing at row " + std::to_string(i)); return TVR_E_CSR; }
    for (int64_t k = s; k < e; ++k) {
      const int32_t c = A->col_idx[k];
      if (c < 0 || c >= Nglob) { set_error("CSR: column out of range in row " + std::to_string(i)); return TVR_E_CSR; }
      if (k > s && c <= A->col_idx[k - 1]) { set_error("CSR: columns not strictly ascending in row " + std::to_string(i)); return TVR_E_CSR; }
      if (!std::isfinite(A->val[k])) { set_error("CSR: non-finite value in row " + std::to_string(i)); return TVR_E_CSR; }
    }
    if (e > s) {
      const int64_t cf = A->col_idx[s], cl = A->col_idx[e - 1];
      if (cf < colmin || cl >= colmax) {
        set_error("row " + std::to_string(i) + " touches voxels outside the slab");
        return TVR_E_NOT_SEPARABLE;
      }
      const int64_t zf = (cf - colmin) / p->plane, zl = (cl - colmin) / p->plane;
      if (zf != zl) p->separable = false;
      row_slice[i] = (int32_t)zf;
    }
  }
  for (int64_t i = 0; i < m_full; ++i)
    if (!std::isfinite(b_host[i])) { set_error("b: non-finite entry"); return TVR_E_ARG; }
  // slice-major row order: assign empty rows to the slice of the previous non-empty row
  if (p->separable) {
    int32_t cur = 0;
    for (int64_t i = 0; i < m; ++i) {
      if (row_slice[i] < 0) row_slice[i] = cur;
      if (row_slice[i] < cur) { p->separable = false; break; }
      cur = row_slice[i];
    }
  }
  if (p->separable && !sliced) {
    p->slice_row.assign(p->nzA + 1, m);
    p->slice_row[0] = 0;
    int64_t i = 0;
    for (int z = 1; z <= p->nzA; ++z) {
      while (i < m && row_slice[i] < z) ++i;
      p->slice_row[z] = i;
    }
  }
  if (sliced) {  // every row is inside the one stored slice; operator rows are z m_s + i
    p->slice_row.resize(p->nzA + 1);
    for (int z = 0; z <= p->nzA; ++z) p->slice_row[z] = (int64_t)z * m;
    p->m_s = m;
    p->nnz_s = nnz;
  }

  p->m = m_full;
  p->n = p->plane * p->nzl;
  p->ncol = p->plane * p->nzA;
  p->nnz = sliced ? nnz * p->nzA : nnz;  // entries of the operator
  const int64_t n = sliced ? p->plane : p->ncol;  // rows of the stored A^T

  // ---- device and stream (everything above is host-only validation) ----
  if (p->device < 0) TVR_CUDA(cudaGetDevice(&p->device));
  TVR_CUDA(cudaSetDevice(p->device));
  TVR_CUDA(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device));
  TVR_CUDA(cudaDeviceGetAttribute(&p->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device));
  if (user_stream) {
    p->stream = user_stream;
  } else {
    // a BLOCKING stream: it orders after work on the legacy default stream (torch's default
    // stream producing x_dev, e.g. torch.zeros), so inputs are complete before the passes read them
    TVR_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamDefault));
    p->own_stream = true;
  }
  // every rank's slab bounds (the slabs must tile [0, nz) in rank order); collective
  if (p->world > 1) TVR_TRY(slab_table(p));

  // ---- device copies (columns made slab-local) ----
  // Padding: 16-byte chunk loads of whole 16-byte units may read up to 3
  // entries past the end of col/val/b and 2 past row_ptr (the pads are zero, never used).
  const size_t nnz_pad = (size_t)((nnz + 7) / 8 * 8 + 8);  // 8-entry chunks of the 16-bit kernel
  TVR_TRY(dev_alloc(p, (void**)&p->rp, sizeof(int64_t) * (m + 3)));
  TVR_CUDA(cudaMemsetAsync(p->rp, 0, sizeof(int64_t) * (m + 3), p->stream));
  TVR_CUDA(cudaMemcpyAsync(p->rp, rp, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, p->stream));
  TVR_TRY(dev_alloc(p, (void**)&p->col, sizeof(int32_t) * nnz_pad));
  TVR_TRY(dev_alloc(p, (void**)&p->val, sizeof(float) * nnz_pad));
  TVR_CUDA(cudaMemsetAsync(p->col, 0, sizeof(int32_t) * nnz_pad, p->stream));
  TVR_CUDA(cudaMemsetAsync(p->val, 0, sizeof(float) * nnz_pad, p->stream));
  if (colmin == 0) {
    TVR_CUDA(cudaMemcpyAsync(p->col, A->col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, p->stream));
  } else {
    std::vector<int32_t> loc(A->col_idx, A->col_idx + nnz);
    for (auto& c : loc) c -= (int32_t)colmin;
    TVR_CUDA(cudaMemcpyAsync(p->col, loc.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, p->stream));
    TVR_CUDA(cudaStreamSynchronize(p->stream));
  }
  TVR_CUDA(cudaMemcpyAsync(p->val, A->val, sizeof(float) * nnz, cudaMemcpyHostToDevice, p->stream));
  TVR_TRY(dev_alloc(p, (void**)&p->b, sizeof(float) * (m_full + 4)));
  TVR_CUDA(cudaMemsetAsync(p->b, 0, sizeof(float) * (m_full + 4), p->stream));
  TVR_CUDA(cudaMemcpyAsync(p->b, b_host, sizeof(float) * m_full, cudaMemcpyHostToDevice, p->stream));

  // ---- transposed CSR on the device ----
  TVR_TRY(dev_alloc(p, (void**)&p->rpT, sizeof(int64_t) * (n + 3)));
  TVR_CUDA(cudaMemsetAsync(p->rpT, 0, sizeof(int64_t) * (n + 3), p->stream));
  TVR_TRY(dev_alloc(p, (void**)&p->colT, sizeof(int32_t) * nnz_pad));
  TVR_TRY(dev_alloc(p, (void**)&p->valT, sizeof(float) * nnz_pad));
  TVR_CUDA(cudaMemsetAsync(p->colT, 0, sizeof(int32_t) * nnz_pad, p->stream));
  TVR_CUDA(cudaMemsetAsync(p->valT, 0, sizeof(float) * nnz_pad, p->stream));
  {
    void *cnt = nullptr, *sc = nullptr, *sv = nullptr, *sb = nullptr;
    const int64_t nb = (n + 1 + 1023) / 1024;
    TVR_CUDA(cudaMalloc(&cnt, sizeof(int32_t) * std::max<int64_t>(n, 1)));
    TVR_CUDA(cudaMalloc(&sc, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    TVR_CUDA(cudaMalloc(&sv, sizeof(float) * std::max<int64_t>(nnz, 1)));
    TVR_CUDA(cudaMalloc(&sb, sizeof(int64_t) * (nb + 2)));
    cudaError_t e = build_transpose(m, n, nnz, p->rp, p->col, p->val, p->rpT, p->colT, p->valT,
                                    (int32_t*)cnt, (int32_t*)sc, (float*)sv, (int64_t*)sb, p->stream);
    cudaError_t e2 = cudaStreamSynchronize(p->stream);
    cudaFree(cnt); cudaFree(sc); cudaFree(sv); cudaFree(sb);
    if (e != cudaSuccess || e2 != cudaSuccess) {
      set_error(std::string("transpose build: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
      return TVR_E_CUDA;
    }
  }

  // ---- SpMV plans ----
  {
    std::vector<int64_t> rpv(rp, rp + m + 1);
    std::vector<int64_t> wlo, sr;
    std::vector<int32_t> wlen;
    const int nsl = sliced ? 1 : p->nzA;  // slices of the stored matrix
    const std::vector<int64_t> srA = sliced ? std::vector<int64_t>{0, m} : p->slice_row;
    if (p->separable) {
      for (int z = 0; z < nsl; ++z) { wlo.push_back((int64_t)z * p->plane); wlen.push_back((int32_t)p->plane); }
    }
    const double mean_A = m > 0 ? (double)nnz / m : 0.0;
    TVR_TRY(make_plan(p, p->planA, rpv, m, p->separable, srA, wlo, wlen,
                      mean_A, "TVR_LPR_A", true));
    // A^T: rows are voxels; slice z owns voxel rows [z plane, (z+1) plane) and gathers r over
    // the slice's A rows.
    std::vector<int64_t> rpT(n + 1);
    TVR_CUDA(cudaMemcpyAsync(rpT.data(), p->rpT, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, p->stream));
    TVR_CUDA(cudaStreamSynchronize(p->stream));
    wlo.clear(); wlen.clear();
    if (p->separable) {
      for (int z = 0; z <= nsl; ++z) sr.push_back((int64_t)z * p->plane);
      for (int z = 0; z < nsl; ++z) {
        wlo.push_back(srA[z]);
        wlen.push_back((int32_t)(srA[z + 1] - srA[z]));
      }
    }
    const double mean_len = n > 0 ? (double)nnz / n : 0.0;
    TVR_TRY(make_plan(p, p->planT, rpT, n, p->separable, sr, wlo, wlen,
                      mean_len, "TVR_LPR_AT", false));
  }
  // ---- 16-bit column offsets for the staged plans ----
  p->nnz_pad = nnz_pad;
  for (int which = 0; which < 2; ++which) {
    SpmvPlan& pl = which ? p->planT : p->planA;
    if (!pl.v.idx16) continue;
    uint16_t** dst = which ? &p->colT16 : &p->col16;
    TVR_TRY(dev_alloc(p, (void**)dst, sizeof(uint16_t) * nnz_pad));
    TVR_CUDA(cudaMemsetAsync(*dst, 0, sizeof(uint16_t) * nnz_pad, p->stream));
    pl.nrows = which ? n : m;
    if (pl.parts > 1) {
      TVR_TRY(dev_alloc(p, (void**)&pl.part_off, sizeof(uint16_t) * (pl.parts - 1) * pl.nrows));
      TVR_TRY(dev_alloc(p, (void**)&pl.part_acc, sizeof(double) * pl.nrows));
    }
    SpmvArgs a = spmv_args(p, pl, which == 1, nullptr, nullptr, nullptr, nullptr);
    TVR_CUDA(launch_parts_rows(a, false, which ? p->colT : p->col, *dst, pl.part_off, nullptr,
                               p->stream));
  }
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  if (sliced) {  // the sliced-ELL blocks of the one stored slice repeat over the slab's slices
    if (!p->planA.v.idx16 || !p->planT.v.idx16 || p->planA.v.parts || p->planT.v.parts) {
      set_error("tvr_create_sliced: needs 16-bit slice windows (nx*ny and m_s <= 65536)");
      return TVR_E_ARG;
    }
    p->planA.rep = p->planT.rep = p->nzA;
    p->planA.rep_rows = m;          // A pass: slice z writes rows z m_s + i, gathers x's slice z
    p->planA.rep_win = p->plane;
    p->planT.rep_rows = p->plane;   // A^T pass: writes voxels of slice z, gathers r's rows of z
    p->planT.rep_win = m;
  }
  // ---- padded-row copies (TVR_SPMV_PAD=0 disables): 16-bit plans pad rows to 8 entries,
  // int32 global-gather plans to 4; skipped when the copy would not fit in free device memory
  for (int which = 0; which < 2; ++which) {
    SpmvPlan& pl = which ? p->planT : p->planA;
    const bool p16 = pl.v.idx16, p32 = !pl.v.idx16 && !pl.staged;
    if (!(p16 || p32) || pl.v.parts || !env_int("TVR_SPMV_PAD", 1)) continue;
    const int q = p16 ? 8 : 4;  // chunk entries
    const int64_t rows = which ? n : m;
    std::vector<int64_t> rph(rows + 1), rpp(rows + 1);
    TVR_CUDA(cudaMemcpyAsync(rph.data(), which ? p->rpT : p->rp, sizeof(int64_t) * (rows + 1),
                             cudaMemcpyDeviceToHost, p->stream));
    TVR_CUDA(cudaStreamSynchronize(p->stream));
    // int32 sliced ELL for the A^T pass (voxel rows: a block's lanes gather neighbouring ray ids,
    // c5 A^T 5.62 -> 3.69 ms); the A pass keeps the per-row kernel (parallel rays in one block
    // gather unrelated lines: c5 A 6.20 -> 6.99 ms), TVR_SPMV_SELL32 = 0 none / 1 A^T / 2 both
    // TVR_SPMV_SELL32 = 3: the A pass too, with per-block lane / row modes (default when the
    // gathered volume is larger than 32 MB, so that its gathers miss L1 / L2: c5 A 6.18 -> 5.21
    // ms; on f2's 1 MB volume the per-row kernel stays ahead, 91 vs 95 us)
    const int s32 = env_int("TVR_SPMV_SELL32", (double)p->ncol * 4.0 > 32.0 * (1 << 20) ? 3 : 1);
    if (p32 && (s32 >= 2 || (s32 == 1 && which == 1))) {
      TVR_TRY(make_sell32(p, pl, which == 1, rph, rows, which == 0 && s32 == 3));
      if (pl.sell32) continue;
    }
    if (p16 && p->separable && (env_int("TVR_SPMV_SELL", 1) || sliced)) {
      TVR_TRY(make_sell(p, pl, which == 1, rph, rows));
      if (pl.sell) continue;
      if (sliced) {
        set_error("tvr_create_sliced: sliced-ELL copy not built (device memory)");
        return TVR_E_OOM;
      }
    }
    rpp[0] = 0;
    for (int64_t r = 0; r < rows; ++r) rpp[r + 1] = rpp[r] + (rph[r + 1] - rph[r] + q - 1) / q * q;
    const size_t cap = (size_t)rpp[rows] + (size_t)q * 32 * 4 + 8;  // slack: chunks read past the last row
    const size_t need = cap * (p16 ? 6 : 8) + sizeof(int64_t) * (rows + 1);
    size_t fr = 0, tot = 0;
    TVR_CUDA(cudaMemGetInfo(&fr, &tot));
    if (need + ((size_t)1 << 30) > fr) continue;  // keep 1 GB of headroom
    TVR_TRY(upload(p, (void**)&pl.rpp, rpp.data(), sizeof(int64_t) * (rows + 1)));
    TVR_TRY(dev_alloc(p, (void**)&pl.valp, sizeof(float) * cap));
    TVR_CUDA(cudaMemsetAsync(pl.valp, 0, sizeof(float) * cap, p->stream));
    if (p16) {
      TVR_TRY(dev_alloc(p, (void**)&pl.col16p, sizeof(uint16_t) * cap));
      TVR_CUDA(cudaMemsetAsync(pl.col16p, 0, sizeof(uint16_t) * cap, p->stream));
      TVR_CUDA(launch_pad_rows(rows, which ? p->rpT : p->rp, pl.rpp, which ? p->colT16 : p->col16,
                               which ? p->valT : p->val, pl.col16p, pl.valp, p->stream));
      // a window too large for shared memory: stage its first part (leaving >= 80 KB of L1 for
      // the streaming loads and the rest of the gathers), one 1024-thread CTA per SM
      if (!pl.staged && env_int("TVR_SPMV_HALF", 1)) {
        const int32_t maxlen = pl.max_win;
        const int budget = env_int("TVR_SPMV_HALF_KB", 148) * 1024;
        const int h = std::min<int>(maxlen, (int)((budget / 4) * 32 / 33) / 32 * 32);
        SpmvVariant w = pl.v;
        w.half = true;
        w.unroll = 2;
        const size_t sm = sizeof(float) * ((size_t)h + (size_t)h / 32 + 1);
        if (h > 0 && maxlen > h && p->separable && (w.lpr == 4 || w.lpr == 8 || w.lpr == 16) &&
            spmv16p_occupancy(w, 1024, sm) >= 1) {
          pl.v = w;
          pl.block = 1024;
          pl.smem = sm;
          pl.part_len = h;
        }
      }
      // a staged window that fits one 512-thread CTA per SM only: one 1024-thread CTA instead
      if (pl.staged && pl.block == 512 && spmv16p_occupancy(pl.v, 512, pl.smem) == 1 &&
          env_int("TVR_SPMV_WIDE", 1)) {
        SpmvVariant w = pl.v;
        w.unroll = 2;
        if (spmv16p_occupancy(w, 1024, pl.smem) >= 1 && (w.lpr == 4 || w.lpr == 8 || w.lpr == 16)) {
          pl.v = w;
          pl.block = 1024;
        }
      }
      pl.pad_grid = std::min<int64_t>((int64_t)p->num_sms * spmv16p_occupancy(pl.v, pl.block, pl.smem),
                                      std::max<int64_t>(1, pl.nitems));
    } else {
      TVR_TRY(dev_alloc(p, (void**)&pl.col32p, sizeof(int32_t) * cap));
      TVR_CUDA(cudaMemsetAsync(pl.col32p, 0, sizeof(int32_t) * cap, p->stream));
      TVR_CUDA(launch_pad_rows32(rows, which ? p->rpT : p->rp, pl.rpp, which ? p->colT : p->col,
                                 which ? p->valT : p->val, pl.col32p, pl.valp, p->stream));
      pl.pad_grid = std::min<int64_t>((int64_t)p->num_sms * spmv32p_occupancy(pl.v, pl.block),
                                      std::max<int64_t>(1, pl.nitems));
    }
    TVR_CUDA(cudaStreamSynchronize(p->stream));
    pl.pad = true;
  }
  // the int32 columns are no longer read by any pass: release them (c3: 7.7 GB each)
  if (p->planA.v.idx16) { dev_free(p, p->col); p->col = nullptr; }
  if (p->planT.v.idx16) { dev_free(p, p->colT); p->colT = nullptr; }

  // extended-precision evaluation of the UPN / GP iterates (A (x + x_lo)): the
  // sliced-ELL A-pass kernels have the lo gathers; one rank or z-slabs (VIEWS would all-gather
  // the lo parts too); TVR_EXT_EVAL=0 evaluates at the hi parts
  p->ext_eval = !views_dist(p) && !sliced && env_int("TVR_EXT_EVAL", 1) != 0 &&
                (p->planA.sell32 || (p->planA.sell && spmv16s_lo_ok(p->planA.sv)));

  // ---- work vectors ----
  const int NVOL = 13, NDAT = 4;  // 10-12: lo parts of the extended-precision solver iterates
  // slab + one halo plane per side; VIEWS_REP: the whole volume, the slab at its z0 offset
  const bool rep = rep_dist(p);
  const size_t volbytes = sizeof(float) * (size_t)(p->plane * (rep ? p->nz : p->nzl + 2));
  for (int i = 0; i < NVOL; ++i) {
    float* q = nullptr;
    TVR_TRY(dev_alloc(p, (void**)&q, volbytes));
    TVR_CUDA(cudaMemsetAsync(q, 0, volbytes, p->stream));
    p->vol.push_back(q + (rep ? (int64_t)p->z0 * p->plane : p->plane));
    if (rep) p->vol_base.push_back(q);
  }
  for (int i = 0; i < NDAT; ++i) {
    float* q = nullptr;
    TVR_TRY(dev_alloc(p, (void**)&q, sizeof(float) * std::max<int64_t>(m_full, 1)));
    p->dat.push_back(q);
  }
  if (p->world > 1) TVR_TRY(dev_alloc(p, (void**)&p->xhalo, sizeof(float) * 2 * p->plane));
  if (views_dist(p)) {
    TVR_TRY(dev_alloc(p, (void**)&p->xfull, sizeof(float) * p->ncol));
    TVR_TRY(dev_alloc(p, (void**)&p->wfull, sizeof(float) * p->ncol));
    // fused reduce-scatter: needs the padded int32 A^T kernel and peer-mapped inboxes
    if (env_int("TVR_FUSED_RS", 1) && (p->planT.pad || p->planT.sell32) && !p->planT.v.idx16)
      TVR_TRY(setup_fused_rs(p));
  }
  tv_set_grid(p->num_sms);
  const int64_t maxgrid = std::max<int64_t>({(int64_t)p->planA.grid, (int64_t)p->planT.grid,
                                             (int64_t)tv_num_blocks(p->nx, p->ny, p->nzl),
                                             (int64_t)p->num_sms * 8});
  p->partials_cap = maxgrid * 8;  // kMaxScalars (common.cuh)
  TVR_TRY(dev_alloc(p, (void**)&p->partials, sizeof(double) * p->partials_cap));
  TVR_TRY(dev_alloc(p, (void**)&p->counter, 64));
  TVR_CUDA(cudaMemsetAsync(p->counter, 0, 64, p->stream));
  TVR_TRY(dev_alloc(p, (void**)&p->dscal, sizeof(double) * 64));
  TVR_CUDA(cudaMemsetAsync(p->dscal, 0, sizeof(double) * 64, p->stream));
  TVR_CUDA(cudaMallocHost((void**)&p->hscal, sizeof(double) * 64 * (std::max(1, p->world) + 1)));
  if (p->world > 1 || p->comm) {
    TVR_TRY(dev_alloc(p, (void**)&p->dgather, sizeof(double) * 64 * p->world));
    TVR_TRY(dev_alloc(p, (void**)&p->dsum, sizeof(double) * 64));
  }
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  return TVR_OK;
}

void tvr_destroy(tvr_problem* p) {
  if (!p) return;
  if (p->stream) {
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
  }
  dist_release(p);
  dev_free_all(p);
  if (p->e2e_exec) cudaGraphExecDestroy(p->e2e_exec);
  for (auto e : p->pipe_ev) cudaEventDestroy(e);
  if (p->s_in) cudaStreamDestroy(p->s_in);
  if (p->s_out) cudaStreamDestroy(p->s_out);
  if (p->s_a) cudaStreamDestroy(p->s_a);
  for (auto& t : p->pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  for (auto e : p->event_pool) cudaEventDestroy(e);
  if (p->hscal) cudaFreeHost(p->hscal);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

int tvr_create(tvr_problem** out, const tvr_csr* A, const float* b_host, tvr_grid grid,
               double alpha, double tau, double lo, double hi, const tvr_dist* dist) {
  if (!out) { set_error("tvr_create: out is NULL"); return TVR_E_ARG; }
  *out = nullptr;
  tvr_problem* p = new (std::nothrow) tvr_problem();
  if (!p) { set_error("host allocation failed"); return TVR_E_OOM; }
  int s;
  try {
    s = create_impl(p, A, b_host, grid, alpha, tau, lo, hi, dist, false);
  } catch (const std::exception& ex) {
    set_error(std::string("tvr_create: ") + ex.what());
    s = TVR_E_OOM;
  }
  if (s != TVR_OK) {
    tvr_destroy(p);
    return s;
  }
  *out = p;
  return TVR_OK;
}

int tvr_create_sliced(tvr_problem** out, const tvr_csr* A_slice, const float* b_host,
                      tvr_grid grid, double alpha, double tau, double lo, double hi,
                      const tvr_dist* dist) {
  if (!out) { set_error("tvr_create_sliced: out is NULL"); return TVR_E_ARG; }
  *out = nullptr;
  tvr_problem* p = new (std::nothrow) tvr_problem();
  if (!p) { set_error("host allocation failed"); return TVR_E_OOM; }
  int s;
  try {
    s = create_impl(p, A_slice, b_host, grid, alpha, tau, lo, hi, dist, true);
  } catch (const std::exception& ex) {
    set_error(std::string("tvr_create_sliced: ") + ex.what());
    s = TVR_E_OOM;
  }
  if (s != TVR_OK) {
    tvr_destroy(p);
    return s;
  }
  *out = p;
  return TVR_OK;
}

int tvr_sell_partition(const int32_t* blk_steps, const int32_t* blk_slice, int64_t nblk, int nwarps,
                       int grid, double blk_cost, double seg_cost, double lambda, int64_t* tab_out) {
  if (!blk_steps || !blk_slice || !tab_out || nblk < 0 || nwarps < 1 || grid < 1 ||
      !(lambda >= 0.0 && lambda <= 1.0) || !(blk_cost >= 0.0) || !(seg_cost >= 0.0)) {
    set_error("tvr_sell_partition: bad arguments");
    return TVR_E_ARG;
  }
  const std::vector<int32_t> k(blk_steps, blk_steps + nblk), sl(blk_slice, blk_slice + nblk);
  const std::vector<int64_t> tab = makespan_partition(k, sl, nwarps, grid, blk_cost, seg_cost, lambda);
  std::copy(tab.begin(), tab.end(), tab_out);
  return TVR_OK;
}

int tvr_get_info(const tvr_problem* p, tvr_info* info) {
  if (!p || !info) { set_error("tvr_get_info: NULL"); return TVR_E_ARG; }
  info->m_local = p->m;
  info->n_local = p->n;
  info->nnz_local = p->nnz;
  info->z0 = p->z0;
  info->z1 = p->z1;
  info->slab_staged_A = p->planA.staged ? 1 : 0;
  info->slab_staged_AT = p->planT.staged ? 1 : 0;
  info->device_bytes = p->device_bytes;
  info->n_cols_local = p->ncol;
  info->views_fused_rs = p->fused_rs ? 1 : 0;
  info->views_rep = rep_dist(p) ? 1 : 0;
  info->point_allgathers = p->n_gathers;
  info->dist_graph_solves = p->n_dist_graph;
  info->dist_graph_exchanges = p->n_dist_exch;
  for (int i = 0; i < 3; ++i) info->gather_layout_blocks[i] = p->planA.sell32_layout_blocks[i];
  info->slice_shared = p->sliced ? p->nzA : 0;
  return TVR_OK;
}

// Volume input from a caller pointer: in slab mode copied into an internal buffer whose halo
// planes are then exchanged; on one GPU used in place.
// A caller's volume vector at world > 1: its boundary planes go to the neighbours and theirs land
// in p->xhalo (planes -1 and nzl), so the stencil reads the caller's slab in place.
static int exchange_caller_halo(tvr_problem* p, const float* x_dev) {
  if (p->world == 1) return TVR_OK;
  return halo_exchange_to(p, x_dev, p->xhalo, p->xhalo + p->plane);
}

// alpha grad TV(x) (+ w) on a caller's x after exchange_caller_halo (a4)
static int pass_tv_caller(tvr_problem* p, const float* x, const float* w, float* g, double alpha) {
  if (p->world == 1)
    return pass_tv_grad(p, x, nullptr, 0.0, w, nullptr, 0.0, g, nullptr, nullptr, nullptr, 0.0, 1,
                        alpha, nullptr);
  TVArgs a = tv_args(p, 1);
  a.alpha = alpha;
  a.w1 = w;
  a.g_out = g;
  const double bytes = (double)n_local(p) * (4.0 + (w ? 4.0 : 0.0) + (g ? 4.0 : 0.0));
  return launch(p, K_TV_GRAD, bytes, [&] {
    return launch_tv_grad_plain_h(a, x, p->xhalo, p->xhalo + p->plane, p->stream);
  });
}

static int objective_grad_impl(tvr_problem* p, const float* x_dev, double* f_out, float* g_dev,
                               tvr_fparts* parts) {
  const float* x = x_dev;
  TVR_TRY(exchange_caller_halo(p, x));
  float* r = datvec(p, 0);
  TVR_TRY(pass_residual(p, x, r, 0));
  float* w = nullptr;
  if (g_dev) {
    w = volvec(p, 8);
    TVR_TRY(pass_AT(p, r, w));
  }
  TVR_TRY(pass_tv_caller(p, x, w, g_dev, p->alpha));
  TVR_TRY(fetch_scalars(p, 8));
  const double fid = 0.5 * p->hscal[0], tv = p->hscal[1];
  const double f = fid + p->alpha * tv;
  if (f_out) *f_out = f;
  if (parts) { parts->fidelity = fid; parts->tv = tv; parts->f = f; }
  if (!std::isfinite(f)) { set_error("non-finite objective"); return TVR_E_NONFINITE; }
  return TVR_OK;
}

int tvr_objective_grad(tvr_problem* p, const float* x_dev, double* f_out, float* g_dev,
                       tvr_fparts* parts) {
  NvtxRange nv("tvr_objective_grad");
  if (!p || !x_dev) { set_error("tvr_objective_grad: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  return objective_grad_impl(p, x_dev, f_out, g_dev, parts);
}

static bool pinned(const void* ptr) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// End-to-end gradient with the transfers overlapped (one GPU, slice-separable A, per-row SpMV
// kernels, pinned host buffers): the volume is cut into C slab chunks; chunk c's x goes up on a
// copy stream while the previous chunks compute, its A pass (rows of its slices), A^T pass (its
// voxels) and stencil (its planes; needs the first plane of chunk c+1) run as soon as their
// inputs are there, and its g goes down on a second copy stream.  Per-element results are the
// unchunked passes' (same kernels, same rows); the fidelity and TV sums are added per chunk in
// chunk order (equal to the single-launch sums to rounding).
static int objective_grad_host_pipelined(tvr_problem* p, const float* xh, double* f_out, float* gh,
                                         tvr_fparts* parts, int C) {
  const int nz = p->nzl;
  const int64_t plane = p->plane;
  float* x = volvec(p, 7);
  float* g = volvec(p, 6);
  float* w = volvec(p, 8);
  float* r = datvec(p, 0);
  if (!p->s_in) {
    TVR_CUDA(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
    TVR_CUDA(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
    TVR_CUDA(cudaStreamCreateWithFlags(&p->s_a, cudaStreamNonBlocking));
    p->pipe_ev.resize(3 * 16 + 2);
    for (auto& e : p->pipe_ev) TVR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TVR_TRY(dev_alloc(p, (void**)&p->partials2, sizeof(double) * p->partials_cap));
    TVR_TRY(dev_alloc(p, (void**)&p->counter2, 64));
    TVR_CUDA(cudaMemsetAsync(p->counter2, 0, 64, p->stream));
  }
  // TVR_E2E_ASTREAM=1: the A passes run on their own stream (with their own reduction scratch),
  // so chunk c+1's A pass can start while chunk c's A^T pass and stencil finish
  const bool astream = env_int("TVR_E2E_ASTREAM", 1) != 0;
  auto ev_a = [&](int c) { return p->pipe_ev[2 + 32 + c]; };
  cudaEvent_t ev_start = p->pipe_ev[0], ev_done = p->pipe_ev[1];
  auto ev_in = [&](int c) { return p->pipe_ev[2 + c]; };
  auto ev_g = [&](int c) { return p->pipe_ev[2 + 16 + c]; };
  std::vector<int> z(C + 1);
  // tapered chunks: the first chunk's upload and the last chunk's download are the exposed
  // transfers, so the end chunks get half the weight of the middle ones (TVR_E2E_TAPER=0: equal)
  {
    const bool taper = env_int("TVR_E2E_TAPER", 1) != 0 && C > 2;
    const double tw = taper ? std::min(1.0, std::max(0.05, env_int("TVR_E2E_TAPER_PCT", 60) / 100.0)) : 1.0;
    const double total = C - 2.0 + 2.0 * tw;
    double acc = 0.0;
    z[0] = 0;
    for (int c = 0; c < C; ++c) {
      acc += (c == 0 || c == C - 1) ? tw : 1.0;
      z[c + 1] = std::max(z[c] + 1, (int)std::lround(nz * acc / total));
    }
    z[C] = nz;
  }
  // slice-shared operator in groups of Z slices: chunk boundaries on group boundaries (a group's
  // pass reads all its slices' inputs and writes all its rows)
  {
    auto grp = [](const SpmvPlan& pl) { return pl.sell ? pl.sv.zgroup : 1; };
    const int ga = grp(p->planA), gt = grp(p->planT);
    const int G = ga / std::gcd(ga, gt) * gt;
    if (G > 1) {
      std::vector<int> za(1, 0);
      for (int c = 1; c < C; ++c) {
        const int zr = (int)std::lround((double)z[c] / G) * G;
        if (zr > za.back() && zr < nz) za.push_back(zr);
      }
      za.push_back(nz);
      z = za;
      C = (int)za.size() - 1;
    }
  }
  constexpr int SA = 16, ST = 24;  // scalar slots: A chunk c at SA + c, stencil chunk c at ST + 6 c
  // TVR_E2E_TRACE=1: timing events at every stage, printed to stderr (diagnostics)
  const bool trace = env_int("TVR_E2E_TRACE", 0) != 0;
  std::vector<std::pair<std::string, cudaEvent_t>> tr;
  auto mark = [&](const std::string& name, cudaStream_t st) -> int {
    if (!trace) return TVR_OK;
    cudaEvent_t e;
    TVR_CUDA(cudaEventCreate(&e));
    TVR_CUDA(cudaEventRecord(e, st));
    tr.emplace_back(name, e);
    return TVR_OK;
  };
  // The whole pipeline (copies, events, passes on three streams) as one enqueue; replayed as a
  // CUDA graph while the host buffers and chunking stay the same (TVR_E2E_GRAPH=0: eager)
  auto enqueue = [&]() -> int {
    TVR_TRY(mark("start", p->stream));
    TVR_CUDA(cudaEventRecord(ev_start, p->stream));
    TVR_CUDA(cudaStreamWaitEvent(p->s_in, ev_start, 0));
    TVR_CUDA(cudaStreamWaitEvent(p->s_out, ev_start, 0));
    // TVR_E2E_UPFRONT=1: x goes up whole before any pass (an H2D copy running under the SpMV
    // passes slows them by ~25 %, measured; D2H copies do not), only the downloads overlap
    const bool upfront = env_int("TVR_E2E_UPFRONT", 0) != 0;
    for (int c = 0; c < C; ++c) {
      const size_t off = (size_t)z[c] * plane, cnt = (size_t)(z[c + 1] - z[c]) * plane;
      if (!upfront || c == 0)
        TVR_CUDA(cudaMemcpyAsync(x + off, xh + off, sizeof(float) * (upfront ? (size_t)nz * plane : cnt),
                                 cudaMemcpyHostToDevice, p->s_in));
      TVR_CUDA(cudaEventRecord(ev_in(c), p->s_in));
      TVR_TRY(mark("in" + std::to_string(c), p->s_in));
    }
    const double bytes_row = entry_bytes(p->planA) * (double)p->nnz / nz;  // per slice, for counters
    for (int c = 0; c < C; ++c) {
      if (astream) {
        TVR_CUDA(cudaStreamWaitEvent(p->s_a, ev_in(c), 0));
        // run the A pass on s_a with the second reduction scratch
        std::swap(p->stream, p->s_a);
        std::swap(p->partials, p->partials2);
        std::swap(p->counter, p->counter2);
        const int st = launch(p, K_SPMV_A, bytes_row * (z[c + 1] - z[c]), [&] {
          return run_spmv(p, p->planA, false, x, p->b, r, nullptr, p->dscal + SA + c, z[c], z[c + 1]);
        });
        std::swap(p->stream, p->s_a);
        std::swap(p->partials, p->partials2);
        std::swap(p->counter, p->counter2);
        TVR_TRY(st);
        TVR_CUDA(cudaEventRecord(ev_a(c), p->s_a));
        TVR_CUDA(cudaStreamWaitEvent(p->stream, ev_a(c), 0));
      } else {
        TVR_CUDA(cudaStreamWaitEvent(p->stream, ev_in(c), 0));
        TVR_TRY(mark("A" + std::to_string(c) + ">", p->stream));
        TVR_TRY(launch(p, K_SPMV_A, bytes_row * (z[c + 1] - z[c]), [&] {
          return run_spmv(p, p->planA, false, x, p->b, r, nullptr, p->dscal + SA + c, z[c], z[c + 1]);
        }));
        TVR_TRY(mark("A" + std::to_string(c) + "<", p->stream));
      }
      if (gh) {
        TVR_TRY(launch(p, K_SPMV_AT, bytes_row * (z[c + 1] - z[c]), [&] {
          return run_spmv(p, p->planT, true, r, nullptr, w, nullptr, nullptr, z[c], z[c + 1]);
        }));
        TVR_TRY(mark("AT" + std::to_string(c) + "<", p->stream));
      }
      if (c + 1 < C) TVR_CUDA(cudaStreamWaitEvent(p->stream, ev_in(c + 1), 0));  // plane z[c+1]
      TVArgs a = tv_args(p, ST + 6 * c);
      const int64_t off = (int64_t)z[c] * plane;
      a.zg0 = p->z0 + z[c];
      a.nzl = z[c + 1] - z[c];
      a.w1 = gh ? w + off : nullptr;
      a.g_out = gh ? g + off : nullptr;
      const double N = (double)a.nzl * plane;
      TVR_TRY(mark("TV" + std::to_string(c) + ">", p->stream));
      TVR_TRY(launch(p, K_TV_GRAD, N * (gh ? 12.0 : 8.0),
                     [&] { return launch_tv_grad_plain(a, x + off, p->stream); }));
      TVR_TRY(mark("TV" + std::to_string(c) + "<", p->stream));
      if (gh) {
        TVR_CUDA(cudaEventRecord(ev_g(c), p->stream));
        TVR_CUDA(cudaStreamWaitEvent(p->s_out, ev_g(c), 0));
        TVR_CUDA(cudaMemcpyAsync(gh + off, g + off, sizeof(float) * N, cudaMemcpyDeviceToHost, p->s_out));
        TVR_TRY(mark("out" + std::to_string(c), p->s_out));
      }
    }
    TVR_CUDA(cudaEventRecord(ev_done, p->s_out));
    TVR_CUDA(cudaStreamWaitEvent(p->stream, ev_done, 0));
    TVR_CUDA(cudaMemcpyAsync(p->hscal, p->dscal, sizeof(double) * 64, cudaMemcpyDeviceToHost, p->stream));
    TVR_TRY(mark("end", p->stream));
    return TVR_OK;
  };
  const bool graph = !trace && !p->prof && env_int("TVR_E2E_GRAPH", 1) != 0;
  if (graph) {
    if (!p->e2e_exec || p->e2e_xh != xh || p->e2e_gh != gh || p->e2e_z != z) {
      if (p->e2e_exec) { cudaGraphExecDestroy(p->e2e_exec); p->e2e_exec = nullptr; }
      const int64_t l0 = p->launches;
      const double b0 = p->bytes_total;
      TVR_CUDA(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeRelaxed));
      const int st = enqueue();
      cudaGraph_t gr = nullptr;
      const cudaError_t e = cudaStreamEndCapture(p->stream, &gr);
      p->e2e_launches = p->launches - l0;
      p->e2e_bytes = p->bytes_total - b0;
      p->launches = l0;
      p->bytes_total = b0;
      if (st < 0) { if (gr) cudaGraphDestroy(gr); return st; }
      TVR_CUDA(e);
      const cudaError_t ei = cudaGraphInstantiate(&p->e2e_exec, gr, 0);
      cudaGraphDestroy(gr);
      TVR_CUDA(ei);
      p->e2e_xh = xh;
      p->e2e_gh = gh;
      p->e2e_z = z;
    }
    TVR_CUDA(cudaGraphLaunch(p->e2e_exec, p->stream));
    p->launches += p->e2e_launches;
    p->bytes_total += p->e2e_bytes;
  } else {
    TVR_TRY(enqueue());
  }
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  if (trace) {
    std::string line = "e2e trace (us):";
    for (auto& t : tr) {
      float ms = 0.f;
      const cudaError_t e = cudaEventElapsedTime(&ms, tr[0].second, t.second);
      line += " " + t.first + "=" +
              (e == cudaSuccess ? std::to_string((int)std::lround(ms * 1e3)) : cudaGetErrorString(e));
    }
    for (auto& t : tr) cudaEventDestroy(t.second);
    std::fprintf(stderr, "%s\n", line.c_str());
  }
  resolve_pending_timings(p);
  double rsq = 0.0, tv = 0.0;
  for (int c = 0; c < C; ++c) {
    rsq += p->hscal[SA + c];
    tv += p->hscal[ST + 6 * c];
  }
  const double fid = 0.5 * rsq, f = fid + p->alpha * tv;
  if (f_out) *f_out = f;
  if (parts) { parts->fidelity = fid; parts->tv = tv; parts->f = f; }
  if (!std::isfinite(f)) { set_error("non-finite objective"); return TVR_E_NONFINITE; }
  return TVR_OK;
}

int tvr_objective_grad_host(tvr_problem* p, const float* x_host, double* f_out, float* g_host,
                            tvr_fparts* parts) {
  NvtxRange nv("tvr_objective_grad_host");
  if (!p || !x_host) { set_error("tvr_objective_grad_host: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  const int C = std::min(env_int("TVR_E2E_CHUNKS", 3), std::min(6, p->nzl));  // 6: dscal slots
  if (C > 1 && p->world == 1 && p->separable && !p->planA.v.parts && !p->planT.v.parts &&
      pinned(x_host) && (!g_host || pinned(g_host)))
    return objective_grad_host_pipelined(p, x_host, f_out, g_host, parts, C);
  float* x = volvec(p, 7);
  float* g = volvec(p, 6);
  TVR_CUDA(cudaMemcpyAsync(x, x_host, sizeof(float) * p->n, cudaMemcpyHostToDevice, p->stream));
  TVR_TRY(objective_grad_impl(p, x, f_out, g_host ? g : nullptr, parts));
  if (g_host) {
    TVR_CUDA(cudaMemcpyAsync(g_host, g, sizeof(float) * p->n, cudaMemcpyDeviceToHost, p->stream));
    TVR_CUDA(cudaStreamSynchronize(p->stream));
  }
  return TVR_OK;
}

int tvr_residual(tvr_problem* p, const float* x_dev, float* r_dev, double* fid) {
  if (!p || !x_dev || !r_dev) { set_error("tvr_residual: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  TVR_TRY(pass_residual(p, x_dev, r_dev, 0));
  TVR_TRY(fetch_scalars(p, 1));
  if (fid) *fid = 0.5 * p->hscal[0];
  return TVR_OK;
}

int tvr_apply_A(tvr_problem* p, const float* x_dev, float* y_dev) {
  if (!p || !x_dev || !y_dev) { set_error("tvr_apply_A: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  NvtxRange nv("tvr_apply_A");
  const float* src = x_dev;
  TVR_TRY(gather_volume(p, x_dev, &src));
  const double bytes = entry_bytes(p->planA) * (p->sliced ? (double)p->nnz_s : (double)p->nnz) +
                       8.0 * ((p->sliced ? (double)p->m_s : (double)p->m) + 1) + 4.0 * p->ncol +
                       4.0 * p->m;
  TVR_TRY(launch(p, K_SPMV_A, bytes, [&] {
    return run_spmv(p, p->planA, false, src, nullptr, y_dev, nullptr, nullptr);
  }));
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  return TVR_OK;
}

int tvr_apply_AT(tvr_problem* p, const float* y_dev, float* w_dev) {
  if (!p || !y_dev || !w_dev) { set_error("tvr_apply_AT: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  TVR_TRY(pass_AT(p, y_dev, w_dev));
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  return TVR_OK;
}

int tvr_tv(tvr_problem* p, const float* x_dev, double* tv_out, float* grad_dev) {
  if (!p || !x_dev) { set_error("tvr_tv: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  TVR_TRY(exchange_caller_halo(p, x_dev));
  TVR_TRY(pass_tv_caller(p, x_dev, nullptr, grad_dev, 1.0));
  TVR_TRY(fetch_scalars(p, 8));
  if (tv_out) *tv_out = p->hscal[1];
  return TVR_OK;
}

int tvr_gradient_map(tvr_problem* p, const float* x_dev, double nu, double* norm_out, float* G_dev) {
  if (!p || !x_dev || !(nu > 0.0)) { set_error("tvr_gradient_map: bad argument"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  float* g = volvec(p, 5);
  double f;
  TVR_TRY(objective_grad_impl(p, x_dev, &f, g, nullptr));
  TVR_TRY(pass_gmap(p, x_dev, g, nu, G_dev, 0));
  TVR_TRY(fetch_scalars(p, 1));
  if (norm_out) *norm_out = std::sqrt(p->hscal[0]);
  return TVR_OK;
}

int tvr_get_AT(tvr_problem* p, int64_t* rp_h, int32_t* col_h, float* val_h) {
  if (!p) { set_error("tvr_get_AT: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaSetDevice(p->device));
  // the stored transpose: of the slice matrix for a slice-shared problem
  const int64_t rows = p->sliced ? p->plane : p->ncol, nnz = p->sliced ? p->nnz_s : p->nnz;
  if (rp_h) TVR_CUDA(cudaMemcpyAsync(rp_h, p->rpT, sizeof(int64_t) * (rows + 1), cudaMemcpyDeviceToHost, p->stream));
  if (col_h && p->colT16) {
    // the device holds 16-bit window offsets: expand them back to the canonical int32 columns
    int32_t* tmp = nullptr;
    TVR_CUDA(cudaMalloc(&tmp, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    SpmvArgs a = spmv_args(p, p->planT, true, nullptr, nullptr, nullptr, nullptr);
    cudaError_t e = launch_parts_rows(a, true, nullptr, p->colT16, p->planT.part_off, tmp, p->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(col_h, tmp, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    cudaFree(tmp);
    if (e != cudaSuccess) { set_error(std::string("tvr_get_AT: ") + cudaGetErrorString(e)); return TVR_E_CUDA; }
  } else if (col_h) {
    TVR_CUDA(cudaMemcpyAsync(col_h, p->colT, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, p->stream));
  }
  if (val_h) TVR_CUDA(cudaMemcpyAsync(val_h, p->valT, sizeof(float) * nnz, cudaMemcpyDeviceToHost, p->stream));
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  return TVR_OK;
}

int tvr_profile_enable(tvr_problem* p, int on) {
  if (!p) { set_error("tvr_profile_enable: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  resolve_timings(p);
  for (int k = 0; k < K_COUNT; ++k) { p->kt_ms[k] = 0; p->kt_bytes[k] = 0; p->kt_launches[k] = 0; }
  p->prof = on != 0;
  return TVR_OK;
}

int tvr_profile_get(tvr_problem* p, tvr_kernel_stat* out, int cap, int* n_out) {
  if (!p) { set_error("tvr_profile_get: NULL"); return TVR_E_ARG; }
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  resolve_timings(p);
  int n = 0;
  for (int k = 0; k < K_COUNT && n < cap; ++k) {
    if (!out) break;
    std::memset(&out[n], 0, sizeof(tvr_kernel_stat));
    std::strncpy(out[n].name, kKernelNames[k], sizeof(out[n].name) - 1);
    out[n].launches = p->kt_launches[k];
    out[n].total_ms = p->kt_ms[k];
    out[n].bytes = p->kt_bytes[k];
    ++n;
  }
  if (n_out) *n_out = n;
  return TVR_OK;
}

int tvr_set_control(tvr_problem* p, int mode) {
  if (!p || (mode != TVR_CONTROL_HOST && mode != TVR_CONTROL_DEVICE && mode != TVR_CONTROL_AUTO)) {
    set_error("tvr_set_control: bad argument");
    return TVR_E_ARG;
  }
  p->control = mode;
  return TVR_OK;
}

int64_t tvr_launch_count(const tvr_problem* p, int reset) {
  if (!p) return -1;
  const int64_t n = p->launches;
  if (reset) const_cast<tvr_problem*>(p)->launches = 0;
  return n;
}

}  // extern "C"
