// Internal state of a libtvreg problem and the host-side pass functions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/libtvreg.h"
#include "kernels.h"

namespace tvr {

// NVTX range (SURVEY §5 tracing): every pass, exchange and solver phase is a named range on the
// host timeline (header-only NVTX v3; a no-op unless a tool such as nsys / ncu is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
#define TVR_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::tvr::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));            \
      return TVR_E_CUDA;                                                               \
    }                                                                                  \
  } while (0)
#define TVR_TRY(call)            \
  do {                           \
    int _s = (call);             \
    if (_s < 0) return _s;       \
  } while (0)

// Kernel ids for per-kernel timing.
enum KernelId {
  K_SPMV_A = 0,   // a1: r = A v - b (+ sum r^2)
  K_SPMV_AT,      // a2: w = A^T r
  K_TV_GRAD,      // a4: g = w + alpha grad TV (+ BB / stop reductions)
  K_TV_TRIAL,     // a5: v = P_Q(x - s g), TV(v) (+ Armijo / BT / mu reductions)
  K_MOMENTUM,     // a6: sum ((1+beta) r1 - beta r0)^2
  K_PROJECT,
  K_GMAP,
  K_COUNT
};
extern const char* kKernelNames[K_COUNT];

struct SellData {
  int64_t nblk = 0;
  int64_t* off = nullptr;
  int32_t* k = nullptr;
  int32_t* slice = nullptr;
  int64_t* zend = nullptr;
  double* sq = nullptr;
  int64_t* cum = nullptr;
  int32_t* perm = nullptr;
  uint16_t* col16 = nullptr;
  int32_t* col32 = nullptr;    // spmv32s (int32 global columns)
  int64_t* row_start = nullptr;  // spmv32s row-mode blocks: per slot, row start in chunks
  float* val = nullptr;
  int64_t* win_lo = nullptr;   // the plan's windows, shifted to the part
  int32_t* win_len = nullptr;
  int64_t* cta_tab = nullptr;  // CTA ranges of the full-range launch (SellArgs::cta_tab)
  int32_t cta_tab_grid = 0;
  std::vector<int32_t> h_k, h_slice;  // host copies: chunk steps and slice of every block
  std::vector<int64_t> h_slice_end;  // per slice: one past its last block
};

struct SpmvPlan {
  // padded-row copy for spmv16p_kernel (rows on 8-entry boundaries, zero pads)
  bool pad = false;
  int pad_grid = 0;
  int32_t max_win = 0;  // largest slice window (entries)
  // sliced-ELL copy (spmv16s_kernel; replaces the padded copy when built): col16p / valp hold it
  bool sell = false;
  bool sell32 = false;                 // int32 sliced ELL (spmv32s_kernel): sd[0], no windows
  int64_t sell32_row_blocks = 0;       // of its blocks, those in row mode
  int32_t sell32_ilv = 0;              // interleaved CTA chunks of this many blocks (0: ranges)
  bool sell32_zorder = false;          // blocks stored in z order of the voxels they gather
  int32_t sell32_l2 = 0;               // spmv32s L2 policies (SellArgs::l2hint)
  bool sell32_layouts = false;         // columns index the point's gather layouts (p->xs)
  int64_t sell32_layout_blocks[3] = {0, 0, 0};  // blocks per layout (row-major, yx, bricks)
  int32_t rep = 1;                     // slice-shared operator: the blocks repeat per slice
  int64_t rep_rows = 0, rep_win = 0;   // per repetition: output row / gather window offsets
  int64_t rep_total = 0;               // slice groups (sv.zgroup > 1): slices; rep = groups
  int32_t wstride = 0;                 // slice groups: floats between the staged windows
  SellVariant sv;
  std::vector<SellData> sd;            // one structure, or one per column part (sell_parts)
  double* sell_acc = nullptr;          // column parts: per-row fp64 partial sums between parts
  int64_t* rpp = nullptr;
  uint16_t* col16p = nullptr;  // 16-bit plans
  int32_t* col32p = nullptr;   // int32 global-gather plans
  float* valp = nullptr;
  int parts = 1, part_len = 0;       // slice-window parts (16-bit kernel)
  uint16_t* part_off = nullptr;      // (parts-1) x nrows
  double* part_acc = nullptr;        // nrows
  int64_t nrows = 0;
  bool staged = false;
  SpmvVariant v;
  int grid = 0, block = 512;
  size_t smem = 0;
  int64_t nitems = 0;
  int64_t* item_row = nullptr;
  int32_t* item_slice = nullptr;
  int64_t* slice_item_end = nullptr;
  std::vector<int64_t> h_slice_item_end;  // host copy (slice-chunked launches of the e2e pipeline)
  int64_t* win_lo = nullptr;
  int32_t* win_len = nullptr;
};

struct PendingTiming {
  int kid;
  cudaEvent_t a, b;
  double bytes;
};

}  // namespace tvr

struct tvr_problem {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nx = 0, ny = 0, nz = 0, z0 = 0, z1 = 0, nzl = 0;
  int64_t plane = 0, m = 0, n = 0, nnz = 0;
  // columns of the local A (= rows of its A^T) and the slices they span: the slab (n, z0, nzl)
  // in NONE / ZSLAB mode, the whole volume (N, 0, nz) in VIEWS mode
  int64_t ncol = 0;
  int zA0 = 0, nzA = 0;
  double alpha = 0, tau = 0, lo = 0, hi = 0;
  int world = 1, rank = 0, mode = TVR_SHARD_NONE;
  int control = TVR_CONTROL_AUTO;  // solver control (tvr_set_control)
  void* comm = nullptr;
  int num_sms = 148;

  // system matrix (device, local indices) and data
  int64_t* rp = nullptr;
  int32_t* col = nullptr;
  float* val = nullptr;
  int64_t* rpT = nullptr;
  int32_t* colT = nullptr;
  float* valT = nullptr;
  uint16_t* col16 = nullptr;   // 16-bit window offsets (planA.v.idx16)
  uint16_t* colT16 = nullptr;  // (planT.v.idx16)
  size_t nnz_pad = 0;
  float* b = nullptr;
  bool separable = false;
  // slice-shared operator (tvr_create_sliced): the device holds one slice's
  // matrix (m_s rows over the nx*ny voxels of a slice) and its transpose, applied to every slice
  int64_t m_s = 0, nnz_s = 0;
  bool sliced = false;
  std::vector<int64_t> slice_row;  // nzl+1 local row boundaries per slice (separable only)
  tvr::SpmvPlan planA, planT;

  // work vectors: volume vectors carry one halo plane on each side (vol_base + plane)
  std::vector<float*> vol;  // pointers to local plane 0
  std::vector<float*> dat;  // m-vectors

  // reductions
  double* partials = nullptr;
  int64_t partials_cap = 0;
  unsigned* counter = nullptr;
  double* dscal = nullptr;  // 32 doubles
  double* hscal = nullptr;  // pinned mirror

  // world > 1: the halo planes (-1, nzl) of a caller's vector (tvr_objective_grad / tvr_tv read the
  // caller's slab in place; its neighbours' planes land here)
  float* xhalo = nullptr;
  std::vector<float*> vol_base;
  float* xs = nullptr;     // the A pass's point in its three gather layouts (3 ncol floats)
  float* xs_lo = nullptr;  // ... and its lo parts (extended-precision evaluation)
  int64_t n_gathers = 0;  // all-gathers of a point (gather_volume), tvr_info.point_allgathers  // VIEWS_REP: allocation base of each replicated volume vector
  // VIEWS mode with world > 1: full-volume gather target of the A pass and full-volume partial
  // A_p^T r_p before the reduce-scatter; per-rank slab offsets / sizes (elements)
  float* xfull = nullptr;
  float* wfull = nullptr;
  std::vector<int64_t> slab_off, slab_cnt, peer_nzl;  // every rank's slab (world > 1)
  // fused reduce-scatter of the VIEWS A^T pass: this rank's inbox (world slots of inbox_stride
  // floats), per-owner store targets (device array) and the owners' row bounds
  bool fused_rs = false;
  float* inbox = nullptr;
  bool inbox_raw = false;  // NCCL backend: inbox from cudaMalloc (IPC-mappable), freed by dist_release
  bool ext_eval = false;   // UPN / GP iterates can be evaluated at hi + lo (A pass lo gathers)
  bool ext_on = false;     // ... and are, from this point of the current solve on
  int max_smem_optin = 0;  // cudaDevAttrMaxSharedMemoryPerBlockOptin of the device
  int64_t inbox_stride = 0;
  float** out_peer_dev = nullptr;
  int64_t* out_bounds_dev = nullptr;
  std::vector<void*> ipc_opened;  // peer inboxes mapped with cudaIpcOpenMemHandle
  int* barrier_dev = nullptr;

  // e2e pipeline of tvr_objective_grad_host (created on first use)
  cudaStream_t s_in = nullptr, s_out = nullptr, s_a = nullptr;
  double* partials2 = nullptr;   // second reduction scratch (the pipeline's A stream)
  unsigned* counter2 = nullptr;
  // host-buffer pipeline as a CUDA graph, for these host buffers and chunk boundaries
  cudaGraphExec_t e2e_exec = nullptr;
  const float* e2e_xh = nullptr;
  const float* e2e_gh = nullptr;
  std::vector<int> e2e_z;
  int64_t e2e_launches = 0;
  double e2e_bytes = 0.0;
  std::vector<cudaEvent_t> pipe_ev;

  // profiling
  bool prof = false;
  std::vector<tvr::PendingTiming> pending;
  std::vector<cudaEvent_t> event_pool;
  double kt_ms[tvr::K_COUNT] = {0};
  double kt_bytes[tvr::K_COUNT] = {0};
  int64_t kt_launches[tvr::K_COUNT] = {0};
  int64_t launches = 0;
  double bytes_total = 0;  // algorithmic bytes of every pass launched
  double* dgather = nullptr;  // world x 64 scalars (dist)
  double* dsum = nullptr;     // 64 scalars: rank-ordered sums taken on the device (solver graphs)
  int64_t n_dist_graph = 0, n_dist_exch = 0;  // tvr_info.dist_graph_solves / _exchanges

  std::vector<void*> allocs;
  int64_t device_bytes = 0;
};

namespace tvr {

int dev_alloc(tvr_problem* p, void** ptr, size_t bytes);
void dev_free(tvr_problem* p, void* ptr);
float* volvec(tvr_problem* p, int i);
void vol_extent(const tvr_problem* p, float* v, float** first, int64_t* count);
float* datvec(tvr_problem* p, int i);
int64_t n_local(const tvr_problem* p);

// pass functions (enqueue only; scalars land in p->dscal[slot..])
int pass_residual(tvr_problem* p, const float* x, float* r, int slot,          // a1
                  float* r_lo = nullptr, const float* x_lo = nullptr);  // x_lo: A (x + x_lo)
int pass_AT(tvr_problem* p, const float* r, float* w);                          // a2
int pass_tv_grad(tvr_problem* p, const float* x, const float* x0, double beta,  // a4
                 const float* w1, const float* w0, double wbeta, float* g, float* v_out,
                 const float* xp, const float* gp, double stop_step, int slot);
int pass_tv_grad(tvr_problem* p, const float* x, const float* x0, double beta, const float* w1,
                 const float* w0, double wbeta, float* g, float* v_out, const float* xp,
                 const float* gp, double stop_step, int slot, double alpha,
                 const double* dparam = nullptr);  // dparam: device-side (beta, stop_step, wbeta)
int pass_tv_trial(tvr_problem* p, const float* x, const float* g, double s, float* v,  // a5
                  double stop_step, const float* xo, int slot,
                  const double* dparam = nullptr);  // dparam: device-side (s, stop_step)
// extended-precision iterates (hi + lo pairs, tv.cu SrcTrialX / SrcMomentumX): the trial from the
// base state (x, x_lo) writes the state (v, v_lo) and evaluates at v; xo / xo_lo the mu_k
// reference (nullable)
int pass_tv_trial_x(tvr_problem* p, const float* x, const float* x_lo, const float* g, double s,
                    float* v, float* v_lo, const float* xo, const float* xo_lo, int slot,
                    const double* dparam = nullptr);
// gradient w1 + alpha grad TV and the stop reduction at the extended-precision iterate x + x_lo
int pass_tv_grad_x(tvr_problem* p, const float* x, const float* x_lo, const float* w1, float* g,
                   double stop_step, int slot, const double* dparam = nullptr);
// UPN point from (x1, x1_lo), (x0, x0_lo): gradient (w blend) at x1 + beta (x1 - x0) of the hi
// parts, state y = (y, y_lo) from the full pairs
int pass_tv_momentum_x(tvr_problem* p, const float* x1, const float* x1_lo, const float* x0,
                       const float* x0_lo, double beta, const float* w1, const float* w0,
                       float* g, float* y, float* y_lo, int slot, const double* dparam = nullptr);
int pass_momentum(tvr_problem* p, const float* r1, const float* r1lo, const float* r0,  // a6
                  const float* r0lo, double beta, int slot, const double* dbeta = nullptr);
int pass_project(tvr_problem* p, float* x);
int pass_gmap(tvr_problem* p, const float* x, const float* g, double nu, float* G, int slot);

// synchronise the stream, fetch nslots scalars into p->hscal and (dist) sum them over ranks
int fetch_scalars(tvr_problem* p, int nslots);
// halo planes of a volume vector from the z-neighbours (no-op on one GPU)
int halo_exchange(tvr_problem* p, float* v);
// the same exchange for a vector without halo room: v's boundary planes go to the neighbours,
// theirs land in lo (plane -1) and hi (plane nzl)
int halo_exchange_to(tvr_problem* p, const float* v, float* lo, float* hi);
// recompute the halo planes of a trial / momentum point from its inputs' halo planes
// (dparam: the step / beta read on the device from dparam[0], as the stencil's device-control variants)
int halo_fill_trial(tvr_problem* p, const float* x, const float* g, double s, float* v,
                    const double* dparam = nullptr);
int halo_fill_momentum(tvr_problem* p, const float* x1, const float* x0, double beta, float* y,
                       const double* dparam = nullptr);
int halo_fill_trial_x(tvr_problem* p, const float* x, const float* x_lo, const float* g, double s,
                      float* v, float* v_lo, const double* dparam = nullptr);
int halo_fill_momentum_x(tvr_problem* p, const float* x1, const float* x1_lo, const float* x0,
                         const float* x0_lo, double beta, float* y, float* y_lo,
                         const double* dparam = nullptr);
// NCCL communicator (not the in-process thread backend): its collectives are stream work only
bool nccl_backend(const tvr_problem* p);
// halo planes of v (nullable) + scalar all-gather + rank-ordered sum ON THE DEVICE into p->dsum;
// enqueue only (capturable)
int dist_scalars_dev(tvr_problem* p, float* v, int nslots);
int dist_sum_scalars(tvr_problem* p, double* vals, int n);
// halo_exchange(v) then fetch_scalars(nslots), with the halo send / recv and the scalar
// all-gather in ONE NCCL group (one launch, one synchronisation) on the NCCL backend
int halo_exchange_fetch(tvr_problem* p, float* v, int nslots);
// VIEWS mode: the A pass's source (slab -> full volume, all-gathered) and the A^T pass's
// target (full-volume partial -> slab, reduce-scattered); identity on one rank
bool views_dist(const tvr_problem* p);  // VIEWS or VIEWS_REP with world > 1
bool rep_dist(const tvr_problem* p);    // VIEWS_REP with world > 1
int replicate_volume(tvr_problem* p, float* v);
bool valid_comm(const void* comm);  // an NCCL or in-process thread communicator handle
int slab_table(tvr_problem* p);     // every rank's slab, gathered at create time (collective)
int setup_fused_rs(tvr_problem* p); // VIEWS: inboxes mapped on every peer (collective)
int dist_barrier(tvr_problem* p);   // stream-ordered barrier over the ranks (collective)
void dist_release(tvr_problem* p);  // unmap peer memory
int gather_volume(tvr_problem* p, const float* slab, const float** full);
int reduce_scatter_volume(tvr_problem* p, const float* full, float* slab);
void resolve_pending_timings(tvr_problem* p);

}  // namespace tvr
