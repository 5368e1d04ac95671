/* libtvreg.h — C ABI of the B200 hot path for accelerated-gradient TV CT reconstruction.
 *
 * Paper: J. H. Jorgensen, T. L. Jensen, P. C. Hansen, S. H. Jensen, E. Y. Sidky, X. Pan,
 * "Accelerated gradient methods for total-variation-based CT image reconstruction"
 * (arXiv:1105.4002; /root/reference/PAPER.md cited as P:line).
 *
 * The library minimises the Huber-smoothed objective
 *     phi_tau(x) = 1/2 ||A x - b||_2^2 + alpha * sum_j h_tau(||D_j x||_2),   x in Q = [lo, hi]^N
 * (Eq. (1)-(2); h_tau(t) = t - tau/2 for t >= tau, t^2/(2 tau) otherwise; D_j the
 * forward-difference gradient at voxel j with zero differences across each axis' last face)
 * by GPBB (Alg. 1) or UPN (Alg. 3, with BT of Alg. 2),
 * stopping on the gradient map G_nu (Eq. (10)).
 *
 * Conventions for every entry point:
 *  - Every function returns a tvr_status; no C++ exception crosses this boundary.  On a
 *    non-OK status tvr_last_error() returns a thread-local message.
 *  - Volume vectors are fp32, x fastest, then y, then z; in z-slab and views mode a rank's
 *    vectors hold only its slices [z0, z1) (N_local = nx*ny*(z1-z0)).  Data vectors are fp32
 *    of m_local (the rank's rows of A).
 *  - "_dev" pointers are DEVICE pointers on the problem's device, caller-owned (e.g. torch
 *    tensors' data_ptr()); "_host" pointers are host memory (pinned is fastest).
 *  - Calls are ordered on the problem's CUDA stream and return once every host-side output
 *    they report is valid (device outputs are complete when the call returns).  A
 *    library-created stream (tvr_dist NULL or cuda_stream NULL) is a BLOCKING stream: it waits
 *    for work queued on the legacy default stream (e.g. torch's default stream producing x_dev).
 *    With a caller stream, inputs must be produced on that stream or synchronised by the caller.
 *  - In distributed mode every call is collective: all ranks make it in the same order.
 *  - Arithmetic: fp32 storage; fp64 row accumulators, fp64 per-voxel TV math and fp64
 *    fixed-order reductions (deterministic run to run).
 */
#ifndef LIBTVREG_H
#define LIBTVREG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TVR_ABI_VERSION 6

typedef enum {
  TVR_OK = 0,
  TVR_NOT_CONVERGED = 1,    /* solver reached max_iters; x and the result are still filled in */
  TVR_E_ARG = -1,           /* invalid argument (NULL, size, tau <= 0, alpha < 0, lo >= hi, ...) */
  TVR_E_CSR = -2,           /* malformed CSR: row_ptr not monotone / not 0..nnz, column out of
                               range or not strictly ascending within a row, non-finite value */
  TVR_E_NOT_SEPARABLE = -3, /* z-slab mode: a local row touches voxels outside the rank's slab
                               (non-separable geometry: use TVR_SHARD_VIEWS) */
  TVR_E_CUDA = -4,          /* CUDA runtime error (message names the call) */
  TVR_E_NCCL = -5,          /* NCCL error */
  TVR_E_OOM = -6,           /* device allocation failed */
  TVR_E_NONFINITE = -7,     /* non-finite objective or gradient */
  TVR_E_LINESEARCH = -8,    /* GPBB beta < beta_min or BT exceeded bt_max trials */
  TVR_E_THETA = -9          /* UPN theta outside (0, 1] */
} tvr_status;

typedef struct tvr_problem tvr_problem; /* opaque, owned by the library */

/* System matrix A in CSR, HOST arrays, read only during tvr_create (caller keeps ownership).
 * row_ptr[n_rows+1] int64 (row_ptr[0] = 0, row_ptr[n_rows] = nnz, non-decreasing),
 * col_idx[nnz] int32 GLOBAL voxel indices, strictly ascending within each row,
 * val[nnz] fp32 finite.  n_cols = nx*ny*nz (global). */
typedef struct {
  int64_t n_rows, n_cols, nnz;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const float* val;
} tvr_csr;

typedef struct {
  int32_t nx, ny, nz; /* global volume; voxel j = (z*ny + y)*nx + x */
} tvr_grid;

enum { TVR_SHARD_NONE = 0, TVR_SHARD_ZSLAB = 1, TVR_SHARD_VIEWS = 2, TVR_SHARD_VIEWS_REP = 3 };

/* Distribution / placement.  NULL => one GPU, current device, a library-created stream.
 * ZSLAB (P1, slice-separable geometry): rank owns slices [z0, z1) and the rows
 *   of A whose voxels lie there; A and A^T need no communication.
 * VIEWS (P2, any geometry, e.g. rays tilted in z, BJ:11): rank owns an arbitrary block of A's
 *   rows (normally a contiguous range of projection views) with GLOBAL columns, and slices
 *   [z0, z1) of every volume vector.  Before each A pass the slabs of the point are
 *   all-gathered into a full-volume buffer; the A^T pass produces a full-volume partial
 *   A_p^T r_p that is reduce-scattered (fp32 sum) to the slabs.
 * VIEWS_REP (P2 with replicated iterates): rows and slabs as VIEWS, but the
 *   solvers keep every volume vector WHOLE on every rank: trial and momentum points are formed
 *   redundantly outside the slab (no communication), so the A pass needs no all-gather; the
 *   gradient's slab (stencil over the slab, after the A^T reduce-scatter) is all-gathered once
 *   per gradient instead of the point once per A pass.  Same results as VIEWS, bitwise.  The
 *   caller's vectors are still slabs [z0, z1).
 * In ZSLAB / VIEWS the TV stencil exchanges one halo slice with each z-neighbour over NCCL
 * (nccl_comm from tvr_nccl_comm_init) and scalars are all-gathered and summed in rank order.
 * The slabs must tile [0, nz) in rank order (rank r's z1 = rank r+1's z0). */
typedef struct {
  int32_t world, rank, mode;
  int32_t z0, z1;
  void* nccl_comm;   /* communicator from tvr_nccl_comm_init / tvr_local_comm_create, or NULL
                        (world == 1) */
  int32_t device;    /* CUDA device ordinal, or -1 for the current device */
  void* cuda_stream; /* cudaStream_t to order work on, or NULL for a library-created stream */
} tvr_dist;

/* Create a problem for phi_tau(x) = 1/2||Ax - b||^2 + alpha TV_tau(x), x in Q = [lo, hi]^N
 * (Eq. (1)-(2); Q per P:77, a scalar box C22; b = A x_true + e of Eq. (11),
 * P:243-245, supplied by the caller).  Validates A (TVR_E_CSR), copies A and b to device memory,
 * builds the canonical transposed CSR on the device (bit-exact, rows of A^T ascending
 * by source row, values moved bit for bit), and detects slice-separable structure for
 * slab-staged SpMV.  A_local: host CSR (caller-owned, read only during the call).
 * b_host: m_local fp32 values (host, caller-owned).  alpha >= 0 (alpha = 0 allowed, C24),
 * tau > 0 (Huber smoothing, C1), lo < hi (+-INFINITY allowed).  *out receives a library-owned
 * handle (tvr_destroy).  Errors: TVR_E_ARG, TVR_E_CSR, TVR_E_NOT_SEPARABLE, TVR_E_CUDA,
 * TVR_E_NCCL, TVR_E_OOM; on error *out is NULL and nothing is leaked. */
int tvr_create(tvr_problem** out, const tvr_csr* A_local, const float* b_host, tvr_grid grid,
               double alpha, double tau, double lo, double hi, const tvr_dist* dist);

/* Slice-shared operator (structure-exploiting projector; BJ:5, BJ:7).
 * For slice-invariant geometry (parallel beam, rays inside z-slices, the same 2D geometry in
 * every slice: configs c1-c4) the system matrix is block diagonal with one repeated block,
 * A = I_nz (x) A_slice (Eq.(1); the ray model of P:238-245 restricted to one slice):
 *   row z*m_s + i of A has the entries of row i of A_slice on the columns z*nx*ny + c.
 * A_slice: m_s rows, n_cols = nx*ny, HOST CSR with the same rules as tvr_create (columns are
 *   in-slice voxel indices y*nx + x); read only during the call.
 * b_host: m_s * nz_local fp32 (host), slice-major (the rows of slice z0 first).
 * The device stores only A_slice and its transpose (c2: 7.5 MB instead of 1.9 GB) and applies
 * them to every slice; every other call behaves as for tvr_create on the expanded matrix
 * (results equal to fp32 rounding, the same fp64 reductions).  tvr_get_AT returns the
 * transpose of A_slice (nx*ny rows).
 * dist: NULL / NONE or ZSLAB (each rank passes the same A_slice and its slab's rows of b);
 * VIEWS -> TVR_E_ARG.  Needs nx*ny <= 65536 and m_s <= 65536 (16-bit window offsets),
 * else TVR_E_ARG; TVR_E_OOM if the sliced-ELL copy does not fit. */
int tvr_create_sliced(tvr_problem** out, const tvr_csr* A_slice, const float* b_host,
                      tvr_grid grid, double alpha, double tau, double lo, double hi,
                      const tvr_dist* dist);
void tvr_destroy(tvr_problem* p);

typedef struct {
  int64_t m_local, n_local, nnz_local; /* local sizes (n_local = voxels owned) */
  int32_t z0, z1;                      /* owned slices */
  int32_t slab_staged_A, slab_staged_AT; /* SpMV kernel: 0 global gathers, 1 slice staged in
                                           smem, 2 slice staged + TMA bulk-copy pipeline */
  int64_t device_bytes;                /* device memory held by the problem */
  int64_t n_cols_local;                /* columns of the local A (= rows of its A^T): N_local,
                                          or N in VIEWS mode */
  int32_t views_fused_rs;              /* VIEWS mode: 1 if the A^T pass stores into the owners'
                                          inboxes over peer memory (fused reduce-scatter), 0 if
                                          it uses the collective reduce-scatter */
  int32_t slice_shared;                /* tvr_create_sliced: slices sharing the stored slice
                                          matrix (the slab's nz); 0 for tvr_create */
  int32_t views_rep;                   /* VIEWS_REP with world > 1: the solvers' volume vectors
                                          are whole on every rank */
  int64_t point_allgathers;            /* VIEWS modes: all-gathers of a point before an A pass
                                          so far (VIEWS: one per A pass; VIEWS_REP: only for a
                                          caller's slab) */
  int64_t gather_layout_blocks[3];     /* non-separable A pass (int32 sliced ELL with block
                                          modes): 32-ray blocks gathering from the point laid out
                                          row-major, with x / y swapped, in 8x4 bricks */
  int64_t dist_graph_solves;           /* solves run as one CUDA graph WITH the NCCL exchanges
                                          captured in it (device control on an NCCL
                                          communicator, tvr_set_control) */
  int64_t dist_graph_exchanges;        /* ... and the captured exchange groups those graphs
                                          executed (one per line-search / BT trial, one per
                                          accepted gradient) */
} tvr_info;
int tvr_get_info(const tvr_problem* p, tvr_info* info);

/* Objective parts: phi = fidelity + alpha * tv. */
typedef struct {
  double fidelity, tv, f;
} tvr_fparts;

/* One gradient evaluation (the unit of BJ:2's metric): f = phi_tau(x) (Eq. (1)) and
 * g = grad phi_tau(x) = A^T(Ax - b) + alpha grad TV_tau(x) (the gradient of Eq. (1)-(2); TV_tau's
 * gradient sum_j D_j^T (D_j x / max(||D_j x||, tau)), C2), i.e. the A pass with the fused
 * residual (a1), the A^T pass (a2) and the fused stencil (a4).  x_dev, g_dev: N_local fp32
 * DEVICE vectors, caller-owned (g_dev may be NULL: value only, no A^T pass).  f_out: host, the
 * fp64 value (identical on every rank).  parts may be NULL.  Collective in distributed mode.
 * Errors: TVR_E_ARG (NULL x_dev / f_out), TVR_E_CUDA, TVR_E_NCCL. */
int tvr_objective_grad(tvr_problem* p, const float* x_dev, double* f_out, float* g_dev,
                       tvr_fparts* parts);
/* Same computation with HOST x and g (copied inside the call: the end-to-end API). */
int tvr_objective_grad_host(tvr_problem* p, const float* x_host, double* f_out, float* g_host,
                            tvr_fparts* parts);

enum { TVR_STOP_REL = 0, TVR_STOP_ABS_PER_N = 1 };

/* GPBB options; tvr_gpbb_default fills K = 2, sigma = 0.1, beta0 = 0.95,
 * beta_min = 1e-10, eps = 1e-6, TVR_STOP_REL, max_iters = 10000. */
typedef struct {
  int64_t max_iters;
  double eps;
  int32_t stop_mode; /* REL: ||G_nu(x_k)|| <= eps ||G_1(x_0)||; ABS_PER_N: ||G_nu(x_k)||/N <= eps */
  int32_t K;
  double sigma, beta0, beta_min;
} tvr_gpbb_opts;

/* UPN options; tvr_upn_default fills L0 = 1, mu0 = 1 (mu_bar = L_bar), rho_L = 1.3, bt_max = 200. */
typedef struct {
  int64_t max_iters;
  double eps;
  int32_t stop_mode;
  double L0, mu0, rho_L;
  int32_t bt_max;
} tvr_upn_opts;

/* GP options: the paper's baseline comparator, Eq. (6), x_{k+1} = P_Q(x_k - g_k/L_k)
 * with L_k found by BT (Alg. 2) starting from L_{k-1} (the oracle's
 * gp() follows the same steps).  tvr_gp_default fills L0 = 1, rho_L = 1.3, bt_max = 200,
 * eps = 1e-6, TVR_STOP_REL, max_iters = 10000. */
typedef struct {
  int64_t max_iters;
  double eps;
  int32_t stop_mode;
  double L0, rho_L;
  int32_t bt_max;
} tvr_gp_opts;

void tvr_gpbb_default(tvr_gpbb_opts* o);
void tvr_upn_default(tvr_upn_opts* o);
void tvr_gp_default(tvr_gp_opts* o);

/* One record per accepted iteration (GPBB: the iterate tested at the top of iteration k;
 * UPN: x_{k}).  step_or_inv_L = theta_k (GPBB) or 1/L_k (UPN). */
typedef struct {
  int64_t iter;
  double f, gmap_rel, gmap_abs_per_n, step_or_inv_L, mu, L;
  int32_t ls_trials;
  int32_t _pad;
} tvr_record;

typedef struct {
  int32_t converged;
  int32_t _pad;
  int64_t iters, n_f, n_grad, n_ls;
  int64_t n_records; /* records produced (may exceed hist_cap; min(n_records, hist_cap) stored) */
  double f, gmap_rel, gmap_abs_per_n, gmap_ref, seconds, bytes;
} tvr_result;

/* Solve min phi_tau over Q (Eq. (1)) from x_dev_inout (projected onto Q first, C13); on return
 * it holds the last iterate tested by the stopping rule (Eq. (10); C14).
 *   tvr_solve_gpbb: GPBB, Alg. 1: BB step, nonmonotone Armijo line
 *     search over the last K+1 accepted values; readings C6, C11, C21.
 *   tvr_solve_upn: UPN, Alg. 3 with BT, Alg. 2 and the mu_k estimate of
 *     Eq. (9); readings C7-C10.  Its iterates are carried as fp32 hi + lo pairs (the
 *     objective is evaluated at the hi part).
 * x_dev_inout: N_local fp32 device vector, caller-owned.  hist may be NULL; records beyond
 * hist_cap are counted but not stored.  Returns TVR_OK (converged), TVR_NOT_CONVERGED
 * (max_iters; x and res still filled in), TVR_E_LINESEARCH, TVR_E_THETA, TVR_E_NONFINITE,
 * TVR_E_ARG (invalid options), TVR_E_CUDA, TVR_E_NCCL. */
int tvr_solve_gpbb(tvr_problem* p, float* x_dev_inout, const tvr_gpbb_opts* opts, tvr_result* res,
                   tvr_record* hist, int64_t hist_cap);
int tvr_solve_upn(tvr_problem* p, float* x_dev_inout, const tvr_upn_opts* opts, tvr_result* res,
                  tvr_record* hist, int64_t hist_cap);
/* GP (f1): same conventions as tvr_solve_upn; records carry 1/L_k, the stop test runs at x_{k+1}
 * with nu = L_k (as UPN, C11). */
int tvr_solve_gp(tvr_problem* p, float* x_dev_inout, const tvr_gp_opts* opts, tvr_result* res,
                 tvr_record* hist, int64_t hist_cap);

/* ---- inspection hooks (tests) ---- */
/* r = A x - b (the a1 pass: the operand of the fidelity term of Eq. (1), fused with the
 * residual) and *fid = 1/2 ||Ax - b||^2 in fp64 (nullable).  x_dev: N_local fp32 device
 * vector; r_dev: m_local fp32 device vector (caller-owned).  Errors: TVR_E_ARG, TVR_E_CUDA. */
int tvr_residual(tvr_problem* p, const float* x_dev, float* r_dev, double* fid);
/* y = A x (the forward projection of Eq. (1), without b).  x_dev: N_local fp32 device
 * vector (VIEWS mode: the rank's slab; collective), y_dev: m_local fp32 device vector.
 * Row sums in fp64, rounded once to fp32.  Errors: TVR_E_ARG, TVR_E_CUDA, TVR_E_NCCL. */
int tvr_apply_A(tvr_problem* p, const float* x_dev, float* y_dev);
/* w = A^T y (the back-projection in the gradient of Eq. (1)) from the stored transposed
 * CSR, no atomics (the a2 pass, BJ:5).  y_dev: m_local fp32 device vector, w_dev: N_local fp32
 * device vector, caller-owned (VIEWS mode: the rank's slab of sum_p A_p^T y_p; collective).
 * Row sums in fp64, rounded once.  Errors: TVR_E_ARG, TVR_E_CUDA, TVR_E_NCCL. */
int tvr_apply_AT(tvr_problem* p, const float* y_dev, float* w_dev);
/* TV_tau(x) = sum_j h_tau(||D_j x||_2) (Eq. (2), P:81-85 with the Huber smoothing C1 and the
 * Neumann forward differences C3) into *tv_out (fp64, host) and, if grad_dev != NULL, its
 * gradient (C2) as N_local fp32.  x_dev: N_local fp32 device vector.  Errors: TVR_E_ARG,
 * TVR_E_CUDA, TVR_E_NCCL (halo exchange). */
int tvr_tv(tvr_problem* p, const float* x_dev, double* tv_out, float* grad_dev);
/* ||G_nu(x)||_2 with G_nu(x) = nu (x - P_Q(x - grad f(x)/nu)) (Eq. (10)); G_dev nullable. */
int tvr_gradient_map(tvr_problem* p, const float* x_dev, double nu, double* norm_out, float* G_dev);
/* Copy the device transposed CSR to host arrays of n_cols_local+1 / nnz_local entries
 * (n_cols_local = N_local, or N in VIEWS mode, where A^T of the local rows spans the volume).
 * Slice-shared problems (tvr_create_sliced): the transpose of A_slice, nx*ny+1 / nnz_local /
 * slice_shared entries. */
int tvr_get_AT(tvr_problem* p, int64_t* row_ptr_host, int32_t* col_host, float* val_host);

/* ---- per-kernel timing (CUDA events on the problem's stream) ---- */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;
  double bytes; /* algorithmic bytes summed over launches */
} tvr_kernel_stat;
int tvr_profile_enable(tvr_problem* p, int on); /* on=1 clears counters and starts recording */
int tvr_profile_get(tvr_problem* p, tvr_kernel_stat* out, int cap, int* n_out);
/* Number of kernels launched by the library since tvr_create (or the last reset). */
int64_t tvr_launch_count(const tvr_problem* p, int reset);

/* Solver control for GPBB and UPN.  HOST: the scalar logic of every line-search
 * / BT trial runs on the host after a device->host fetch of the pass reductions.  DEVICE: a whole
 * solve is one CUDA graph with conditional while / if nodes; single-thread control kernels take
 * the same decisions in the same fp64 arithmetic (identical iterates), the host waits once; the
 * state rotates by device copies.  With an NCCL communicator (world > 1) DEVICE captures the
 * exchanges in the graph as well: the halo send / recv of the gradient and the scalar all-gather
 * are one NCCL group per decision point, the gathered partials are summed in rank order by a
 * device kernel (the host sum's arithmetic), trial / momentum halo planes are recomputed from
 * device-side step parameters — no host synchronisation per trial.  It
 * is opt-in there (AUTO keeps HOST at world > 1; the in-process thread communicator synchronises
 * on the host and always uses HOST).  TVR_DIST_GRAPH_FORCE=1 takes this path on a one-rank NCCL
 * communicator too (tests).  AUTO (default): DEVICE where launch and synchronisation latency is a visible part of
 * an iteration — GPBB below 2^28 matrix entries (c1 -16 % per iteration; c2 equal), UPN below 2^24
 * (c1 -11 %; its extended-precision graph is slower than host control at c2) — HOST above (c3:
 * the state copies cost 1-2 %).  The environment variable
 * TVR_CONTROL=host|device overrides. */
enum { TVR_CONTROL_HOST = 0, TVR_CONTROL_DEVICE = 1, TVR_CONTROL_AUTO = 2 };
int tvr_set_control(tvr_problem* p, int mode);

/* Inspection hook of the plan builder (host only, no GPU): the CTA block ranges of a sliced-ELL
 * pass (DESIGN §5.2 "CTA ranges by simulated makespan").  blk_steps[i] /
 * blk_slice[i]: 8-entry chunk steps and slice of stored block i (slices ascending); a CTA's range
 * is walked slice segment by slice segment, nwarps warps taking blocks in order.  tab_out
 * (grid + 1 entries): tab_out[c] = first block of CTA c, tab_out[grid] = nblk, non-decreasing.
 * Cost of a range = lambda x list-scheduled makespan + (1 - lambda) x work sum / nwarps, block
 * cost = steps + blk_cost, seg_cost per segment.  TVR_E_ARG on NULL / out-of-range arguments. */
int tvr_sell_partition(const int32_t* blk_steps, const int32_t* blk_slice, int64_t nblk, int nwarps,
                       int grid, double blk_cost, double seg_cost, double lambda, int64_t* tab_out);

/* Inspection hook of the distributed device control: out_dev[s] = sum over r (in rank order,
 * starting from +0.0) of gathered_dev[r * n + s], the kernel the solver graphs run after the
 * scalar all-gather (fixed-order fp64 sums).  Device pointers; synchronises
 * cuda_stream (NULL: the default stream).  TVR_E_ARG on NULL / non-positive sizes. */
int tvr_rank_sum(const double* gathered_dev, int world, int n, double* out_dev, void* cuda_stream);

/* In-process thread communicator (testing the multi-rank paths on one GPU): ranks are host
 * threads of one process, each with its own tvr_problem (same or different devices); every
 * collective is a host barrier, device-to-device copies from the peers' buffers and a second
 * barrier.  Pass the handle as tvr_dist.nccl_comm of every rank.  Not a performance path. */
int tvr_local_comm_create(void** comm_out, int world);
int tvr_local_comm_destroy(void* comm);

/* ---- NCCL bootstrap (z-slab mode) ---- */
int tvr_nccl_unique_id_size(void);
int tvr_nccl_get_unique_id(void* id_out);
int tvr_nccl_comm_init(void** comm_out, const void* id, int world, int rank, int device);
int tvr_nccl_comm_destroy(void* comm);

/* Optional device allocator hook (e.g. the PyTorch caching allocator); NULL restores cudaMalloc. */
typedef void* (*tvr_alloc_fn)(size_t bytes, int device, void* stream, void* ctx);
typedef void (*tvr_free_fn)(void* ptr, int device, void* stream, void* ctx);
int tvr_set_allocator(tvr_alloc_fn alloc_fn, tvr_free_fn free_fn, void* ctx);

const char* tvr_last_error(void);
int tvr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LIBTVREG_H */
