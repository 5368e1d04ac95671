// Distribution.  Both modes: one-slice halo exchange with each
// z-neighbour and a rank-ordered fp64 scalar sum (all-gather of the partial scalars, then a
// fixed-order sum on the host, so every rank sees bitwise-identical scalars and takes the same
// line-search / BT branch).  Trial and momentum points never need a halo exchange: their halo
// planes are recomputed from the halo planes of their inputs with the stencil's own functors
// (bitwise equal to the neighbour's stored values); only gradients are exchanged.
// VIEWS mode (P2, non-separable geometry) adds an all-gather of the point before every A pass
// and a reduce-scatter of the full-volume A_p^T r_p after every A^T pass.
//
// Two communicator backends behind one handle (tvr_dist.nccl_comm):
//  * NCCL (tvr_nccl_comm_init): one process per GPU over NVLink / NVSwitch, the product path;
//  * an in-process thread communicator (tvr_local_comm_create): ranks are host threads of one
//    process, possibly sharing one GPU; every collective is host barrier -> device-to-device
//    copies from the peers' buffers -> host barrier.  No kernel ever waits on another rank, so
//    ranks on one GPU cannot deadlock.  It exists to run the multi-rank library logic (halo
//    planes, P2 gather / reduce-scatter, rank-ordered sums, distributed solvers) on the one-GPU
//    boxes of this build; it is not a performance path.
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "problem.h"

namespace tvr {

#define TVR_NCCL(call)                                                                  \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess) {                                                            \
      ::tvr::set_error(std::string(#call) + ": " + ncclGetErrorString(_r));             \
      return TVR_E_NCCL;                                                                \
    }                                                                                   \
  } while (0)

constexpr uint32_t kNcclMagic = 0x4e43434cu;   // "NCCL"
constexpr uint32_t kLocalMagic = 0x4c4f434cu;  // "LOCL"

struct CommBase {
  uint32_t magic;
};
struct NcclComm : CommBase {
  ncclComm_t c;
};
struct LocalComm : CommBase {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<const void*> ptr;   // per rank: published device pointer
  std::vector<int64_t> val;       // per rank: published integers
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

__global__ void add_inplace_kernel(int64_t n, const float* __restrict__ a, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a[i];
}
static cudaError_t launch_add_inplace(int64_t n, const float* a, float* y, cudaStream_t st) {
  add_inplace_kernel<<<592, 256, 0, st>>>(n, a, y);
  return cudaGetLastError();
}

static ncclComm_t nccl_of(const tvr_problem* p) { return static_cast<NcclComm*>(p->comm)->c; }
static LocalComm* local_of(const tvr_problem* p) {
  auto* b = static_cast<CommBase*>(p->comm);
  return (b && b->magic == kLocalMagic) ? static_cast<LocalComm*>(b) : nullptr;
}

bool valid_comm(const void* comm) {
  if (!comm) return false;
  const uint32_t m = static_cast<const CommBase*>(comm)->magic;
  return m == kNcclMagic || m == kLocalMagic;
}

// Local backend: publish this rank's pointer, wait for all, run copy(peer pointers), wait again
// (so no rank overwrites a published buffer before every peer has read it).
template <class F>
static int local_collective(tvr_problem* p, const void* mine, F&& copy) {
  LocalComm* L = local_of(p);
  TVR_CUDA(cudaStreamSynchronize(p->stream));  // this rank's data is complete
  L->ptr[p->rank] = mine;
  L->barrier();
  const int st = copy(L->ptr);
  cudaError_t e = cudaStreamSynchronize(p->stream);
  L->barrier();
  if (st < 0) return st;
  if (e != cudaSuccess) { set_error(std::string("local collective: ") + cudaGetErrorString(e)); return TVR_E_CUDA; }
  return TVR_OK;
}

int halo_exchange_to(tvr_problem* p, const float* v, float* lo, float* hi) {
  NvtxRange nv("halo_exchange");
  if (p->world <= 1) return TVR_OK;
  const size_t bytes = sizeof(float) * (size_t)p->plane;
  if (LocalComm* L = local_of(p)) {
    (void)L;
    return local_collective(p, v, [&](const std::vector<const void*>& peer) -> int {
      if (p->rank > 0) {  // lower halo = last owned plane of rank - 1
        const float* src = static_cast<const float*>(peer[p->rank - 1]);
        const int nzl_lo = (int)p->peer_nzl[p->rank - 1];
        TVR_CUDA(cudaMemcpyAsync(lo, src + (int64_t)(nzl_lo - 1) * p->plane, bytes,
                                 cudaMemcpyDeviceToDevice, p->stream));
      }
      if (p->rank < p->world - 1) {  // upper halo = first owned plane of rank + 1
        TVR_CUDA(cudaMemcpyAsync(hi, peer[p->rank + 1], bytes, cudaMemcpyDeviceToDevice, p->stream));
      }
      return TVR_OK;
    });
  }
  ncclComm_t comm = nccl_of(p);
  const size_t cnt = (size_t)p->plane;
  TVR_NCCL(ncclGroupStart());
  if (p->rank > 0) {
    TVR_NCCL(ncclSend(v, cnt, ncclFloat, p->rank - 1, comm, p->stream));
    TVR_NCCL(ncclRecv(lo, cnt, ncclFloat, p->rank - 1, comm, p->stream));
  }
  if (p->rank < p->world - 1) {
    TVR_NCCL(ncclSend(v + (int64_t)(p->nzl - 1) * p->plane, cnt, ncclFloat, p->rank + 1, comm, p->stream));
    TVR_NCCL(ncclRecv(hi, cnt, ncclFloat, p->rank + 1, comm, p->stream));
  }
  TVR_NCCL(ncclGroupEnd());
  return TVR_OK;
}

int halo_exchange(tvr_problem* p, float* v) {
  if (rep_dist(p)) return replicate_volume(p, v);
  return halo_exchange_to(p, v, v - p->plane, v + (int64_t)p->nzl * p->plane);
}

// planes of a point recomputed outside the owned slab: the z-neighbours' halo planes (-1, nzl),
// or in VIEWS_REP every plane of the replicated vector outside [z0, z1)
static int fill_lo(const tvr_problem* p) { return rep_dist(p) ? p->z0 : (p->z0 > 0 ? 1 : 0); }
static int fill_hi(const tvr_problem* p) { return rep_dist(p) ? p->nz - p->z1 : (p->z1 < p->nz ? 1 : 0); }

int halo_fill_trial(tvr_problem* p, const float* x, const float* g, double s, float* v,
                    const double* dparam) {
  if (p->world <= 1) return TVR_OK;
  TVR_CUDA(launch_halo_fill_trial(x, g, s, p->lo, p->hi, p->plane, p->nzl, fill_lo(p),
                                  fill_hi(p), v, p->stream, dparam));
  p->launches++;
  return TVR_OK;
}

int halo_fill_momentum(tvr_problem* p, const float* x1, const float* x0, double beta, float* y,
                       const double* dparam) {
  if (p->world <= 1) return TVR_OK;
  TVR_CUDA(launch_halo_fill_momentum(x1, x0, beta, p->plane, p->nzl, fill_lo(p), fill_hi(p), y,
                                     p->stream, dparam));
  p->launches++;
  return TVR_OK;
}

int halo_fill_trial_x(tvr_problem* p, const float* x, const float* x_lo, const float* g, double s,
                      float* v, float* v_lo, const double* dparam) {
  if (p->world <= 1) return TVR_OK;
  TVR_CUDA(launch_halo_fill_trial_x(x, x_lo, g, s, p->lo, p->hi, p->plane, p->nzl, fill_lo(p),
                                    fill_hi(p), v, v_lo, p->stream, dparam));
  p->launches++;
  return TVR_OK;
}

int halo_fill_momentum_x(tvr_problem* p, const float* x1, const float* x1_lo, const float* x0,
                         const float* x0_lo, double beta, float* y, float* y_lo,
                         const double* dparam) {
  if (p->world <= 1) return TVR_OK;
  TVR_CUDA(launch_halo_fill_momentum_x(x1, x1_lo, x0, x0_lo, beta, p->plane, p->nzl, fill_lo(p),
                                       fill_hi(p), y, y_lo, p->stream, dparam));
  p->launches++;
  return TVR_OK;
}

int reduce_gathered_scalars(tvr_problem* p, double* vals, int n);

int halo_exchange_fetch(tvr_problem* p, float* v, int nslots) {
  if (p->world <= 1 || local_of(p) || rep_dist(p)) {
    TVR_TRY(halo_exchange(p, v));
    return fetch_scalars(p, nslots);
  }
  NvtxRange nv("halo_exchange + scalar_allgather");
  ncclComm_t comm = nccl_of(p);
  const size_t cnt = (size_t)p->plane;
  TVR_NCCL(ncclGroupStart());
  if (p->rank > 0) {
    TVR_NCCL(ncclSend(v, cnt, ncclFloat, p->rank - 1, comm, p->stream));
    TVR_NCCL(ncclRecv(v - p->plane, cnt, ncclFloat, p->rank - 1, comm, p->stream));
  }
  if (p->rank < p->world - 1) {
    TVR_NCCL(ncclSend(v + (int64_t)(p->nzl - 1) * p->plane, cnt, ncclFloat, p->rank + 1, comm, p->stream));
    TVR_NCCL(ncclRecv(v + (int64_t)p->nzl * p->plane, cnt, ncclFloat, p->rank + 1, comm, p->stream));
  }
  TVR_NCCL(ncclAllGather(p->dscal, p->dgather, (size_t)nslots, ncclDouble, comm, p->stream));
  TVR_NCCL(ncclGroupEnd());
  return reduce_gathered_scalars(p, p->hscal, nslots);
}

// Device-side rank-ordered sum (solver graphs at world > 1): out[s] =
// ((0 + all[0][s]) + all[1][s]) + ..., the host sum of reduce_gathered_scalars operation for
// operation, so every rank's control kernels read bitwise the scalars the host controller sums.
__global__ void rank_sum_kernel(const double* __restrict__ all, int world, int n,
                                double* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double acc = 0.0;
  for (int r = 0; r < world; ++r) acc = __dadd_rn(acc, all[(size_t)r * n + s]);
  out[s] = acc;
}

bool nccl_backend(const tvr_problem* p) { return p->comm && !local_of(p); }

// The exchanges of halo_exchange_fetch without the host: the halo planes of v (nullable) and the
// scalar all-gather in one NCCL group (VIEWS_REP: the in-place all-gather of v, then the scalars),
// the rank-ordered sum on the device into p->dsum.  Enqueue only -- capturable into the solver
// graphs.  Runs the all-gather on a one-rank communicator too (the forced path of the tests).
int dist_scalars_dev(tvr_problem* p, float* v, int nslots) {
  NvtxRange nv("halo_exchange + scalar_allgather (device sum)");
  ncclComm_t comm = nccl_of(p);
  const size_t cnt = (size_t)p->plane;
  if (v && rep_dist(p)) {
    TVR_TRY(replicate_volume(p, v));
    v = nullptr;
  }
  TVR_NCCL(ncclGroupStart());
  if (v && p->world > 1) {
    if (p->rank > 0) {
      TVR_NCCL(ncclSend(v, cnt, ncclFloat, p->rank - 1, comm, p->stream));
      TVR_NCCL(ncclRecv(v - p->plane, cnt, ncclFloat, p->rank - 1, comm, p->stream));
    }
    if (p->rank < p->world - 1) {
      TVR_NCCL(ncclSend(v + (int64_t)(p->nzl - 1) * p->plane, cnt, ncclFloat, p->rank + 1, comm, p->stream));
      TVR_NCCL(ncclRecv(v + (int64_t)p->nzl * p->plane, cnt, ncclFloat, p->rank + 1, comm, p->stream));
    }
  }
  TVR_NCCL(ncclAllGather(p->dscal, p->dgather, (size_t)nslots, ncclDouble, comm, p->stream));
  TVR_NCCL(ncclGroupEnd());
  rank_sum_kernel<<<1, 64, 0, p->stream>>>(p->dgather, p->world, nslots, p->dsum);
  TVR_CUDA(cudaGetLastError());
  p->launches++;
  return TVR_OK;
}

// rank-ordered sum of the all-gathered scalars (p->dgather, world x n) into vals (host)
int reduce_gathered_scalars(tvr_problem* p, double* vals, int n) {
  double* all = p->hscal + 64;  // world x n staging after the first 64 slots
  TVR_CUDA(cudaMemcpyAsync(all, p->dgather, sizeof(double) * n * p->world, cudaMemcpyDeviceToHost,
                           p->stream));
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  resolve_pending_timings(p);
  for (int s = 0; s < n; ++s) {
    double acc = 0.0;
    for (int r = 0; r < p->world; ++r) acc += all[(size_t)r * n + s];  // rank order
    vals[s] = acc;
  }
  return TVR_OK;
}

int dist_sum_scalars(tvr_problem* p, double* vals, int n) {
  NvtxRange nv("scalar_allgather");
  if (local_of(p)) {
    TVR_TRY(local_collective(p, p->dscal, [&](const std::vector<const void*>& peer) -> int {
      for (int r = 0; r < p->world; ++r)
        TVR_CUDA(cudaMemcpyAsync(p->dgather + (size_t)r * n, peer[r], sizeof(double) * n,
                                 cudaMemcpyDeviceToDevice, p->stream));
      return TVR_OK;
    }));
  } else {
    TVR_NCCL(ncclAllGather(p->dscal, p->dgather, (size_t)n, ncclDouble, nccl_of(p), p->stream));
  }
  return reduce_gathered_scalars(p, vals, n);
}

// Every rank's slab [z0, z1), gathered once at create time (the halo exchange of the local
// backend needs the lower neighbour's plane count; VIEWS mode needs every slab).
int slab_table(tvr_problem* p) {
  std::vector<int64_t> all(2 * p->world);
  if (LocalComm* L = local_of(p)) {
    L->val[2 * p->rank] = p->z0;
    L->val[2 * p->rank + 1] = p->z1;
    L->barrier();
    for (int i = 0; i < 2 * p->world; ++i) all[i] = L->val[i];
    L->barrier();
  } else {
    int64_t* d = nullptr;
    TVR_CUDA(cudaMalloc(&d, sizeof(int64_t) * 2 * (p->world + 1)));
    std::vector<int64_t> mine = {p->z0, p->z1};
    cudaError_t e = cudaMemcpyAsync(d, mine.data(), sizeof(int64_t) * 2, cudaMemcpyHostToDevice,
                                    p->stream);
    ncclResult_t nr = ncclSuccess;
    if (e == cudaSuccess) nr = ncclAllGather(d, d + 2, 2, ncclInt64, nccl_of(p), p->stream);
    if (e == cudaSuccess && nr == ncclSuccess)
      e = cudaMemcpyAsync(all.data(), d + 2, sizeof(int64_t) * 2 * p->world, cudaMemcpyDeviceToHost,
                          p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    cudaFree(d);
    if (nr != ncclSuccess) { set_error(std::string("slab table: ") + ncclGetErrorString(nr)); return TVR_E_NCCL; }
    if (e != cudaSuccess) { set_error(std::string("slab table: ") + cudaGetErrorString(e)); return TVR_E_CUDA; }
  }
  p->slab_off.assign(p->world, 0);
  p->slab_cnt.assign(p->world, 0);
  p->peer_nzl.assign(p->world, 0);
  for (int r = 0; r < p->world; ++r) {
    const int64_t z0 = all[2 * r], z1 = all[2 * r + 1];
    if (z0 != (r == 0 ? 0 : all[2 * r - 1]) || z1 <= z0 || (r == p->world - 1 && z1 != p->nz)) {
      set_error("tvr_create: the ranks' slabs must tile [0, nz) in rank order");
      return TVR_E_ARG;
    }
    p->slab_off[r] = z0 * p->plane;
    p->slab_cnt[r] = (z1 - z0) * p->plane;
    p->peer_nzl[r] = z1 - z0;
  }
  return TVR_OK;
}

// ---- VIEWS mode: rows split by projection views, volume vectors by z-slabs.
bool views_dist(const tvr_problem* p) {
  return (p->mode == TVR_SHARD_VIEWS || p->mode == TVR_SHARD_VIEWS_REP) && p->world > 1;
}
// VIEWS_REP: the library's volume vectors are whole volumes on every rank (a slab pointer v is
// base + z0 plane); a point is made whole once (replicate_volume after its owned slab is
// written, or the trial / momentum fills over the planes outside the slab), so the A pass reads
// it without an all-gather
bool rep_dist(const tvr_problem* p) { return p->mode == TVR_SHARD_VIEWS_REP && p->world > 1; }

// a slab pointer into one of the library's replicated volume vectors (not a caller's slab)
static bool rep_internal(const tvr_problem* p, const float* slab) {
  const float* base = slab - (int64_t)p->z0 * p->plane;
  for (const float* b : p->vol_base)
    if (b == base) return true;
  return false;
}

static bool uniform_slabs(const tvr_problem* p) {
  for (int r = 1; r < p->world; ++r)
    if (p->slab_cnt[r] != p->slab_cnt[0]) return false;
  return true;
}

// x_full[off_r : off_r + cnt_r] = slab of rank r, on every rank (the A pass needs the whole
// point: a tilted ray crosses every slab).  NCCL: equal slabs one ncclAllGather, ragged slabs
// one broadcast per rank inside a group.
int gather_volume(tvr_problem* p, const float* slab, const float** full) {
  NvtxRange nv("views_allgather");
  if (!views_dist(p)) {
    *full = slab;
    return TVR_OK;
  }
  if (rep_dist(p) && rep_internal(p, slab)) {  // already whole on this rank
    *full = slab - (int64_t)p->z0 * p->plane;
    return TVR_OK;
  }
  ++p->n_gathers;
  if (local_of(p)) {
    TVR_TRY(local_collective(p, slab, [&](const std::vector<const void*>& peer) -> int {
      for (int r = 0; r < p->world; ++r)
        TVR_CUDA(cudaMemcpyAsync(p->xfull + p->slab_off[r], peer[r], sizeof(float) * p->slab_cnt[r],
                                 cudaMemcpyDeviceToDevice, p->stream));
      return TVR_OK;
    }));
  } else if (uniform_slabs(p)) {
    TVR_NCCL(ncclAllGather(slab, p->xfull, (size_t)p->slab_cnt[0], ncclFloat, nccl_of(p), p->stream));
  } else {
    TVR_NCCL(ncclGroupStart());
    for (int r = 0; r < p->world; ++r) {
      float* dst = p->xfull + p->slab_off[r];
      TVR_NCCL(ncclBroadcast(r == p->rank ? (const void*)slab : (const void*)dst, dst,
                             (size_t)p->slab_cnt[r], ncclFloat, r, nccl_of(p), p->stream));
    }
    TVR_NCCL(ncclGroupEnd());
  }
  *full = p->xfull;
  return TVR_OK;
}

// VIEWS_REP: every rank's slab of the replicated vector v (slab pointer) lands in everybody's
// copy, in place (the one all-gather of a gradient per iteration that replaces the all-gather of
// the point before every A pass).  NCCL: equal slabs one in-place ncclAllGather, ragged slabs
// one in-place broadcast per rank.
int replicate_volume(tvr_problem* p, float* v) {
  NvtxRange nv("views_rep_allgather");
  float* full = v - (int64_t)p->z0 * p->plane;
  if (local_of(p)) {
    return local_collective(p, full, [&](const std::vector<const void*>& peer) -> int {
      for (int r = 0; r < p->world; ++r) {
        if (r == p->rank) continue;
        TVR_CUDA(cudaMemcpyAsync(full + p->slab_off[r],
                                 static_cast<const float*>(peer[r]) + p->slab_off[r],
                                 sizeof(float) * p->slab_cnt[r], cudaMemcpyDeviceToDevice, p->stream));
      }
      return TVR_OK;
    });
  }
  if (uniform_slabs(p)) {
    TVR_NCCL(ncclAllGather(full + p->slab_off[p->rank], full, (size_t)p->slab_cnt[0], ncclFloat,
                           nccl_of(p), p->stream));
  } else {
    TVR_NCCL(ncclGroupStart());
    for (int r = 0; r < p->world; ++r) {
      float* dst = full + p->slab_off[r];
      TVR_NCCL(ncclBroadcast(dst, dst, (size_t)p->slab_cnt[r], ncclFloat, r, nccl_of(p), p->stream));
    }
    TVR_NCCL(ncclGroupEnd());
  }
  return TVR_OK;
}

// slab = sum over ranks of full[off_rank : off_rank + cnt_rank] (fp32 sums; each rank's partial
// A_p^T r_p already carries fp64-accumulated rows rounded once to fp32).  NCCL: equal slabs one
// ncclReduceScatter, ragged slabs one ncclReduce per rank; local backend: rank-order sum.
int reduce_scatter_volume(tvr_problem* p, const float* full, float* slab) {
  NvtxRange nv("views_reduce_scatter");
  if (local_of(p)) {
    const int64_t cnt = p->slab_cnt[p->rank], off = p->slab_off[p->rank];
    return local_collective(p, full, [&](const std::vector<const void*>& peer) -> int {
      TVR_CUDA(cudaMemcpyAsync(slab, static_cast<const float*>(peer[0]) + off, sizeof(float) * cnt,
                               cudaMemcpyDeviceToDevice, p->stream));
      for (int r = 1; r < p->world; ++r)
        TVR_CUDA(launch_add_inplace(cnt, static_cast<const float*>(peer[r]) + off, slab, p->stream));
      return TVR_OK;
    });
  }
  if (uniform_slabs(p)) {
    TVR_NCCL(ncclReduceScatter(full, slab, (size_t)p->slab_cnt[0], ncclFloat, ncclSum, nccl_of(p),
                               p->stream));
  } else {
    TVR_NCCL(ncclGroupStart());
    for (int r = 0; r < p->world; ++r) {
      const float* src = full + p->slab_off[r];
      TVR_NCCL(ncclReduce(src, r == p->rank ? (void*)slab : (void*)src, (size_t)p->slab_cnt[r],
                          ncclFloat, ncclSum, r, nccl_of(p), p->stream));
    }
    TVR_NCCL(ncclGroupEnd());
  }
  return TVR_OK;
}

// Stream-ordered barrier: on return every rank's work enqueued before the barrier is complete
// (NCCL: a one-int all-reduce on the stream; local: stream sync + host barrier).
int dist_barrier(tvr_problem* p) {
  if (p->world <= 1) return TVR_OK;
  if (LocalComm* L = local_of(p)) {
    TVR_CUDA(cudaStreamSynchronize(p->stream));
    L->barrier();
    return TVR_OK;
  }
  TVR_NCCL(ncclAllReduce(p->barrier_dev, p->barrier_dev, 1, ncclInt, ncclSum, nccl_of(p), p->stream));
  return TVR_OK;
}

// Fused reduce-scatter of the VIEWS A^T pass: every rank owns an inbox with
// one slot per rank; the A^T kernel of rank q stores row i (global voxel) into slot q of the
// inbox of i's owner, directly through peer memory (NVLink), so the transfer happens inside the
// kernel, row by row; the owner then sums its slots in rank order.  Pointers: local backend
// from the shared process; NCCL backend via CUDA IPC handles all-gathered over NCCL.
int setup_fused_rs(tvr_problem* p) {
  const int W = p->world;
  int64_t stride = 0;
  for (int r = 0; r < W; ++r) stride = std::max(stride, p->slab_cnt[r]);
  p->inbox_stride = stride;
  const size_t inbox_bytes = sizeof(float) * (size_t)stride * W;
  if (local_of(p)) {
    TVR_TRY(dev_alloc(p, (void**)&p->inbox, inbox_bytes));
  } else {
    // CUDA IPC maps a whole allocation and returns its base address, so the inbox must be an
    // allocation of its own (never a sub-block of a caching-allocator segment): raw cudaMalloc
    if (cudaMalloc((void**)&p->inbox, inbox_bytes) != cudaSuccess) {
      cudaGetLastError();
      p->inbox = nullptr;
      set_error("fused RS: inbox allocation failed");
      return TVR_E_OOM;
    }
    p->inbox_raw = true;
  }
  TVR_TRY(dev_alloc(p, (void**)&p->barrier_dev, 64));
  TVR_CUDA(cudaMemsetAsync(p->barrier_dev, 0, 64, p->stream));
  std::vector<float*> base(W, nullptr);
  if (LocalComm* L = local_of(p)) {
    TVR_CUDA(cudaStreamSynchronize(p->stream));
    L->ptr[p->rank] = p->inbox;
    L->barrier();
    for (int r = 0; r < W; ++r) base[r] = (float*)L->ptr[r];
    L->barrier();
  } else {
    cudaIpcMemHandle_t mine;
    TVR_CUDA(cudaIpcGetMemHandle(&mine, p->inbox));
    char* d = nullptr;
    TVR_CUDA(cudaMalloc(&d, sizeof(cudaIpcMemHandle_t) * (W + 1)));
    std::vector<cudaIpcMemHandle_t> all(W);
    cudaError_t e = cudaMemcpyAsync(d, &mine, sizeof(mine), cudaMemcpyHostToDevice, p->stream);
    ncclResult_t nr = ncclSuccess;
    if (e == cudaSuccess)
      nr = ncclAllGather(d, d + sizeof(mine), sizeof(mine), ncclChar, nccl_of(p), p->stream);
    if (e == cudaSuccess && nr == ncclSuccess)
      e = cudaMemcpyAsync(all.data(), d + sizeof(mine), sizeof(mine) * W, cudaMemcpyDeviceToHost,
                          p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    cudaFree(d);
    if (nr != ncclSuccess) { set_error(std::string("fused RS: ") + ncclGetErrorString(nr)); return TVR_E_NCCL; }
    if (e != cudaSuccess) { set_error(std::string("fused RS: ") + cudaGetErrorString(e)); return TVR_E_CUDA; }
    int ok = 1;
    for (int r = 0; r < W && ok; ++r) {
      if (r == p->rank) { base[r] = p->inbox; continue; }
      void* q = nullptr;
      if (cudaIpcOpenMemHandle(&q, all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      p->ipc_opened.push_back(q);
      base[r] = (float*)q;
    }
    // every rank must take the same path: the fused mode only if all ranks mapped all peers
    int* flag = p->barrier_dev + 1;
    TVR_CUDA(cudaMemcpyAsync(flag, &ok, sizeof(int), cudaMemcpyHostToDevice, p->stream));
    TVR_NCCL(ncclAllReduce(flag, flag, 1, ncclInt, ncclMin, nccl_of(p), p->stream));
    TVR_CUDA(cudaMemcpyAsync(&ok, flag, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
    TVR_CUDA(cudaStreamSynchronize(p->stream));
    if (!ok) {  // no peer mapping somewhere: keep the NCCL reduce-scatter
      dist_release(p);
      return TVR_OK;
    }
  }
  // store target for owner o: slot `rank` of o's inbox, shifted so the global row indexes it
  std::vector<float*> tgt(W);
  std::vector<int64_t> bounds(W + 1);
  for (int o = 0; o < W; ++o) {
    tgt[o] = base[o] + (int64_t)p->rank * stride - p->slab_off[o];
    bounds[o] = p->slab_off[o];
  }
  bounds[W] = p->slab_off[W - 1] + p->slab_cnt[W - 1];
  TVR_TRY(dev_alloc(p, (void**)&p->out_peer_dev, sizeof(float*) * W));
  TVR_TRY(dev_alloc(p, (void**)&p->out_bounds_dev, sizeof(int64_t) * (W + 1)));
  TVR_CUDA(cudaMemcpyAsync(p->out_peer_dev, tgt.data(), sizeof(float*) * W, cudaMemcpyHostToDevice,
                           p->stream));
  TVR_CUDA(cudaMemcpyAsync(p->out_bounds_dev, bounds.data(), sizeof(int64_t) * (W + 1),
                           cudaMemcpyHostToDevice, p->stream));
  TVR_CUDA(cudaStreamSynchronize(p->stream));
  p->fused_rs = true;
  return TVR_OK;
}

void dist_release(tvr_problem* p) {
  for (void* q : p->ipc_opened) cudaIpcCloseMemHandle(q);
  p->ipc_opened.clear();
  if (p->inbox_raw && p->inbox) cudaFree(p->inbox);
  if (p->inbox_raw) p->inbox = nullptr;
  p->inbox_raw = false;
  p->fused_rs = false;
}

}  // namespace tvr

using namespace tvr;

extern "C" {

int tvr_rank_sum(const double* gathered_dev, int world, int n, double* out_dev, void* cuda_stream) {
  if (!gathered_dev || !out_dev || world < 1 || n < 1) { set_error("tvr_rank_sum: bad arguments"); return TVR_E_ARG; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  rank_sum_kernel<<<(n + 63) / 64, 64, 0, st>>>(gathered_dev, world, n, out_dev);
  TVR_CUDA(cudaGetLastError());
  TVR_CUDA(cudaStreamSynchronize(st));
  return TVR_OK;
}

int tvr_nccl_unique_id_size(void) { return (int)sizeof(ncclUniqueId); }

int tvr_nccl_get_unique_id(void* id_out) {
  if (!id_out) { set_error("tvr_nccl_get_unique_id: NULL"); return TVR_E_ARG; }
  ncclUniqueId id;
  TVR_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return TVR_OK;
}

int tvr_nccl_comm_init(void** comm_out, const void* id, int world, int rank, int device) {
  if (!comm_out || !id || world < 1 || rank < 0 || rank >= world) {
    set_error("tvr_nccl_comm_init: bad argument");
    return TVR_E_ARG;
  }
  if (device >= 0) TVR_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  TVR_NCCL(ncclCommInitRank(&comm, world, uid, rank));
  auto* h = new NcclComm();
  h->magic = kNcclMagic;
  h->c = comm;
  *comm_out = h;
  return TVR_OK;
}

int tvr_nccl_comm_destroy(void* comm) {
  if (!comm) return TVR_OK;
  auto* h = static_cast<NcclComm*>(comm);
  if (h->magic != kNcclMagic) { set_error("tvr_nccl_comm_destroy: not an NCCL communicator"); return TVR_E_ARG; }
  const ncclResult_t r = ncclCommDestroy(h->c);
  h->magic = 0;
  delete h;
  if (r != ncclSuccess) { set_error(std::string("ncclCommDestroy: ") + ncclGetErrorString(r)); return TVR_E_NCCL; }
  return TVR_OK;
}

int tvr_local_comm_create(void** comm_out, int world) {
  if (!comm_out || world < 1) { set_error("tvr_local_comm_create: bad argument"); return TVR_E_ARG; }
  auto* L = new LocalComm();
  L->magic = kLocalMagic;
  L->world = world;
  L->ptr.assign(world, nullptr);
  L->val.assign(2 * world, 0);
  *comm_out = L;
  return TVR_OK;
}

int tvr_local_comm_destroy(void* comm) {
  if (!comm) return TVR_OK;
  auto* L = static_cast<LocalComm*>(comm);
  if (L->magic != kLocalMagic) { set_error("tvr_local_comm_destroy: not a local communicator"); return TVR_E_ARG; }
  L->magic = 0;
  delete L;
  return TVR_OK;
}

}  // extern "C"
