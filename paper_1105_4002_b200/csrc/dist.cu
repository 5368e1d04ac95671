// Distribution over NCCL.  Both modes: one-slice halo exchange with each
// z-neighbour (ncclSend/ncclRecv inside one group) and a rank-ordered fp64 scalar sum
// (ncclAllGather of the partial scalars, then a fixed-order sum on the host, so every rank
// sees bitwise-identical scalars and takes the same line-search / BT branch).
// Trial and momentum points never need a halo exchange: their halo planes are recomputed
// from the halo planes of their inputs with the stencil's own functors (bitwise equal to the
// neighbour's stored values); only gradients are exchanged.
// VIEWS mode (P2, non-separable geometry) adds an all-gather of the point before every A pass
// and a reduce-scatter of the full-volume A_p^T r_p after every A^T pass.
#include <nccl.h>

#include <cstring>
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

int halo_exchange(tvr_problem* p, float* v) {
  if (p->world <= 1) return TVR_OK;
  ncclComm_t comm = (ncclComm_t)p->comm;
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
  TVR_NCCL(ncclGroupEnd());
  return TVR_OK;
}

int halo_fill_trial(tvr_problem* p, const float* x, const float* g, double s, float* v) {
  if (p->world <= 1) return TVR_OK;
  TVR_CUDA(launch_halo_fill_trial(x, g, s, p->lo, p->hi, p->plane, p->nzl, p->z0 > 0,
                                  p->z1 < p->nz, v, p->stream));
  p->launches++;
  return TVR_OK;
}

int halo_fill_momentum(tvr_problem* p, const float* x1, const float* x0, double beta, float* y) {
  if (p->world <= 1) return TVR_OK;
  TVR_CUDA(launch_halo_fill_momentum(x1, x0, beta, p->plane, p->nzl, p->z0 > 0, p->z1 < p->nz, y,
                                     p->stream));
  p->launches++;
  return TVR_OK;
}

int dist_sum_scalars(tvr_problem* p, double* vals, int n) {
  ncclComm_t comm = (ncclComm_t)p->comm;
  TVR_NCCL(ncclAllGather(p->dscal, p->dgather, (size_t)n, ncclDouble, comm, p->stream));
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

// ---- VIEWS mode: rows split by projection views, volume vectors by z-slabs.
bool views_dist(const tvr_problem* p) { return p->mode == TVR_SHARD_VIEWS && p->world > 1; }

static bool uniform_slabs(const tvr_problem* p) {
  for (int r = 1; r < p->world; ++r)
    if (p->slab_cnt[r] != p->slab_cnt[0]) return false;
  return true;
}

// Every rank's slab [z0, z1), all-gathered once at create time; the slabs must tile [0, nz).
int views_slab_table(tvr_problem* p) {
  int64_t* d = nullptr;
  TVR_CUDA(cudaMalloc(&d, sizeof(int64_t) * 2 * (p->world + 1)));
  std::vector<int64_t> mine = {p->z0, p->z1}, all(2 * p->world);
  cudaError_t e = cudaMemcpyAsync(d, mine.data(), sizeof(int64_t) * 2, cudaMemcpyHostToDevice,
                                  p->stream);
  ncclResult_t nr = ncclSuccess;
  if (e == cudaSuccess)
    nr = ncclAllGather(d, d + 2, 2, ncclInt64, (ncclComm_t)p->comm, p->stream);
  if (e == cudaSuccess && nr == ncclSuccess)
    e = cudaMemcpyAsync(all.data(), d + 2, sizeof(int64_t) * 2 * p->world, cudaMemcpyDeviceToHost,
                        p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  cudaFree(d);
  if (nr != ncclSuccess) { set_error(std::string("slab table: ") + ncclGetErrorString(nr)); return TVR_E_NCCL; }
  if (e != cudaSuccess) { set_error(std::string("slab table: ") + cudaGetErrorString(e)); return TVR_E_CUDA; }
  p->slab_off.assign(p->world, 0);
  p->slab_cnt.assign(p->world, 0);
  for (int r = 0; r < p->world; ++r) {
    const int64_t z0 = all[2 * r], z1 = all[2 * r + 1];
    if (z0 != (r == 0 ? 0 : all[2 * r - 1]) || z1 <= z0 || (r == p->world - 1 && z1 != p->nz)) {
      set_error("tvr_create: VIEWS slabs must tile [0, nz) in rank order");
      return TVR_E_ARG;
    }
    p->slab_off[r] = z0 * p->plane;
    p->slab_cnt[r] = (z1 - z0) * p->plane;
  }
  return TVR_OK;
}

// x_full[off_r : off_r + cnt_r] = slab of rank r, on every rank (the A pass needs the whole
// point: a tilted ray crosses every slab).  Equal slabs: one ncclAllGather; ragged slabs: one
// broadcast per rank inside a group.
int gather_volume(tvr_problem* p, const float* slab, const float** full) {
  if (!views_dist(p)) {
    *full = slab;
    return TVR_OK;
  }
  ncclComm_t comm = (ncclComm_t)p->comm;
  if (uniform_slabs(p)) {
    TVR_NCCL(ncclAllGather(slab, p->xfull, (size_t)p->slab_cnt[0], ncclFloat, comm, p->stream));
  } else {
    TVR_NCCL(ncclGroupStart());
    for (int r = 0; r < p->world; ++r) {
      float* dst = p->xfull + p->slab_off[r];
      TVR_NCCL(ncclBroadcast(r == p->rank ? (const void*)slab : (const void*)dst, dst,
                             (size_t)p->slab_cnt[r], ncclFloat, r, comm, p->stream));
    }
    TVR_NCCL(ncclGroupEnd());
  }
  *full = p->xfull;
  return TVR_OK;
}

// slab = sum over ranks of full[off_rank : off_rank + cnt_rank] (fp32 sum inside NCCL; each
// rank's partial A_p^T r_p already carries fp64-accumulated rows rounded once to fp32).
int reduce_scatter_volume(tvr_problem* p, const float* full, float* slab) {
  ncclComm_t comm = (ncclComm_t)p->comm;
  if (uniform_slabs(p)) {
    TVR_NCCL(ncclReduceScatter(full, slab, (size_t)p->slab_cnt[0], ncclFloat, ncclSum, comm,
                               p->stream));
  } else {
    TVR_NCCL(ncclGroupStart());
    for (int r = 0; r < p->world; ++r) {
      const float* src = full + p->slab_off[r];
      TVR_NCCL(ncclReduce(src, r == p->rank ? (void*)slab : (void*)src, (size_t)p->slab_cnt[r],
                          ncclFloat, ncclSum, r, comm, p->stream));
    }
    TVR_NCCL(ncclGroupEnd());
  }
  return TVR_OK;
}

}  // namespace tvr

using namespace tvr;

extern "C" {

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
  *comm_out = (void*)comm;
  return TVR_OK;
}

int tvr_nccl_comm_destroy(void* comm) {
  if (!comm) return TVR_OK;
  TVR_NCCL(ncclCommDestroy((ncclComm_t)comm));
  return TVR_OK;
}

}  // extern "C"
