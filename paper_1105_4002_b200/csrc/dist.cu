// z-slab distribution over NCCL: one-slice halo exchange with each
// z-neighbour (ncclSend/ncclRecv inside one group) and a rank-ordered fp64 scalar sum
// (ncclAllGather of the partial scalars, then a fixed-order sum on the host, so every rank
// sees bitwise-identical scalars and takes the same line-search / BT branch).
// Trial and momentum points never need a halo exchange: their halo planes are recomputed
// from the halo planes of their inputs with the stencil's own functors (bitwise equal to the
// neighbour's stored values); only gradients are exchanged.
#include <nccl.h>

#include <cstring>
#include <string>

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
