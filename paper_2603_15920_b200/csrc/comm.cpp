// comm.cpp — multi-GPU plumbing: NCCL communicator
// bootstrap (unique id broadcast by the caller through torch.distributed),
// halo exchange of ghost cells and deterministic all-gather reductions.
//
// Halo: the owned cells adjacent to peer q are packed (send list, ascending
// new id) and sent; the receive lands directly in the contiguous ghost slice
// of q (ghosts are ordered by (peer, new id), §8(c) O-9 step 7), so there is
// no unpack kernel.  Reductions that steer control flow use ncclAllGather of
// the per-rank partials followed by a fixed rank-order sum on every rank, so
// every rank sees bitwise-identical Krylov scalars.
#include <nccl.h>

#include <cstring>
#include <vector>

#include "internal.h"

struct dfvm_comm {
  ncclComm_t nccl = nullptr;
  int n_ranks = 1, rank = 0, device = 0;
};

namespace dfvm {

template <class T>
void launch_pack(T* buf, const T* x, const int32_t* idx, int64_t n, int nc, cudaStream_t s);

static dfvm_status nccl_error(ncclResult_t r, const char* where) {
  set_error(DFVM_E_NCCL, std::string(where) + ": " + ncclGetErrorString(r));
  return DFVM_E_NCCL;
}
#define DFVM_NCCL(call)                                          \
  do {                                                           \
    ncclResult_t r_ = (call);                                    \
    if (r_ != ncclSuccess) return nccl_error(r_, #call);         \
  } while (0)

static dfvm_status ensure_halo_buffers(dfvm_mesh* m) {
  const Part& P = m->part;
  if (m->d_send_idx || P.send_gid.empty()) return DFVM_OK;
  std::vector<int32_t> idx(P.send_gid.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int32_t)(P.send_gid[i] - P.lo);
  DFVM_CUDA(cudaMalloc(&m->d_send_idx, idx.size() * 4));
  DFVM_CUDA(cudaMemcpy(m->d_send_idx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice));
  m->halo_bytes = idx.size() * 9 * 8;   // up to 9 fp64 components
  DFVM_CUDA(cudaMalloc(&m->d_send, m->halo_bytes));
  return DFVM_OK;
}

dfvm_status halo_exchange(dfvm_mesh* m, void* data, int nc, cudaStream_t s) {
  const Part& P = m->part;
  if (P.P == 1 || P.peers.empty()) return DFVM_OK;
  if (!m->comm) { set_error(DFVM_E_NCCL, "multi-part mesh without communicator"); return DFVM_E_NCCL; }
  if (dfvm_status st = ensure_halo_buffers(m)) return st;
  const bool f64 = m->precision == DFVM_F64;
  const size_t eb = f64 ? 8 : 4;
  const int64_t ns = (int64_t)P.send_gid.size();
  if (f64) launch_pack<double>((double*)m->d_send, (const double*)data, m->d_send_idx, ns, nc, s);
  else launch_pack<float>((float*)m->d_send, (const float*)data, m->d_send_idx, ns, nc, s);
  const ncclDataType_t dt = f64 ? ncclFloat64 : ncclFloat32;
  DFVM_NCCL(ncclGroupStart());
  for (size_t i = 0; i < P.peers.size(); ++i) {
    const int q = P.peers[i];
    const int64_t so = P.peer_send_off[i], sn = P.peer_send_off[i + 1] - so;
    const int64_t go = P.peer_ghost_off[i], gn = P.peer_ghost_off[i + 1] - go;
    DFVM_NCCL(ncclSend((const char*)m->d_send + so * nc * eb, (size_t)(sn * nc), dt, q, m->comm->nccl, s));
    DFVM_NCCL(ncclRecv((char*)data + (P.n_own + go) * nc * eb, (size_t)(gn * nc), dt, q, m->comm->nccl, s));
  }
  DFVM_NCCL(ncclGroupEnd());
  return DFVM_OK;
}

// all-gather of `n` doubles per rank into gathered[n_ranks][n]
dfvm_status allgather_f64(dfvm_mesh* m, const double* local, double* gathered, int n, cudaStream_t s) {
  if (m->part.P == 1) {
    if (local != gathered) DFVM_CUDA(cudaMemcpyAsync(gathered, local, n * 8, cudaMemcpyDeviceToDevice, s));
    return DFVM_OK;
  }
  DFVM_NCCL(ncclAllGather(local, gathered, (size_t)n, ncclFloat64, m->comm->nccl, s));
  return DFVM_OK;
}

}  // namespace dfvm

using namespace dfvm;

extern "C" {

dfvm_status dfvm_comm_unique_id(uint8_t id[128]) {
  ncclUniqueId u;
  DFVM_NCCL(ncclGetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId must be 128 bytes");
  std::memcpy(id, &u, 128);
  return DFVM_OK;
}

dfvm_status dfvm_comm_create(int n_ranks, int rank, const uint8_t id[128], int device, dfvm_comm** out) {
  if (!out || !id || n_ranks < 1 || rank < 0 || rank >= n_ranks) {
    set_error(DFVM_E_INVALID_ARG, "bad communicator arguments");
    return DFVM_E_INVALID_ARG;
  }
  DFVM_CUDA(cudaSetDevice(device));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  dfvm_comm* c = new dfvm_comm();
  c->n_ranks = n_ranks; c->rank = rank; c->device = device;
  ncclResult_t r = ncclCommInitRank(&c->nccl, n_ranks, u, rank);
  if (r != ncclSuccess) { delete c; return nccl_error(r, "ncclCommInitRank"); }
  *out = c;
  return DFVM_OK;
}

dfvm_status dfvm_comm_destroy(dfvm_comm* c) {
  if (!c) return DFVM_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
  return DFVM_OK;
}

}  // extern "C"
