// comm.cpp — multi-GPU plumbing.
//
// Two transports behind one interface:
//  * NCCL (production): communicator bootstrapped from a 128-byte unique id
//    the caller broadcasts with torch.distributed; one process per GPU over
//    NVLink / NVSwitch.
//  * local: n ranks as host threads of one process (any devices, including
//    all on one GPU), device-to-device copies with CUDA-event handshakes and
//    host barriers.  It runs the identical partitioned solver code path, so
//    the multi-rank logic (halo slices, rank-order reductions, Windkessel
//    shares, gauge ownership) is testable on a single B200.
//
// Halo: the owned cells adjacent to peer q are packed (send list, ascending
// new id) and land directly in q's contiguous ghost slice for this rank
// (ghosts are ordered by (peer, new id), §8(c) O-9 step 7): no unpack.
// Reductions that steer control flow are all-gathers of the per-rank
// partial totals followed by a fixed rank-order sum on every rank, so all
// ranks take bitwise-identical decisions.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"

namespace dfvm {

// in-process group shared by the rank threads
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long generation = 0;
  int refs = 0;
  // mailboxes: published per (src, dst) pointer; per-rank events
  std::vector<const void*> box;      // [n * n]
  std::vector<cudaEvent_t> posted;  // [n] recorded after the publisher's pack / kernel
  std::vector<cudaEvent_t> consumed; // [n] recorded after the rank's copies
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long g = generation;
    if (++arrived == n) { arrived = 0; ++generation; cv.notify_all(); }
    else cv.wait(lk, [&] { return generation != g; });
  }
};

}  // namespace dfvm

struct dfvm_comm {
  int backend = 0;   // 0 NCCL, 1 local
  ncclComm_t nccl = nullptr;
  dfvm::LocalGroup* grp = nullptr;
  int n_ranks = 1, rank = 0, device = 0;
};

namespace dfvm {

// NCCL is resolved lazily (dlopen) when the first NCCL communicator is
// created: the library has no link-time NCCL dependency, so loading it never
// shadows the NCCL build a host framework (torch) brings; dlopen of the
// soname returns the copy already loaded in the process.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};
static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
#define SYM(name, field) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name)); if (!a.field) return a;
    SYM("ncclGetUniqueId", GetUniqueId) SYM("ncclCommInitRank", CommInitRank) SYM("ncclCommDestroy", CommDestroy)
    SYM("ncclGroupStart", GroupStart) SYM("ncclGroupEnd", GroupEnd) SYM("ncclSend", Send) SYM("ncclRecv", Recv)
    SYM("ncclAllGather", AllGather) SYM("ncclGetErrorString", GetErrorString)
#undef SYM
    a.ok = true;
    return a;
  }();
  return api;
}

template <class T>
void launch_pack(T* buf, const T* x, const int32_t* idx, int64_t n, int nc, cudaStream_t s);

static dfvm_status nccl_error(ncclResult_t r, const char* where) {
  set_error(DFVM_E_NCCL, std::string(where) + ": " + (nccl().ok ? nccl().GetErrorString(r) : "libnccl.so.2 not loadable"));
  return DFVM_E_NCCL;
}
#define DFVM_NCCL(call)                                          \
  do {                                                           \
    ncclResult_t r_ = (call);                                    \
    if (r_ != ncclSuccess) return nccl_error(r_, #call);         \
  } while (0)

dfvm_status halo_exchange_p(dfvm_mesh* m, void* data, int nc, bool f64, cudaStream_t s);

// local transport: every rank publishes, all wait for everybody's data,
// copy, then wait until every peer has consumed before the published
// buffers may be overwritten by the next stream operation.
static dfvm_status local_finish(LocalGroup* G, int rank, cudaStream_t s) {
  DFVM_CUDA(cudaEventRecord(G->consumed[rank], s));
  G->barrier();
  for (int q = 0; q < G->n; ++q)
    if (q != rank) DFVM_CUDA(cudaStreamWaitEvent(s, G->consumed[q], 0));
  G->barrier();
  return DFVM_OK;
}

// Halo of one partitioned vector space (level 0: the mesh's cells; AMG
// coarse levels: their aggregates): owned rows [0, n_own), ghosts in
// contiguous per-peer slices ordered by the owner's local index; the send
// list to peer q (owned rows, ascending) is q's ghost slice for this rank in
// the same order, so a receive lands directly in the slice (no unpack).
dfvm_status halo_exchange_lists(dfvm_mesh* m, HaloLists& L, void* data, int nc, bool f64, cudaStream_t s) {
  if (m->part.P == 1 || L.peers.empty()) return DFVM_OK;
  if (!m->comm) { set_error(DFVM_E_NCCL, "multi-part mesh without communicator"); return DFVM_E_NCCL; }
  const size_t eb = f64 ? 8 : 4;
  const int64_t ns = L.send_off.back();
  if (!L.d_send_idx && ns) {
    dfvm_status st;
    if ((st = dev_alloc_n(&L.d_send_idx, (size_t)ns, nullptr, false))) return st;
    DFVM_CUDA(cudaMemcpy(L.d_send_idx, L.send_idx.data(), (size_t)ns * 4, cudaMemcpyHostToDevice));
    L.buf_bytes = (size_t)ns * 9 * 8;   // up to 9 fp64 components
    if ((st = dev_alloc(&L.d_send, L.buf_bytes, nullptr, false))) return st;
    DFVM_CUDA(cudaStreamSynchronize(nullptr));   // once: ordered before the caller's (non-blocking) stream uses them
  }
  if (ns) {
    if (f64) launch_pack<double>((double*)L.d_send, (const double*)data, L.d_send_idx, ns, nc, s);
    else launch_pack<float>((float*)L.d_send, (const float*)data, L.d_send_idx, ns, nc, s);
  }
  dfvm_comm* C = m->comm;
  if (C->backend == 0) {
    const ncclDataType_t dt = f64 ? ncclFloat64 : ncclFloat32;
    DFVM_NCCL(nccl().GroupStart());
    for (size_t i = 0; i < L.peers.size(); ++i) {
      const int q = L.peers[i];
      const int64_t so = L.send_off[i], sn = L.send_off[i + 1] - so;
      const int64_t go = L.ghost_off[i], gn = L.ghost_off[i + 1] - go;
      DFVM_NCCL(nccl().Send((const char*)L.d_send + so * nc * eb, (size_t)(sn * nc), dt, q, C->nccl, s));
      DFVM_NCCL(nccl().Recv((char*)data + (L.n_own + go) * nc * eb, (size_t)(gn * nc), dt, q, C->nccl, s));
    }
    DFVM_NCCL(nccl().GroupEnd());
    return DFVM_OK;
  }
  LocalGroup* G = C->grp;
  const int me = C->rank;
  for (size_t i = 0; i < L.peers.size(); ++i)
    G->box[(size_t)me * G->n + L.peers[i]] = (const char*)L.d_send + L.send_off[i] * nc * eb;
  DFVM_CUDA(cudaEventRecord(G->posted[me], s));
  G->barrier();
  for (size_t i = 0; i < L.peers.size(); ++i) {
    const int q = L.peers[i];
    const int64_t go = L.ghost_off[i], gn = L.ghost_off[i + 1] - go;
    DFVM_CUDA(cudaStreamWaitEvent(s, G->posted[q], 0));
    DFVM_CUDA(cudaMemcpyAsync((char*)data + (L.n_own + go) * nc * eb, G->box[(size_t)q * G->n + me],
                              (size_t)(gn * nc) * eb, cudaMemcpyDeviceToDevice, s));
  }
  return local_finish(G, me, s);
}

static void ensure_mesh_halo(dfvm_mesh* m) {
  HaloLists& L = m->halo0;
  if (L.ready) return;
  const Part& P = m->part;
  L.n_own = P.n_own;
  L.peers = P.peers;
  L.send_off = P.peer_send_off;
  L.ghost_off = P.peer_ghost_off;
  L.send_idx.resize(P.send_gid.size());
  for (size_t i = 0; i < P.send_gid.size(); ++i) L.send_idx[i] = (int32_t)(P.send_gid[i] - P.lo);
  L.ready = true;
}

dfvm_status halo_exchange(dfvm_mesh* m, void* data, int nc, cudaStream_t s) {
  return halo_exchange_p(m, data, nc, m->precision == DFVM_F64, s);
}

// element type given explicitly (f64 or f32), e.g. the fp32 AMG hierarchy of
// an fp64 solver; the send buffer is sized for 9 fp64 components
dfvm_status halo_exchange_p(dfvm_mesh* m, void* data, int nc, bool f64, cudaStream_t s) {
  if (m->part.P == 1) return DFVM_OK;
  ensure_mesh_halo(m);
  return halo_exchange_lists(m, m->halo0, data, nc, f64, s);
}

bool comm_is_local(const dfvm_comm* c) { return c && c->backend == 1; }

// all-gather of `n` doubles per rank into gathered[n_ranks][n] (rank order)
dfvm_status allgather_f64(dfvm_mesh* m, const double* local, double* gathered, int n, cudaStream_t s) {
  if (m->part.P == 1) {
    if (local != gathered) DFVM_CUDA(cudaMemcpyAsync(gathered, local, n * 8, cudaMemcpyDeviceToDevice, s));
    return DFVM_OK;
  }
  dfvm_comm* C = m->comm;
  if (C->backend == 0) {
    DFVM_NCCL(nccl().AllGather(local, gathered, (size_t)n, ncclFloat64, C->nccl, s));
    return DFVM_OK;
  }
  LocalGroup* G = C->grp;
  const int me = C->rank;
  G->box[(size_t)me * G->n + me] = local;
  DFVM_CUDA(cudaEventRecord(G->posted[me], s));
  G->barrier();
  for (int q = 0; q < G->n; ++q) {
    if (q != me) DFVM_CUDA(cudaStreamWaitEvent(s, G->posted[q], 0));
    DFVM_CUDA(cudaMemcpyAsync(gathered + (size_t)q * n, G->box[(size_t)q * G->n + q], n * 8,
                              cudaMemcpyDeviceToDevice, s));
  }
  return local_finish(G, me, s);
}

}  // namespace dfvm

using namespace dfvm;

extern "C" {

dfvm_status dfvm_comm_unique_id(uint8_t id[128]) {
  ncclUniqueId u;
  if (!nccl().ok) return nccl_error(ncclSystemError, "dlopen(libnccl.so.2)");
  DFVM_NCCL(nccl().GetUniqueId(&u));
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
  if (!nccl().ok) { delete c; return nccl_error(ncclSystemError, "dlopen(libnccl.so.2)"); }
  ncclResult_t r = nccl().CommInitRank(&c->nccl, n_ranks, u, rank);
  if (r != ncclSuccess) { delete c; return nccl_error(r, "ncclCommInitRank"); }
  *out = c;
  return DFVM_OK;
}

dfvm_status dfvm_comm_create_local(int n_ranks, const int* devices, dfvm_comm** out) {
  if (!out || n_ranks < 1) { set_error(DFVM_E_INVALID_ARG, "bad local communicator arguments"); return DFVM_E_INVALID_ARG; }
  LocalGroup* G = new LocalGroup();
  G->n = n_ranks;
  G->refs = n_ranks;
  G->box.assign((size_t)n_ranks * n_ranks, nullptr);
  G->posted.resize(n_ranks);
  G->consumed.resize(n_ranks);
  for (int r = 0; r < n_ranks; ++r) {
    DFVM_CUDA(cudaSetDevice(devices ? devices[r] : 0));
    DFVM_CUDA(cudaEventCreateWithFlags(&G->posted[r], cudaEventDisableTiming));
    DFVM_CUDA(cudaEventCreateWithFlags(&G->consumed[r], cudaEventDisableTiming));
    dfvm_comm* c = new dfvm_comm();
    c->backend = 1; c->grp = G; c->n_ranks = n_ranks; c->rank = r; c->device = devices ? devices[r] : 0;
    out[r] = c;
  }
  return DFVM_OK;
}

dfvm_status dfvm_comm_destroy(dfvm_comm* c) {
  if (!c) return DFVM_OK;
  if (c->nccl) nccl().CommDestroy(c->nccl);
  if (c->grp && --c->grp->refs == 0) {
    for (auto e : c->grp->posted) cudaEventDestroy(e);
    for (auto e : c->grp->consumed) cudaEventDestroy(e);
    delete c->grp;
  }
  delete c;
  return DFVM_OK;
}

}  // extern "C"
