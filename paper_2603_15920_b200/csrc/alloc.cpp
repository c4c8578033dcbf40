// alloc.cpp — device workspace allocation of libdfvm (SURVEY.md §8(b) row b3:
// "workspace comes from an optional caller allocator callback (so the torch
// caching allocator can be plugged in), else cudaMallocAsync").
//
// Every device buffer the library owns (mesh arrays, boundary values,
// library-owned fields, solver and AMG workspace, halo buffers, the
// import/export staging buffer) is obtained here.  Allocation and zero-fill
// are stream-ordered on the stream passed in (the caller's stream for lazy
// allocations inside a compute call; the legacy stream, followed by a
// synchronisation, for allocations made by *_create calls), so a buffer is
// never touched by a kernel on a non-blocking stream before its memset has
// completed.
#include <mutex>
#include <unordered_map>

#include "internal.h"

namespace dfvm {

namespace {
struct Allocator {
  dfvm_alloc_fn alloc = nullptr;
  dfvm_free_fn free_ = nullptr;
  void* ctx = nullptr;
};
std::mutex g_mu;
Allocator g_alloc;
std::unordered_map<void*, size_t>& live() {
  static std::unordered_map<void*, size_t> m;
  return m;
}
int64_t g_live_bytes = 0;
}  // namespace

dfvm_status dev_alloc(void** p, size_t bytes, cudaStream_t s, bool zero) {
  *p = nullptr;
  if (bytes == 0) bytes = 1;
  Allocator a;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    a = g_alloc;
  }
  void* q = nullptr;
  if (a.alloc) {
    q = a.alloc(bytes, (dfvm_stream)s, a.ctx);
    if (!q) {
      set_error(DFVM_E_OOM, "caller allocator returned NULL for " + std::to_string(bytes) + " bytes");
      return DFVM_E_OOM;
    }
  } else {
    DFVM_CUDA(cudaMallocAsync(&q, bytes, s));
  }
  if (zero) {
    cudaError_t e = cudaMemsetAsync(q, 0, bytes, s);
    if (e != cudaSuccess) {
      dev_free(q, s);
      return cuda_error(e, "cudaMemsetAsync(workspace)");
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_mu);
    live()[q] = bytes;
    g_live_bytes += (int64_t)bytes;
  }
  *p = q;
  return DFVM_OK;
}

void dev_free(void* p, cudaStream_t s) {
  if (!p) return;
  size_t bytes = 0;
  Allocator a;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = live().find(p);
    if (it == live().end()) return;   // not ours (never free foreign memory)
    bytes = it->second;
    live().erase(it);
    g_live_bytes -= (int64_t)bytes;
    a = g_alloc;
  }
  if (a.free_) a.free_(p, bytes, (dfvm_stream)s, a.ctx);
  else cudaFreeAsync(p, s);
}

int64_t dev_live_bytes() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_live_bytes;
}

}  // namespace dfvm

using namespace dfvm;

extern "C" {

dfvm_status dfvm_set_allocator(dfvm_alloc_fn alloc, dfvm_free_fn free_, void* ctx) {
  if ((alloc == nullptr) != (free_ == nullptr)) {
    set_error(DFVM_E_INVALID_ARG, "dfvm_set_allocator needs both callbacks (or both NULL for the default)");
    return DFVM_E_INVALID_ARG;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  if (!live().empty()) {
    set_error(DFVM_E_INVALID_ARG, "dfvm_set_allocator called while " + std::to_string(live().size()) +
              " library allocations are live (destroy every mesh / field / solver first)", (int64_t)live().size());
    return DFVM_E_INVALID_ARG;
  }
  g_alloc.alloc = alloc;
  g_alloc.free_ = free_;
  g_alloc.ctx = ctx;
  return DFVM_OK;
}

int64_t dfvm_live_device_bytes(void) { return dev_live_bytes(); }

}  // extern "C"
