// dev.cuh — device helpers shared by the libdfvm kernels: grid sizing,
// warp-per-SELL-slice iteration, deterministic two-level reductions.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <cuda_runtime.h>

#include "internal.h"

namespace dfvm {

// Programmatic dependent launch: inside the captured Krylov
// graphs the edges between consecutive kernel nodes are made programmatic
// (solver.cu make_programmatic), so a kernel's blocks may become resident
// while its predecessor is still running.  Every kernel therefore starts by
// waiting for the completion and memory of the grids it depends on
// (griddepcontrol.wait; a no-op for a kernel launched without a programmatic
// dependency) — nothing is read or written before it.
#define PDL_ENTRY() asm volatile("griddepcontrol.wait;" ::: "memory")

constexpr int kThreads = 256;          // 8 warps per block
constexpr int kWarpsPerBlock = kThreads / 32;
constexpr int kMaxBlocks = 148 * 8;    // one full wave of 256-thread blocks on 148 SMs

// Debug / coverage knob DFVM_MAX_BLOCKS=k (read once): caps every
// grid-stride launch at k blocks, so small parity meshes exercise the
// multi-slice-per-warp loops (and their next-slice prefetch) that only the
// full-size meshes reach otherwise.  Unset (default): no cap beyond one wave.
inline int grid_cap() {
  static const int cap = [] {
    const char* e = getenv("DFVM_MAX_BLOCKS");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : kMaxBlocks;
  }();
  return cap;
}
inline int grid_for_slices(int n_slices) {
  int b = (n_slices + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int mx = kMaxBlocks < grid_cap() ? kMaxBlocks : grid_cap();
  return b < 1 ? 1 : (b > mx ? mx : b);
}
inline int grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  const int mx = kMaxBlocks < grid_cap() ? kMaxBlocks : grid_cap();
  return (int)(b < 1 ? 1 : (b > mx ? mx : b));
}

// Resident-block cap of a kernel: (blocks per SM from the occupancy API) x
// (SM count), so a grid-stride kernel runs as exactly one full wave.  Cached
// per kernel; a fixed function of (kernel, device), so the reduction
// structure (and hence the bits) stays deterministic run to run.
inline int occ_cap(const void* fn) {
  // guarded: the in-process multi-rank path calls this from several host threads
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  int dev = 0, nsm = 148, b = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, 0) != cudaSuccess || b < 1) b = 1;
  int cap = b * nsm < kMaxBlocks ? b * nsm : kMaxBlocks;
  if (cap > grid_cap()) cap = grid_cap();
  cache[fn] = cap;
  return cap;
}
template <class K> inline int grid_slices(K fn, int n_slices) {
  const int need = (n_slices + kWarpsPerBlock - 1) / kWarpsPerBlock, cap = occ_cap((const void*)fn);
  return need < 1 ? 1 : (need > cap ? cap : need);
}
template <class K> inline int grid_rows(K fn, int64_t n) {
  const int64_t need = (n + kThreads - 1) / kThreads;
  const int cap = occ_cap((const void*)fn);
  return (int)(need < 1 ? 1 : (need > cap ? cap : need));
}

// Timing event on a stream that may be capturing into a CUDA graph: inside a
// capture the record must be an external event node (else it is only a
// capture dependency and never fires on replay); outside a capture a plain
// record (the external flag is an error there).
inline cudaError_t record_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                                             : cudaEventRecord(ev, s);
}

template <class T> __device__ __forceinline__ V4<T> ld4(const V4<T>* p);
// fp64 records (32 B, 32-B aligned) in ONE 256-bit load (sm_100: LDG.E.ENL2.256):
// a gathered face record costs one L1 request instead of two 128-bit ones —
// the gather kernels are bound by L1 requests, not DRAM bytes (ncu)
template <> __device__ __forceinline__ V4<double> ld4<double>(const V4<double>* p) {
  V4<double> r;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
template <> __device__ __forceinline__ V4<float> ld4<float>(const V4<float>* p) {
  float4 a = __ldg(reinterpret_cast<const float4*>(p));
  return V4<float>{a.x, a.y, a.z, a.w};
}

// A {a, b} pair stored 2-aligned (fp64 16 B / fp32 8 B): one load
template <class T> __device__ __forceinline__ void ld2(const T* p, T& a, T& b);
template <> __device__ __forceinline__ void ld2<double>(const double* p, double& a, double& b) {
  const double2 u = __ldg(reinterpret_cast<const double2*>(p));
  a = u.x; b = u.y;
}
template <> __device__ __forceinline__ void ld2<float>(const float* p, float& a, float& b) {
  const float2 u = __ldg(reinterpret_cast<const float2*>(p));
  a = u.x; b = u.y;
}

// Gather of a 3-vector from an AoS [n][3] array that is read-only during the
// kernel: two loads (one 128-bit, one 64-bit, by the 16-byte parity of the
// address) instead of three 64-bit ones — fewer L1 requests per gathered
// neighbour; never reads outside the 24-byte element.
template <class T> __device__ __forceinline__ void ld3(const T* p, T& a, T& b, T& c);
template <> __device__ __forceinline__ void ld3<double>(const double* p, double& a, double& b, double& c) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    const double2 u = __ldg(reinterpret_cast<const double2*>(p));
    a = u.x; b = u.y; c = __ldg(p + 2);
  } else {
    a = __ldg(p);
    const double2 u = __ldg(reinterpret_cast<const double2*>(p + 1));
    b = u.x; c = u.y;
  }
}
// fp32: one 64-bit + one 32-bit load by the 8-byte parity of the address
// (12-byte elements are 4-byte aligned)
template <> __device__ __forceinline__ void ld3<float>(const float* p, float& a, float& b, float& c) {
  if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) {
    const float2 u = __ldg(reinterpret_cast<const float2*>(p));
    a = u.x; b = u.y; c = __ldg(p + 2);
  } else {
    a = __ldg(p);
    const float2 u = __ldg(reinterpret_cast<const float2*>(p + 1));
    b = u.x; c = u.y;
  }
}

// Deterministic block + grid reduction of NV doubles.
// Every thread passes its partial values; block partials are written in
// block order, and the last block to arrive (atomic ticket) sums them in a
// fixed strided order followed by a fixed tree.  Returns true in thread 0 of
// the last block, with the grid totals in `out`.  The ticket is reset.
template <int NV>
__device__ __forceinline__ void warp_sum(double (&v)[NV]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_down_sync(0xffffffffu, v[i], o);
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*sh)[NV]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  warp_sum<NV>(v);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) sh[wid][i] = v[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NV; ++i) {
      double s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w][i];
      v[i] = s;
    }
  }
  __syncthreads();
}

template <int NV>
__device__ bool grid_sum(double (&v)[NV], double* partials, unsigned* ticket, double (&out)[NV]) {
  __shared__ double sh[32][NV];
  __shared__ bool last;
  block_sum<NV>(v, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[(size_t)blockIdx.x * NV + i] = v[i];
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double a[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) a[i] = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
    for (int i = 0; i < NV; ++i) a[i] += __ldcg(&partials[(size_t)b * NV + i]);
  block_sum<NV>(a, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = a[i];
    *ticket = 0;
  }
  return threadIdx.x == 0;
}

// max-reduction variant (for continuity), same structure
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace dfvm
