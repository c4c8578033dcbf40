// dev.cuh — device helpers shared by the libdfvm kernels: grid sizing,
// warp-per-SELL-slice iteration, deterministic two-level reductions.
#pragma once
#include <cstdint>
#include <unordered_map>
#include <cuda_runtime.h>

#include "internal.h"

namespace dfvm {

constexpr int kThreads = 256;          // 8 warps per block
constexpr int kWarpsPerBlock = kThreads / 32;
constexpr int kMaxBlocks = 148 * 8;    // one full wave of 256-thread blocks on 148 SMs

inline int grid_for_slices(int n_slices) {
  int b = (n_slices + kWarpsPerBlock - 1) / kWarpsPerBlock;
  return b < 1 ? 1 : (b > kMaxBlocks ? kMaxBlocks : b);
}
inline int grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  return (int)(b < 1 ? 1 : (b > kMaxBlocks ? kMaxBlocks : b));
}

// Resident-block cap of a kernel: (blocks per SM from the occupancy API) x
// (SM count), so a grid-stride kernel runs as exactly one full wave.  Cached
// per kernel; a fixed function of (kernel, device), so the reduction
// structure (and hence the bits) stays deterministic run to run.
inline int occ_cap(const void* fn) {
  static std::unordered_map<const void*, int> cache;
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  int dev = 0, nsm = 148, b = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, 0) != cudaSuccess || b < 1) b = 1;
  const int cap = b * nsm < kMaxBlocks ? b * nsm : kMaxBlocks;
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

template <class T> __device__ __forceinline__ V4<T> ld4(const V4<T>* p);
template <> __device__ __forceinline__ V4<double> ld4<double>(const V4<double>* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldg(q), b = __ldg(q + 1);
  return V4<double>{a.x, a.y, b.x, b.y};
}
template <> __device__ __forceinline__ V4<float> ld4<float>(const V4<float>* p) {
  float4 a = __ldg(reinterpret_cast<const float4*>(p));
  return V4<float>{a.x, a.y, a.z, a.w};
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
