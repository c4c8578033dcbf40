// ops.cu — sm_100a kernels of the FVM operators (SURVEY.md §8(a) a6, and
// the north-star `fvm_grad/div/laplacian apply`).
//
// All cell operators are deterministic cell-gathers over the SELL-32
// incidence layout (internal.h): one warp handles 32 consecutive (RCM-
// ordered) rows, one thread per row, incidence k of the warp's rows is one
// coalesced 256-byte int2 load; face geometry records (32 B, fp64) and
// neighbour values are gathered through L2 (RCM keeps the two reads of a
// face within the bandwidth window).  No atomics: the per-cell sum runs over
// the row's incidences in ascending face order (P:297-305 eq:aggregate
// realised as a gather, reading A-20).
#include <cstdlib>
#include <cuda_runtime.h>

#include "dev.cuh"
#include "launch.h"

namespace dfvm {

// ----------------------------------------------------------- import/export
template <class T>
__global__ void k_import(T* __restrict__ dst, const double* __restrict__ src, const int32_t* __restrict__ map,
                         int64_t n, int nc, bool oriented) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t m = map[i];
    const bool neg = oriented && (m < 0);
    const int64_t o = m < 0 ? (int64_t)(~m) : m;
    for (int k = 0; k < nc; ++k) {
      const double v = src[o * nc + k];
      dst[i * nc + k] = (T)(neg ? -v : v);
    }
  }
}
template <class T>
__global__ void k_export(double* __restrict__ dst, const T* __restrict__ src, const int32_t* __restrict__ map,
                         int64_t n, int nc, bool oriented) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t m = map[i];
    const bool neg = oriented && (m < 0);
    const int64_t o = m < 0 ? (int64_t)(~m) : m;
    for (int k = 0; k < nc; ++k) {
      const double v = (double)src[i * nc + k];
      dst[o * nc + k] = neg ? -v : v;
    }
  }
}
template <class T>
void launch_import(T* dst, const double* src, const int32_t* map, int64_t n, int nc, bool oriented, cudaStream_t s) {
  if (n <= 0) return;
  k_import<T><<<grid_for(n), kThreads, 0, s>>>(dst, src, map, n, nc, oriented);
  count_launch();
}
template <class T>
void launch_export(double* dst, const T* src, const int32_t* map, int64_t n, int nc, bool oriented, cudaStream_t s) {
  if (n <= 0) return;
  k_export<T><<<grid_for(n), kThreads, 0, s>>>(dst, src, map, n, nc, oriented);
  count_launch();
}

// Gather kernels load their incidences in batches of kB: first the kB int2
// records of the row, then every face record / neighbour value they point
// to, then the arithmetic in ascending incidence order (the summation order
// of the one-at-a-time loop, so results are bitwise unchanged).  Each thread
// keeps ~kB x (record + value) independent loads in flight instead of a
// dependent chain per face.
constexpr int kB = 4;
// fp32 operator kernels at 6 resident blocks / SM (C5 fp32, round 2,
// tools/op_ab.py: grad_s 0.59 -> 0.78, grad_U 0.50 -> 0.61, Laplacian
// 0.48 -> 0.65 of the HBM peak; 8 blocks/SM or deeper batches lower;
// profiles/r02_ops_f32_variants_c5.json)
constexpr int kOpsF32Default = 1;

// ------------------------------------------------------------ interpolate
// phi_f = w phi_O + (1 - w) phi_N; boundary: fixed value or phi_O;
// empty faces: 0.  Face-parallel (coalesced over the face arrays); internal
// faces in batches of kB per thread.
template <class T, int NC>
__global__ void k_interp(DevMesh<T> M, const T* __restrict__ x, const uint8_t* __restrict__ bkind,
                         const T* __restrict__ bval, T* __restrict__ xf) {
  PDL_ENTRY();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = tid; i0 < M.F; i0 += kB * nt) {
    int2 c[kB];
    T w[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t i = i0 + u * nt;
      c[u] = i < M.F ? __ldg(&M.fcell[i]) : make_int2(0, 0);
      w[u] = i < M.F ? __ldg(&M.fw[i]) : T(0);
    }
    T xo[kB][NC], xn[kB][NC];
#pragma unroll
    for (int u = 0; u < kB; ++u)
#pragma unroll
      for (int k = 0; k < NC; ++k) { xo[u][k] = x[(int64_t)c[u].x * NC + k]; xn[u][k] = x[(int64_t)c[u].y * NC + k]; }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t i = i0 + u * nt;
      if (i < M.F)
#pragma unroll
        for (int k = 0; k < NC; ++k) xf[i * NC + k] = w[u] * xo[u][k] + (T(1) - w[u]) * xn[u][k];
    }
  }
  const int64_t nb = (int64_t)M.B + M.E;
  for (int64_t j = tid; j < nb; j += nt) {
    const int64_t i = M.F + j;
    if (j < M.B) {
      const int b = (int)j;
      const int o = M.bcell[b];
#pragma unroll
      for (int k = 0; k < NC; ++k) xf[i * NC + k] = bkind[b] ? x[(int64_t)o * NC + k] : bval[(int64_t)b * NC + k];
    } else {
#pragma unroll
      for (int k = 0; k < NC; ++k) xf[i * NC + k] = T(0);
    }
  }
}

// ------------------------------------------------------------ Gauss grad
// G_c = (1/V_c) [sum_f s_cf phi_f S_f + sum_b phi_b S_b] (eq:gauss_green
// P:207-213), G[c][k][l] = d phi^k / d x^l.
template <class T, int NC, bool FACEVALS, int KB, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_grad(DevMesh<T> M, const T* __restrict__ x,
                                                   const uint8_t* __restrict__ bkind, const T* __restrict__ bval,
                                                   const T* __restrict__ fv, T* __restrict__ G) {
  PDL_ENTRY();
  __shared__ T sh_out[kWarpsPerBlock][32 * 3 * NC];   // staged outputs of the warp's 32 rows
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  // software pipeline over the warp's slices: the next slice's metadata and
  // first incidence batch are in flight while this slice's face records load
  int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int len = 0;
  const int2* e = M.inc;
  int2 en[KB];
  if (s < M.n_slices) {
    len = __ldg(&M.sl_len[s]);
    e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
  }
#pragma unroll
  for (int u = 0; u < KB; ++u) en[u] = (u < len) ? __ldg(&e[u * 32]) : make_int2(0, -2);
  for (; s < M.n_slices; s += nw) {
    const int sn = s + nw;
    int len_n = 0;
    const int2* e_n = M.inc;
    if (sn < M.n_slices) {
      len_n = __ldg(&M.sl_len[sn]);
      e_n = M.inc + __ldg(&M.sl_ptr[sn]) + lane;
    }
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    T xc[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) xc[k] = T(0);
    if (!FACEVALS && live) {
      if (NC == 3) ld3(&x[(int64_t)row * NC], xc[0], xc[NC > 1 ? 1 : 0], xc[NC > 2 ? 2 : 0]);
      else xc[0] = x[row];
    }
    T acc[NC][3];
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k][0] = acc[k][1] = acc[k][2] = T(0);
    int2 en_n[KB];
    for (int j0 = 0; j0 < len; j0 += KB) {
      if (j0 > 0)
#pragma unroll
        for (int u = 0; u < KB; ++u) en[u] = (j0 + u < len) ? __ldg(&e[(j0 + u) * 32]) : make_int2(0, -2);
      V4<T> g[KB];
      T v[KB][NC];
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        g[u] = V4<T>{T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int k = 0; k < NC; ++k) v[u][k] = T(0);
        if (en[u].y >= 0) {
          const int f = en[u].x >= 0 ? en[u].x : ~en[u].x;
          g[u] = ld4(&M.fgeo[f]);
#pragma unroll
          if (NC == 3 && !FACEVALS)          // 3-vector gather in two loads (grad_U 0.456 -> 0.477)
            ld3(&x[(int64_t)en[u].y * NC], v[u][0], v[u][NC > 1 ? 1 : 0], v[u][NC > 2 ? 2 : 0]);
          else
#pragma unroll
            for (int k = 0; k < NC; ++k) v[u][k] = FACEVALS ? fv[(int64_t)f * NC + k] : x[(int64_t)en[u].y * NC + k];
        } else if (en[u].y == -1) {
          const int b = en[u].x;
          g[u] = ld4(&M.bgeo[b]);
#pragma unroll
          for (int k = 0; k < NC; ++k)
            v[u][k] = FACEVALS ? fv[((int64_t)M.F + b) * NC + k] : (bkind[b] ? xc[k] : bval[(int64_t)b * NC + k]);
        }
      }
      if (j0 + KB >= len)                    // last batch: prefetch the next slice's first batch
#pragma unroll
        for (int u = 0; u < KB; ++u) en_n[u] = (u < len_n) ? __ldg(&e_n[u * 32]) : make_int2(0, -2);
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        if (en[u].y >= 0) {
          const bool own = en[u].x >= 0;
          const T sg = own ? T(1) : T(-1);
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            T pf;
            if (FACEVALS) {
              pf = v[u][k];
            } else {
              const T xO = own ? xc[k] : v[u][k], xN = own ? v[u][k] : xc[k];
              pf = g[u].w * xO + (T(1) - g[u].w) * xN;
            }
            acc[k][0] += sg * pf * g[u].x; acc[k][1] += sg * pf * g[u].y; acc[k][2] += sg * pf * g[u].z;
          }
        } else if (en[u].y == -1) {
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            const T pb = v[u][k];
            acc[k][0] += pb * g[u].x; acc[k][1] += pb * g[u].y; acc[k][2] += pb * g[u].z;
          }
        }
      }
    }
    if (len == 0)
#pragma unroll
      for (int u = 0; u < KB; ++u) en_n[u] = (u < len_n) ? __ldg(&e_n[u * 32]) : make_int2(0, -2);
    // the warp's 32 rows x 3NC outputs are contiguous: stage them in shared
    // memory and store them coalesced (3NC full-line stores instead of 3NC
    // stride-3NC ones)
    if (live) {
      const T V = M.vol[row];
#pragma unroll
      for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int l = 0; l < 3; ++l) sh_out[wib][lane * 3 * NC + 3 * k + l] = acc[k][l] / V;
    }
    __syncwarp();
    {
      const int nlive = min(32, M.n_own - s * 32);
      T* gout = G + (int64_t)s * 32 * 3 * NC;
      for (int i = lane; i < nlive * 3 * NC; i += 32) gout[i] = sh_out[wib][i];
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < KB; ++u) en[u] = en_n[u];
    len = len_n;
    e = e_n;
  }
}

// ------------------------------------------------------------ divergence
// D_c = sum_f s_cf F_f + sum_b F_b (not divided by V)
template <class T>
__global__ void __launch_bounds__(kThreads) k_div(DevMesh<T> M, const T* __restrict__ flux, T* __restrict__ out) {
  PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < M.n_slices; s += nw) {
    const int row = s * 32 + lane;
    T acc = T(0);
    const int len = __ldg(&M.sl_len[s]);
    const int2* e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
    for (int j0 = 0; j0 < len; j0 += kB) {
      int2 en[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) en[u] = (j0 + u < len) ? __ldg(&e[(j0 + u) * 32]) : make_int2(0, -2);
      T v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        v[u] = T(0);
        if (en[u].y >= 0) v[u] = flux[en[u].x >= 0 ? en[u].x : ~en[u].x];
        else if (en[u].y == -1) v[u] = flux[M.F + en[u].x];
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (en[u].y >= 0) {
          if (en[u].x >= 0) acc += v[u]; else acc -= v[u];
        } else if (en[u].y == -1) {
          acc += v[u];
        }
      }
    }
    if (row < M.n_own) out[row] = acc;
  }
}

// ------------------------------------------------------------ Laplacian
// y_c = sum_f s_cf gamma_f [delta_f (x_N - x_O) + k_f . (w G_O + (1-w) G_N)]
//     + sum_{b fixed} gamma_c delta_b (x_b - x_c)   (eq:nonortho_flux P:240-250)
template <class T, bool GAMMA, int KB, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_lap(DevMesh<T> M, const T* __restrict__ gamma, const T* __restrict__ x,
                                                  const T* __restrict__ G, const uint8_t* __restrict__ bkind,
                                                  const T* __restrict__ bval, T* __restrict__ y) {
  PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  // software pipeline over the warp's slices (as in k_grad)
  int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int len = 0;
  const int2* e = M.inc;
  int2 en[KB];
  if (s < M.n_slices) {
    len = __ldg(&M.sl_len[s]);
    e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
  }
#pragma unroll
  for (int u = 0; u < KB; ++u) en[u] = (u < len) ? __ldg(&e[u * 32]) : make_int2(0, -2);
  for (; s < M.n_slices; s += nw) {
    const int sn = s + nw;
    int len_n = 0;
    const int2* e_n = M.inc;
    if (sn < M.n_slices) {
      len_n = __ldg(&M.sl_len[sn]);
      e_n = M.inc + __ldg(&M.sl_ptr[sn]) + lane;
    }
    int2 en_n[KB];
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    const T xc = live ? x[row] : T(0);
    const T gc = (GAMMA && live) ? gamma[row] : T(1);
    T Gc[3] = {T(0), T(0), T(0)};
    if (live) { Gc[0] = G[3 * (int64_t)row]; Gc[1] = G[3 * (int64_t)row + 1]; Gc[2] = G[3 * (int64_t)row + 2]; }
    T acc = T(0);
    for (int j0 = 0; j0 < len; j0 += KB) {
      if (j0 > 0)
#pragma unroll
        for (int u = 0; u < KB; ++u) en[u] = (j0 + u < len) ? __ldg(&e[(j0 + u) * 32]) : make_int2(0, -2);
      T w[KB], xn[KB], Gn[KB][3], gn[KB];
      V4<T> c[KB];
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        w[u] = xn[u] = gn[u] = T(0);
        Gn[u][0] = Gn[u][1] = Gn[u][2] = T(0);
        c[u] = V4<T>{T(0), T(0), T(0), T(0)};
        if (en[u].y >= 0) {
          const int f = en[u].x >= 0 ? en[u].x : ~en[u].x;
          const int n = en[u].y;
          w[u] = __ldg(&M.fw[f]);
          c[u] = ld4(&M.fcor[f]);
          xn[u] = x[n];
          if (sizeof(T) == 4)       // fp32: the gradient gather in two loads (fp64: three measured faster)
            ld3(&G[3 * (int64_t)n], Gn[u][0], Gn[u][1], Gn[u][2]);
          else {
            Gn[u][0] = G[3 * (int64_t)n]; Gn[u][1] = G[3 * (int64_t)n + 1]; Gn[u][2] = G[3 * (int64_t)n + 2];
          }
          if (GAMMA) gn[u] = gamma[n];
        } else if (en[u].y == -1) {
          const int b = en[u].x;
          if (bkind[b] == 0) { c[u].w = ld4(&M.bgeo[b]).w; xn[u] = bval[b]; }
        }
      }
      if (j0 + KB >= len)                    // last batch: prefetch the next slice's first batch
#pragma unroll
        for (int u = 0; u < KB; ++u) en_n[u] = (u < len_n) ? __ldg(&e_n[u * 32]) : make_int2(0, -2);
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        if (en[u].y >= 0) {
          const bool own = en[u].x >= 0;
          const T wO = w[u], wN = T(1) - w[u];
          const T xO = own ? xc : xn[u], xN = own ? xn[u] : xc;
          const T GO0 = own ? Gc[0] : Gn[u][0], GO1 = own ? Gc[1] : Gn[u][1], GO2 = own ? Gc[2] : Gn[u][2];
          const T GN0 = own ? Gn[u][0] : Gc[0], GN1 = own ? Gn[u][1] : Gc[1], GN2 = own ? Gn[u][2] : Gc[2];
          T gf = T(1);
          if (GAMMA) gf = wO * (own ? gc : gn[u]) + wN * (own ? gn[u] : gc);
          const T corr = c[u].x * (wO * GO0 + wN * GN0) + c[u].y * (wO * GO1 + wN * GN1) + c[u].z * (wO * GO2 + wN * GN2);
          const T q = gf * (c[u].w * (xN - xO) + corr);
          acc += own ? q : -q;
        } else if (en[u].y == -1) {
          if (bkind[en[u].x] == 0) acc += gc * c[u].w * (xn[u] - xc);
        }
      }
    }
    if (len == 0)
#pragma unroll
      for (int u = 0; u < KB; ++u) en_n[u] = (u < len_n) ? __ldg(&e_n[u * 32]) : make_int2(0, -2);
    if (live) y[row] = acc;
#pragma unroll
    for (int u = 0; u < KB; ++u) en[u] = en_n[u];
    len = len_n;
    e = e_n;
  }
}

// ------------------------------------------------------------ launchers
template <class T>
void launch_interpolate(const DevMesh<T>& M, const T* x, int nc, const uint8_t* bk, const T* bv, T* xf, cudaStream_t s) {
  // one wave of resident blocks (the 3-vector variant holds 96 registers):
  // a second wave would revisit the cells the first one left in L2 long ago
  const int64_t nf = (int64_t)M.F + M.B + M.E;
  if (nc == 1) k_interp<T, 1><<<grid_rows(k_interp<T, 1>, nf), kThreads, 0, s>>>(M, x, bk, bv, xf);
  else k_interp<T, 3><<<grid_rows(k_interp<T, 3>, nf), kThreads, 0, s>>>(M, x, bk, bv, xf);
  count_launch();
}
// Batch depth KB and minimum resident blocks MINB (register cap 64), measured
// on C5 (sweep of 5 {KB, MINB} variants, profiles/r01_ops_variants_c5.json):
// shallow batches at 4 resident blocks per SM beat deeper batches at lower
// occupancy (grad_s 0.62 -> 0.78, lap 0.45 -> 0.64 of the HBM peak).  Grids
// are one full wave of resident blocks (occupancy API).
// fp32 variants (DFVM_OPS_F32, read per launch, for A/B): the fp32 kernels
// need fewer registers, so more resident blocks / deeper batches fit:
//   0: the fp64 settings; 1: 6 blocks/SM; 2: 8 blocks/SM; 3: batch 4 at 6 blocks/SM
static int ops_f32_variant() {
  const char* e = getenv("DFVM_OPS_F32");
  return e ? atoi(e) : kOpsF32Default;
}
template <class T, int NC, bool FV>
static void grad_any(const DevMesh<T>& M, const T* x, const uint8_t* bk, const T* bv, const T* fv, T* G, cudaStream_t s) {
  const int v = sizeof(T) == 4 ? ops_f32_variant() : 0;
  if (v == 1) {
    auto fn = k_grad<T, NC, FV, NC == 1 ? 2 : 1, 6>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, x, bk, bv, fv, G);
  } else if (v == 2) {
    auto fn = k_grad<T, NC, FV, NC == 1 ? 2 : 1, 8>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, x, bk, bv, fv, G);
  } else if (v == 3) {
    auto fn = k_grad<T, NC, FV, NC == 1 ? 4 : 2, 6>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, x, bk, bv, fv, G);
  } else {
    auto fn = k_grad<T, NC, FV, NC == 1 ? 2 : 1, 4>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, x, bk, bv, fv, G);
  }
}
template <class T>
void launch_grad(const DevMesh<T>& M, const T* x, int nc, const uint8_t* bk, const T* bv, T* G, cudaStream_t s) {
  if (nc == 1) grad_any<T, 1, false>(M, x, bk, bv, nullptr, G, s);
  else grad_any<T, 3, false>(M, x, bk, bv, nullptr, G, s);
  count_launch();
}
template <class T>
void launch_grad_faces(const DevMesh<T>& M, const T* fv, int nc, T* G, cudaStream_t s) {
  if (nc == 1) grad_any<T, 1, true>(M, nullptr, nullptr, nullptr, fv, G, s);
  else grad_any<T, 3, true>(M, nullptr, nullptr, nullptr, fv, G, s);
  count_launch();
}
template <class T>
void launch_div(const DevMesh<T>& M, const T* flux, T* out, cudaStream_t s) {
  k_div<T><<<grid_for_slices(M.n_slices), kThreads, 0, s>>>(M, flux, out);
  count_launch();
}
template <class T, bool GA>
static void lap_any(const DevMesh<T>& M, const T* gamma, const T* x, const T* G, const uint8_t* bk, const T* bv, T* y,
                    cudaStream_t s) {
  const int v = sizeof(T) == 4 ? ops_f32_variant() : 0;
  if (v == 1) {
    auto fn = k_lap<T, GA, 1, 6>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, gamma, x, G, bk, bv, y);
  } else if (v == 2) {
    auto fn = k_lap<T, GA, 1, 8>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, gamma, x, G, bk, bv, y);
  } else if (v == 3) {
    auto fn = k_lap<T, GA, 2, 6>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, gamma, x, G, bk, bv, y);
  } else {
    auto fn = k_lap<T, GA, 1, 4>;
    fn<<<grid_slices(fn, M.n_slices), kThreads, 0, s>>>(M, gamma, x, G, bk, bv, y);
  }
}
template <class T>
void launch_laplacian(const DevMesh<T>& M, const T* gamma, const T* x, const T* G, const uint8_t* bk, const T* bv,
                      T* y, cudaStream_t s) {
  if (gamma) lap_any<T, true>(M, gamma, x, G, bk, bv, y, s);
  else lap_any<T, false>(M, gamma, x, G, bk, bv, y, s);
  count_launch();
}

#define INST(T)                                                                                          \
  template void launch_import<T>(T*, const double*, const int32_t*, int64_t, int, bool, cudaStream_t);   \
  template void launch_export<T>(double*, const T*, const int32_t*, int64_t, int, bool, cudaStream_t);   \
  template void launch_interpolate<T>(const DevMesh<T>&, const T*, int, const uint8_t*, const T*, T*,    \
                                      cudaStream_t);                                                     \
  template void launch_grad<T>(const DevMesh<T>&, const T*, int, const uint8_t*, const T*, T*, cudaStream_t); \
  template void launch_grad_faces<T>(const DevMesh<T>&, const T*, int, T*, cudaStream_t);                \
  template void launch_div<T>(const DevMesh<T>&, const T*, T*, cudaStream_t);                            \
  template void launch_laplacian<T>(const DevMesh<T>&, const T*, const T*, const T*, const uint8_t*,     \
                                    const T*, T*, cudaStream_t);
INST(double)
INST(float)

}  // namespace dfvm

namespace dfvm {
// time-varying boundary values (A-41): val[b] = base[b] * g[wave of b]
template <class T>
__global__ void k_bc_wave(T* __restrict__ val, const T* __restrict__ base, const int8_t* __restrict__ wid, int64_t B,
                          int nc, WaveG<T> g) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    const int w = wid[i];
    if (w >= 0)
      for (int k = 0; k < nc; ++k) val[i * nc + k] = base[i * nc + k] * g.g[w];
  }
}
template <class T>
void launch_bc_wave(T* val, const T* base, const int8_t* wid, int64_t B, int nc, const WaveG<T>& g, cudaStream_t s) {
  if (B <= 0) return;
  k_bc_wave<T><<<grid_for(B), kThreads, 0, s>>>(val, base, wid, B, nc, g);   // counted by the caller
}
template void launch_bc_wave<double>(double*, const double*, const int8_t*, int64_t, int, const WaveG<double>&, cudaStream_t);
template void launch_bc_wave<float>(float*, const float*, const int8_t*, int64_t, int, const WaveG<float>&, cudaStream_t);

// halo pack: buf[i][k] = x[idx[i]][k]  (send list of owned interface cells)
template <class T>
__global__ void k_pack(T* __restrict__ buf, const T* __restrict__ x, const int32_t* __restrict__ idx, int64_t n, int nc) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < nc; ++k) buf[i * nc + k] = x[(int64_t)idx[i] * nc + k];
}
template <class T>
void launch_pack(T* buf, const T* x, const int32_t* idx, int64_t n, int nc, cudaStream_t s) {
  if (n <= 0) return;
  k_pack<T><<<grid_for(n), kThreads, 0, s>>>(buf, x, idx, n, nc);
  count_launch();
}
template void launch_pack<double>(double*, const double*, const int32_t*, int64_t, int, cudaStream_t);
template void launch_pack<float>(float*, const float*, const int32_t*, int64_t, int, cudaStream_t);
}  // namespace dfvm
