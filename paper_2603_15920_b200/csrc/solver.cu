// solver.cu — the PISO step on B200 (PAPER.md
// §2.4.2, Table 1): momentum LDU assembly, 3-component
// BiCGStab predictor, H / rAU / HbyA, phiHbyA, pressure coefficients, the
// Jacobi-PCG pressure solve, Rhie-Chow flux correction, velocity correction,
// Windkessel outlets and the continuity diagnostic.
//
// Krylov control runs on the device: every reduction is a deterministic
// two-level sum (block partials in block order, then the last block to
// arrive sums them in a fixed order) and that last block updates the solver
// scalars (alpha, beta, residual, convergence, stagnation) in a device
// control block.  Every Krylov kernel first checks the control block and
// exits when the solve is done, so the host enqueues iterations in chunks
// and reads the control block once per chunk (no per-iteration host sync).
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "dev.cuh"
#include "amg.h"
#include "launch.h"
#include "prof.h"
#include "krylov.cuh"

namespace dfvm {

dfvm_status halo_exchange(dfvm_mesh* m, void* data, int nc, cudaStream_t s);

// y_row = diag_row x_row + sum_j coef_j x_nb(j) over the matrix SELL entries
template <class T, int NC>
__device__ __forceinline__ void sell_apply(const DevMesh<T>& M, int s, int lane, const T* __restrict__ coef,
                                           const T* __restrict__ x, T (&acc)[NC]) {
  const int len = __ldg(&M.ms_len[s]);
  const int base = __ldg(&M.ms_ptr[s]) + lane;
  int j = 0;
  // batches of 4 incidences: all coefficient / column loads first, then all
  // gathers, then the FMAs (same summation order), so each thread keeps 8+4
  // independent loads in flight instead of a dependent chain per entry
  for (; j + 4 <= len; j += 4) {
    T a[4];
    int n[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = __ldg(&coef[base + 32 * (j + u)]);
      n[u] = __ldg(&M.mnb[base + 32 * (j + u)]);
    }
    T v[4][NC];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < NC; ++k) v[u][k] = x[(int64_t)n[u] * NC + k];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < NC; ++k) acc[k] += a[u] * v[u][k];
  }
  for (; j < len; ++j) {
    const int idx = base + 32 * j;
    const T a = __ldg(&coef[idx]);
    const int n = __ldg(&M.mnb[idx]);
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] += a * x[(int64_t)n * NC + k];
  }
}

#define SLICE_LOOP(M)                                                                      \
  const int lane = threadIdx.x & 31;                                                       \
  const int nw_ = (gridDim.x * blockDim.x) >> 5;                                           \
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < (M).n_slices; s += nw_)

// ============================================================ momentum / transport
// O-5 transport LDU for NC components (momentum: NC = 3, field 'U', nu;
// passive scalar: NC = 1, field 's', Gamma): diag, b (time + BC + explicit
// non-orthogonal terms), rhs = b - V grad p (when gp != NULL), SELL
// coefficients (upper for the owner side, lower for the neighbour side).
// conv: 0 upwind, 1 central (implicit via the face weight), 2 SOU, 3 QUICK —
// 2/3: implicit upwind + explicit deferred correction m (x^HO - x_C)
// (eq:deferred_correction, eq:sou P:200-206, SPEC.md:233 QUICK),
// with dO = x_f - x_O, dN = x_f - x_N per face.
// HO: deferred-correction (SOU / QUICK) code compiled in; EXPL: theta != 1
// (the explicit part A_s x^n).  The upwind / central backward-Euler variant
// (the bench path) compiles without either (fewer registers, higher
// occupancy; the same arithmetic).
template <class T, int NC, bool HO = true, bool EXPL = true>
__global__ void __launch_bounds__(kThreads) k_transport_assemble(DevMesh<T> M, const T* __restrict__ U,
    const T* __restrict__ phi, const T* __restrict__ gU, const T* __restrict__ gp, const uint8_t* __restrict__ bk,
    const T* __restrict__ bv, T nu, T rdt, T theta, int conv, int kcorr, const V4<T>* __restrict__ fdO,
    const V4<T>* __restrict__ fdN, T* __restrict__ udiag, T* __restrict__ bU, T* __restrict__ rhsU,
    T* __restrict__ ucoef, T* __restrict__ ucoefT) {
  PDL_ENTRY();
  const bool explicit_part = EXPL && theta != T(1);
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    const T V = live ? M.vol[row] : T(0);
    T diag = T(0);           // diagonal of the spatial operator A_s
    T bb[NC], xc[NC], ax[NC];  // b_s (explicit sources); x^n_c; sum_nb a_s x^n_nb (theta != 1)
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      bb[k] = T(0);
      ax[k] = T(0);
      xc[k] = live ? U[NC * (int64_t)row + k] : T(0);
    }
    const int len = __ldg(&M.sl_len[s]);
    const int2* e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
    const int mbase = __ldg(&M.ms_ptr[s]) + lane;
    int mj = 0;
    for (int j = 0; j < len; ++j) {
      const int2 en = __ldg(&e[j * 32]);
      if (en.y >= 0) {
        const bool own = en.x >= 0;
        const int f = own ? en.x : ~en.x;
        const T w = __ldg(&M.fw[f]);
        const V4<T> c = ld4(&M.fcor[f]);
        const T md = phi[f];
        const T lam = conv == 1 ? w : (md >= T(0) ? T(1) : T(0));
        const T nd = nu * c.w;
        T cf, cfT;   // this row's coefficient and the transposed one (the other row's, NEXT-3)
        if (own) { diag += lam * md + nd; cf = (T(1) - lam) * md - nd; cfT = -lam * md - nd; }
        else { diag += -(T(1) - lam) * md + nd; cf = -lam * md - nd; cfT = (T(1) - lam) * md - nd; }
        ucoefT[mbase + 32 * mj] = theta * cfT;
        ucoef[mbase + 32 * (mj++)] = theta * cf;
        const int n = en.y;
        if (explicit_part)
#pragma unroll
          for (int k = 0; k < NC; ++k) ax[k] += cf * U[NC * (int64_t)n + k];
        const int O = own ? row : n, N = own ? n : row;
        T cr[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) cr[k] = T(0);
        if (kcorr) {
          // (the row's own gradient hoisted into registers was measured
          // slower: 74 registers against 56, 6.24 against 6.12 ms/step)
          const T* GO = gU + 3 * NC * (int64_t)O;
          const T* GN = gU + 3 * NC * (int64_t)N;
#pragma unroll
          for (int k = 0; k < NC; ++k)
            cr[k] = nu * (c.x * (w * GO[3 * k] + (T(1) - w) * GN[3 * k]) +
                          c.y * (w * GO[3 * k + 1] + (T(1) - w) * GN[3 * k + 1]) +
                          c.z * (w * GO[3 * k + 2] + (T(1) - w) * GN[3 * k + 2]));
        }
        if (HO && conv >= 2) {
          const bool up_own = md >= T(0);
          const int Cc = up_own ? O : N, D = up_own ? N : O;
          const V4<T> a = ld4(up_own ? &fdO[f] : &fdN[f]);            // d_Cf = x_f - x_C
          const V4<T> o4 = ld4(&fdO[f]), n4 = ld4(&fdN[f]);
          T dCD[3] = {o4.x - n4.x, o4.y - n4.y, o4.z - n4.z};           // x_N - x_O
          if (!up_own) { dCD[0] = -dCD[0]; dCD[1] = -dCD[1]; dCD[2] = -dCD[2]; }
          const T fCD = (a.x * dCD[0] + a.y * dCD[1] + a.z * dCD[2]) /
                        (dCD[0] * dCD[0] + dCD[1] * dCD[1] + dCD[2] * dCD[2]);
          const T* GC = gU + 3 * NC * (int64_t)Cc;
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            const T gd = GC[3 * k] * a.x + GC[3 * k + 1] * a.y + GC[3 * k + 2] * a.z;
            const T xC = U[NC * (int64_t)Cc + k], xD = U[NC * (int64_t)D + k];
            const T hi = conv == 2 ? xC + gd : xC + T(0.5) * (gd + (xD - xC) * fCD);
            const T dc = md * (hi - xC);
            cr[k] = cr[k] - dc;        // owner row: + (corr - dc); neighbour row: - (corr - dc)
          }
        }
        if (own) {
#pragma unroll
          for (int k = 0; k < NC; ++k) bb[k] += cr[k];
        } else {
#pragma unroll
          for (int k = 0; k < NC; ++k) bb[k] -= cr[k];
        }
      } else if (en.y == -1) {
        const int b = en.x;
        const T mb = phi[M.F + b];
        if (bk[b] == 0) {
          const T nd = nu * ld4(&M.bgeo[b]).w;
          diag += nd;
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            const T ub = bv[NC * (int64_t)b + k];
            bb[k] += -mb * ub + nd * ub;
          }
        } else {
          diag += mb;
        }
      }
    }
    if (live) {
      // theta method (Table 1, A-40): diag = V/dt + theta diag_s,
      // b = V/dt x^n + b_s - (1 - theta) (A_s x^n)
      const T vdt = V * rdt;
      udiag[row] = vdt + theta * diag;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const T axk = diag * xc[k] + ax[k];
        const T bk_ = vdt * xc[k] + bb[k] - (T(1) - theta) * axk;
        bU[NC * (int64_t)row + k] = bk_;
        rhsU[NC * (int64_t)row + k] = gp ? bk_ - V * gp[3 * (int64_t)row + k] : bk_;
      }
    }
  }
}

template <class T, int NC>
static void launch_transport_assemble(int n_slices, cudaStream_t st, DevMesh<T> M, const T* U, const T* phi, const T* gU,
                                      const T* gp, const uint8_t* bk, const T* bv, T nu, T rdt, T theta, int conv,
                                      int kcorr, const V4<T>* fdO, const V4<T>* fdN, T* udiag, T* bU, T* rhsU, T* ucoef,
                                      T* ucoefT) {
  const bool ho = conv >= 2, ex = theta != T(1);
#define KTA(H, E)                                                                                                   \
  k_transport_assemble<T, NC, H, E><<<grid_slices(k_transport_assemble<T, NC, H, E>, n_slices), kThreads, 0, st>>>( \
      M, U, phi, gU, gp, bk, bv, nu, rdt, theta, conv, kcorr, \
                                                              fdO, fdN, udiag, bU, rhsU, ucoef, ucoefT)
  if (ho && ex) KTA(true, true);
  else if (ho) KTA(true, false);
  else if (ex) KTA(false, true);
  else KTA(false, false);
#undef KTA
}

template <class T, int NC>
__global__ void __launch_bounds__(kThreads) k_apply(DevMesh<T> M, const T* __restrict__ diag,
    const T* __restrict__ coef, const T* __restrict__ x, T* __restrict__ y) {
  PDL_ENTRY();
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    T acc[NC];
    const T d = live ? diag[row] : T(0);
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = live ? d * x[(int64_t)row * NC + k] : T(0);
    sell_apply<T, NC>(M, s, lane, coef, x, acc);
    if (live)
#pragma unroll
      for (int k = 0; k < NC; ++k) y[(int64_t)row * NC + k] = acc[k];
  }
}

// rAU = V / a_P alone (the AMG side stream's pressure matrix, ahead of the
// momentum solve); k_HbyA then leaves rAU alone (write_rau = 0)
template <class T>
__global__ void k_rAU(int n, const T* __restrict__ vol, const T* __restrict__ udiag, T* __restrict__ rAU) {
  PDL_ENTRY();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rAU[i] = vol[i] / udiag[i];
}

// H = b - sum_nb a U_nb; rAU = V / a_P; HbyA = H / a_P (eq:Ap_H P:333-335)
template <class T>
__global__ void __launch_bounds__(kThreads) k_HbyA(DevMesh<T> M, const T* __restrict__ bU, const T* __restrict__ udiag,
    const T* __restrict__ ucoef, const T* __restrict__ U, T* __restrict__ rAU, T* __restrict__ HbyA, int write_rau = 1) {
  PDL_ENTRY();
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    T acc[3] = {T(0), T(0), T(0)};
    sell_apply<T, 3>(M, s, lane, ucoef, U, acc);
    if (live) {
      const T d = udiag[row];
      if (write_rau) rAU[row] = M.vol[row] / d;
#pragma unroll
      for (int k = 0; k < 3; ++k) HbyA[3 * (int64_t)row + k] = (bU[3 * (int64_t)row + k] - acc[k]) / d;
    }
  }
}

// phiHbyA_f = interp(HbyA) . S_f; boundary: U_b . S_b (fixed U) or HbyA_O . S_b
// Optional ddtCorr (A-42, OpenFOAM's Euler ddtCorr) on internal faces:
// phiHbyA += rAU_f c_f (phi^n - U^n_f . S) / dt, c_f = 1 - min(|d| / (|phi^n| + 1e-15), 1)
template <class T>
__global__ void k_phiHbyA(DevMesh<T> M, const T* __restrict__ HbyA, const uint8_t* __restrict__ bk,
                          const T* __restrict__ bv, T* __restrict__ out, const T* __restrict__ Uold,
                          const T* __restrict__ phiold, const T* __restrict__ rAU, T rdt) {
  PDL_ENTRY();
  const int64_t total = (int64_t)M.F + M.B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < M.F) {
      const int2 c = __ldg(&M.fcell[i]);
      const V4<T> g = ld4(&M.fgeo[i]);
      const T* a = HbyA + 3 * (int64_t)c.x;
      const T* b = HbyA + 3 * (int64_t)c.y;
      T v = (g.w * a[0] + (T(1) - g.w) * b[0]) * g.x + (g.w * a[1] + (T(1) - g.w) * b[1]) * g.y +
            (g.w * a[2] + (T(1) - g.w) * b[2]) * g.z;
      if (Uold) {
        const T* uo = Uold + 3 * (int64_t)c.x;
        const T* un = Uold + 3 * (int64_t)c.y;
        const T uS = (g.w * uo[0] + (T(1) - g.w) * un[0]) * g.x + (g.w * uo[1] + (T(1) - g.w) * un[1]) * g.y +
                     (g.w * uo[2] + (T(1) - g.w) * un[2]) * g.z;
        const T ph = phiold[i];
        const T d = ph - uS;
        const T cc = T(1) - fmin(fabs(d) / (fabs(ph) + T(1e-15)), T(1));
        const T rf = g.w * rAU[c.x] + (T(1) - g.w) * rAU[c.y];
        v += rf * cc * d * rdt;
      }
      out[i] = v;
    } else {
      const int b = (int)(i - M.F);
      const V4<T> g = ld4(&M.bgeo[b]);
      const T* h = bk[b] ? HbyA + 3 * (int64_t)M.bcell[b] : bv + 3 * (int64_t)b;
      out[i] = h[0] * g.x + h[1] * g.y + h[2] * g.z;
    }
  }
}

// pressure coefficients (eq:pressure_poisson LHS; A-8): pcoef = -c_f,
// pdiag = sum c_f + sum c_b, prhs0 = -D(phiHbyA) + sum c_b p_b, gauge (A-12)
// mode: bit 0 writes the matrix (pcoef, pdiag), bit 1 the right-hand side
// prhs0 (the matrix part alone runs ahead of the momentum solve on the AMG
// side stream, the right-hand side in the corrector)
template <class T>
__global__ void __launch_bounds__(kThreads) k_pcoef(DevMesh<T> M, const T* __restrict__ rAU,
    const T* __restrict__ phiHbyA, const uint8_t* __restrict__ bkp, const T* __restrict__ bvp, int ref_row,
    T p_ref, T* __restrict__ pcoef, T* __restrict__ pdiag, T* __restrict__ prhs0, int mode = 3) {
  PDL_ENTRY();
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    const T ra = live ? rAU[row] : T(0);
    T diag = T(0), rhs = T(0);
    const int len = __ldg(&M.sl_len[s]);
    const int2* e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
    const int mbase = __ldg(&M.ms_ptr[s]) + lane;
    int mj = 0;
    for (int j = 0; j < len; ++j) {
      const int2 en = __ldg(&e[j * 32]);
      if (en.y >= 0) {
        const bool own = en.x >= 0;
        const int f = own ? en.x : ~en.x;
        T w, d;
        ld2(M.fwd + 2 * (int64_t)f, w, d);
        const T rn = rAU[en.y];
        const T cf = (w * (own ? ra : rn) + (T(1) - w) * (own ? rn : ra)) * d;
        if (mode & 1) pcoef[mbase + 32 * mj] = -cf;
        ++mj;
        diag += cf;
        if (mode & 2) rhs -= own ? phiHbyA[f] : -phiHbyA[f];
      } else if (en.y == -1) {
        const int b = en.x;
        if (mode & 2) rhs -= phiHbyA[M.F + b];
        if (bkp[b] == 0) {
          const T cb = ra * ld4(&M.bgeo[b]).w;
          diag += cb;
          if (mode & 2) rhs += cb * bvp[b];
        }
      }
    }
    if (live) {
      if (row == ref_row) { rhs += diag * p_ref; diag = diag + diag; }
      if (mode & 1) pdiag[row] = diag;
      if (mode & 2) prhs0[row] = rhs;
    }
  }
}

// NEXT-3, eq:implicit_diff P:366-370: dL/drAU through the converged solve
// A(rAU) p = rhs given lambda = A^-T dL/dp (derivation: oracle
// orc_pressure_vjp).  Per face dL/dc_f = -(lambda_O - lambda_N)(p_O - p_N)
// (+ lambda_r (p_ref - p_r) if the face touches the gauge row r), split to
// the rows by dc_f/drAU = (w, 1-w) delta_f; fixed-value boundary faces
// -lambda_O p_O delta_b.  p, lambda need valid ghosts.
template <class T>
__global__ void __launch_bounds__(kThreads) k_pvjp(DevMesh<T> M, const T* __restrict__ p, const T* __restrict__ lam,
    const uint8_t* __restrict__ bkp, const int32_t* __restrict__ corig, int ref_orig, T p_ref, T* __restrict__ grad) {
  PDL_ENTRY();
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    const T pc = live ? p[row] : T(0), lc = live ? lam[row] : T(0);
    const bool rc = live && ref_orig >= 0 && corig[row] == ref_orig;
    T acc = T(0);
    const int len = __ldg(&M.sl_len[s]);
    const int2* e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
    for (int j = 0; j < len; ++j) {
      const int2 en = __ldg(&e[j * 32]);
      if (en.y >= 0) {
        const bool own = en.x >= 0;
        const int f = own ? en.x : ~en.x;
        const int n = en.y;
        const T pn = p[n], ln = lam[n];
        const T pO = own ? pc : pn, pN = own ? pn : pc, lO = own ? lc : ln, lN = own ? ln : lc;
        T d = -(lO - lN) * (pO - pN);
        if (ref_orig >= 0) {
          if (rc) d += lc * (p_ref - pc);
          else if (corig[n] == ref_orig) d += ln * (p_ref - pn);
        }
        const T w = __ldg(&M.fw[f]);
        acc += d * (own ? w : T(1) - w) * ld4(&M.fcor[f]).w;
      } else if (en.y == -1) {
        const int b = en.x;
        if (bkp[b] == 0) acc += -lc * pc * ld4(&M.bgeo[b]).w;
      }
    }
    if (live) grad[row] = acc;
  }
}

// prhs = prhs0 + sum_f s_cf rAU_f k_f . (grad p)_f  (explicit non-orthogonal part)
template <class T>
__global__ void __launch_bounds__(kThreads) k_prhs(DevMesh<T> M, const T* __restrict__ rAU, const T* __restrict__ gp,
    const T* __restrict__ prhs0, T* __restrict__ prhs) {
  PDL_ENTRY();
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    const T ra = live ? rAU[row] : T(0);
    T acc = live ? prhs0[row] : T(0);
    // the row's own gradient in registers: 3 gathered loads per incidence, not 6
    T gc[3] = {T(0), T(0), T(0)};
    if (live)
#pragma unroll
      for (int k = 0; k < 3; ++k) gc[k] = gp[3 * (int64_t)row + k];
    const int len = __ldg(&M.sl_len[s]);
    const int2* e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
    for (int j = 0; j < len; ++j) {
      const int2 en = __ldg(&e[j * 32]);
      if (en.y < 0) continue;
      const bool own = en.x >= 0;
      const int f = own ? en.x : ~en.x;
      const int n = en.y;
      const V4<T> c = ld4(&M.fkw[f]);   // {k, w}
      const T w = c.w;
      const T rn = rAU[n];
      T gn[3], GO[3], GN[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        gn[k] = gp[3 * (int64_t)n + k];
        GO[k] = own ? gc[k] : gn[k];
        GN[k] = own ? gn[k] : gc[k];
      }
      const T rf = w * (own ? ra : rn) + (T(1) - w) * (own ? rn : ra);
      const T kg = c.x * (w * GO[0] + (T(1) - w) * GN[0]) + c.y * (w * GO[1] + (T(1) - w) * GN[1]) +
                   c.z * (w * GO[2] + (T(1) - w) * GN[2]);
      acc += own ? rf * kg : -(rf * kg);
    }
    if (live) prhs[row] = acc;
  }
}

// Rhie-Chow flux correction (A-9)
template <class T>
__global__ void k_fluxcorr(DevMesh<T> M, const T* __restrict__ phiHbyA, const T* __restrict__ p,
                           const T* __restrict__ rAU, const T* __restrict__ gp, const uint8_t* __restrict__ bkp,
                           const T* __restrict__ bvp, int kcorr, T* __restrict__ phi) {
  PDL_ENTRY();
  const int64_t total = (int64_t)M.F + M.B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < M.F) {
      const int2 cc = __ldg(&M.fcell[i]);
      const T w = __ldg(&M.fw[i]);
      const V4<T> c = ld4(&M.fcor[i]);
      const T rf = w * rAU[cc.x] + (T(1) - w) * rAU[cc.y];
      T v = phiHbyA[i] - rf * c.w * (p[cc.y] - p[cc.x]);
      if (kcorr) {
        const T* GO = gp + 3 * (int64_t)cc.x;
        const T* GN = gp + 3 * (int64_t)cc.y;
        const T kg = c.x * (w * GO[0] + (T(1) - w) * GN[0]) + c.y * (w * GO[1] + (T(1) - w) * GN[1]) +
                     c.z * (w * GO[2] + (T(1) - w) * GN[2]);
        v -= rf * kg;
      }
      phi[i] = v;
    } else {
      const int b = (int)(i - M.F);
      if (bkp[b] == 0) {
        const int o = M.bcell[b];
        const T cb = rAU[o] * ld4(&M.bgeo[b]).w;
        phi[i] = phiHbyA[i] - cb * (bvp[b] - p[o]);
      } else {
        phi[i] = phiHbyA[i];
      }
    }
  }
}

// U = HbyA - rAU grad p with the Gauss gradient of the new p (eq:velocity_correction
// P:344-346); the gradient is stored for the next corrector / step.
template <class T>
__global__ void __launch_bounds__(kThreads) k_Ucorr(DevMesh<T> M, const T* __restrict__ p,
    const uint8_t* __restrict__ bkp, const T* __restrict__ bvp, const T* __restrict__ HbyA,
    const T* __restrict__ rAU, T* __restrict__ U, T* __restrict__ gp) {
  PDL_ENTRY();
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    const T pc = live ? p[row] : T(0);
    T a0 = T(0), a1 = T(0), a2 = T(0);
    const int len = __ldg(&M.sl_len[s]);
    const int2* e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
    for (int j = 0; j < len; ++j) {
      const int2 en = __ldg(&e[j * 32]);
      if (en.y >= 0) {
        const bool own = en.x >= 0;
        const int f = own ? en.x : ~en.x;
        const V4<T> g = ld4(&M.fgeo[f]);
        const T pn = p[en.y];
        const T pf = g.w * (own ? pc : pn) + (T(1) - g.w) * (own ? pn : pc);
        const T sp = own ? pf : -pf;
        a0 += sp * g.x; a1 += sp * g.y; a2 += sp * g.z;
      } else if (en.y == -1) {
        const int b = en.x;
        const V4<T> g = ld4(&M.bgeo[b]);
        const T pb = bkp[b] ? pc : bvp[b];
        a0 += pb * g.x; a1 += pb * g.y; a2 += pb * g.z;
      }
    }
    if (live) {
      const T V = M.vol[row];
      const T g0 = a0 / V, g1 = a1 / V, g2 = a2 / V;
      gp[3 * (int64_t)row] = g0; gp[3 * (int64_t)row + 1] = g1; gp[3 * (int64_t)row + 2] = g2;
      const T r = rAU[row];
      U[3 * (int64_t)row] = HbyA[3 * (int64_t)row] - r * g0;
      U[3 * (int64_t)row + 1] = HbyA[3 * (int64_t)row + 1] - r * g1;
      U[3 * (int64_t)row + 2] = HbyA[3 * (int64_t)row + 2] - r * g2;
    }
  }
}

// continuity max_c |D_c(phi)|, sum_c |D_c(phi)|, non-finite flag; the last
// block also commits the Windkessel states of the step (p_c^n <- p_c^{n+1}).
template <class T>
__global__ void __launch_bounds__(kThreads) k_continuity(DevMesh<T> M, const T* __restrict__ phi,
    const T* __restrict__ U, const T* __restrict__ p, double* partials, unsigned* ticket, double* out,
    WKDev* wk, int n_wk, Red red) {
  PDL_ENTRY();
  double mx = 0, sm = 0, nf = 0;
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    T acc = T(0);
    const int len = __ldg(&M.sl_len[s]);
    const int2* e = M.inc + __ldg(&M.sl_ptr[s]) + lane;
    for (int j = 0; j < len; ++j) {
      const int2 en = __ldg(&e[j * 32]);
      if (en.y >= 0) { if (en.x >= 0) acc += phi[en.x]; else acc -= phi[~en.x]; }
      else if (en.y == -1) acc += phi[M.F + en.x];
    }
    if (row < M.n_own) {
      const double a = fabs((double)acc);
      mx = fmax(mx, a);
      sm += a;
      const T u0 = U[3 * (int64_t)row], u1 = U[3 * (int64_t)row + 1], u2 = U[3 * (int64_t)row + 2];
      if (!isfinite((double)u0) || !isfinite((double)u1) || !isfinite((double)u2) || !isfinite((double)p[row])) nf = 1;
    }
  }
  // max via the sum machinery: reduce (sum, nonfinite) and max separately
  __shared__ double shm[32];
  double wm = warp_max(mx);
  if ((threadIdx.x & 31) == 0) shm[threadIdx.x >> 5] = wm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = fmax(b, shm[w]);
    mx = b;
  }
  double v[2] = {sm, nf}, tot[2];
  const double* maxp = partials + 2 * gridDim.x;
  if (threadIdx.x == 0) const_cast<double*>(maxp)[blockIdx.x] = mx;
  if (grid_sum<2>(v, partials, ticket, tot)) {
    double m2 = 0;
    for (unsigned b = 0; b < gridDim.x; ++b) m2 = fmax(m2, __ldcg(&maxp[b]));
    if (red.nranks > 1) { red.local[0] = m2; red.local[1] = tot[0]; red.local[2] = tot[1]; return; }
    out[0] = m2; out[1] = tot[0]; out[2] = tot[1] > 0 ? 1.0 : 0.0;
    for (int i = 0; i < n_wk; ++i) wk[i].pc_n = wk[i].pc_new;
  }
}

// cross-rank continuity: max / sum / non-finite over ranks, then the
// Windkessel commit (every rank holds the same outlet states)
__global__ void k_continuity_fin(const double* __restrict__ all, int P, double* out, WKDev* wk, int n_wk) {
  PDL_ENTRY();
  double mx = 0, sm = 0, nf = 0;
  for (int r = 0; r < P; ++r) { mx = fmax(mx, all[3 * r]); sm += all[3 * r + 1]; nf += all[3 * r + 2]; }
  out[0] = mx; out[1] = sm; out[2] = nf > 0 ? 1.0 : 0.0;
  for (int i = 0; i < n_wk; ++i) wk[i].pc_n = wk[i].pc_new;
}

// Windkessel (eq:windkessel_Q P:406-410, eq:windkessel_discrete P:420-425):
// one block per outlet; Q = sum_b phi_b (fixed order), p_c^{n+1} from the
// start-of-step p_c^n (A-19), p_o = p_c + R_p Q, BC value p_o / rho.
__device__ __forceinline__ double wk_update(WKDev& W, double Q, double dt) {
  double pc;
  if (W.scheme == 0) { const double ex = exp(-dt / (W.Rd * W.C)); pc = W.pc_n * ex + W.Rd * Q * (1.0 - ex); }
  else if (W.scheme == 1) pc = W.pc_n + dt * (Q - W.pc_n / W.Rd) / W.C;
  else pc = (W.pc_n + dt * Q / W.C) / (1.0 + dt / (W.Rd * W.C));
  W.pc_new = pc; W.Q = Q; W.p_o = pc + W.Rp * Q;
  return W.p_o;
}

template <class T>
__global__ void k_windkessel(DevMesh<T> M, const T* __restrict__ phi, WKDev* wk, const int* __restrict__ fptr,
                             const int* __restrict__ faces, double dt, double rho, T* __restrict__ bvp, Red red) {
  PDL_ENTRY();
  const int o = blockIdx.x;
  double q = 0;
  for (int i = fptr[o] + threadIdx.x; i < fptr[o + 1]; i += blockDim.x) q += (double)phi[M.F + faces[i]];
  __shared__ double sh[32][1];
  double v[1] = {q};
  block_sum<1>(v, sh);
  if (red.nranks > 1) {          // this rank's share of Q; k_windkessel_fin completes it
    if (threadIdx.x == 0) red.local[o] = v[0];
    return;
  }
  __shared__ double po_s;
  if (threadIdx.x == 0) po_s = wk_update(wk[o], v[0], dt) / rho;
  __syncthreads();
  for (int i = fptr[o] + threadIdx.x; i < fptr[o + 1]; i += blockDim.x) bvp[faces[i]] = (T)po_s;
}

// cross-rank Windkessel: Q = rank-order sum of the gathered shares
template <class T>
__global__ void k_windkessel_fin(const double* __restrict__ all, int P, int n_wk, WKDev* wk,
                                 const int* __restrict__ fptr, const int* __restrict__ faces, double dt, double rho,
                                 T* __restrict__ bvp) {
  PDL_ENTRY();
  const int o = blockIdx.x;
  __shared__ double po_s;
  if (threadIdx.x == 0) {
    double Q = 0;
    for (int r = 0; r < P; ++r) Q += all[r * n_wk + o];
    po_s = wk_update(wk[o], Q, dt) / rho;
  }
  __syncthreads();
  for (int i = fptr[o] + threadIdx.x; i < fptr[o + 1]; i += blockDim.x) bvp[faces[i]] = (T)po_s;
}

template <class T>
__global__ void k_add_at(T* a, const T* b, int i) {
  PDL_ENTRY(); a[i] += b[i]; }

// ============================================================ Jacobi PCG
// r = b - A x; partials b.b, r.r, r.z  -> control start
template <class T>
__global__ void __launch_bounds__(kThreads) k_cg_init(DevMesh<T> M, const T* __restrict__ diag,
    const T* __restrict__ coef, const T* __restrict__ b, const T* __restrict__ x, T* __restrict__ r,
    double* partials, unsigned* ticket, KCtl* ctl, Red red) {
  PDL_ENTRY();
  double v[3] = {0, 0, 0};
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    T acc[1] = {live ? diag[row] * x[row] : T(0)};
    sell_apply<T, 1>(M, s, lane, coef, x, acc);
    if (live) {
      const T rr = b[row] - acc[0];
      r[row] = rr;
      v[0] += (double)b[row] * (double)b[row];
      v[1] += (double)rr * (double)rr;
      v[2] += (double)rr * (double)rr / (double)diag[row];
    }
  }
  double t[3];
  if (grid_sum<3>(v, partials, ticket, t)) red_finish<3>(red, CTL_CG_INIT, ctl, t);
}

// Three kernels per PCG iteration; the x update of iteration k is deferred
// into the p update of iteration k+1 (x is never read inside the loop), so
// per iteration the method moves 108 N + 24 F bytes (fp64) instead of
// 116 N + 24 F.  k_cg_final applies the last pending x update.
//   k_cg_p:    x += alpha_{k-1} pd_{k-1};  pd_k = r_k / diag + beta_k pd_{k-1}
//   k_cg_spmv: q = A pd_k; partial pd.q -> alpha_k
//   k_cg_r:    r_{k+1} = r_k - alpha_k q; partials r.r, r.z -> check, beta
template <class T>
__global__ void k_cg_p(int n, const T* __restrict__ r, const T* __restrict__ diag, T* __restrict__ pd,
                       T* __restrict__ x, const KCtl* ctl) {
  PDL_ENTRY();
  if (ctl->done) return;
  const T beta = (T)ctl->beta, alpha = (T)ctl->alpha;
  const bool first = ctl->it == 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const T z = r[i] / diag[i];
    if (first) { pd[i] = z; continue; }
    const T po = pd[i];
    x[i] += alpha * po;
    pd[i] = z + beta * po;
  }
}

// q = A pd; partial pd.q -> alpha
template <class T>
__global__ void __launch_bounds__(kThreads) k_cg_spmv(DevMesh<T> M, const T* __restrict__ diag,
    const T* __restrict__ coef, const T* __restrict__ pd, T* __restrict__ q, double* partials, unsigned* ticket,
    KCtl* ctl, Red red) {
  PDL_ENTRY();
  if (ctl->done) return;
  double v[1] = {0};
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    const T pr = live ? pd[row] : T(0);
    T acc[1] = {live ? diag[row] * pr : T(0)};
    sell_apply<T, 1>(M, s, lane, coef, pd, acc);
    if (live) { q[row] = acc[0]; v[0] += (double)pr * (double)acc[0]; }
  }
  double t[1];
  if (grid_sum<1>(v, partials, ticket, t)) red_finish<1>(red, CTL_CG_SPMV, ctl, t);
}

template <class T>
__global__ void k_cg_r(int n, const T* __restrict__ q, const T* __restrict__ diag, T* __restrict__ r,
                       double* partials, unsigned* ticket, KCtl* ctl, Red red) {
  PDL_ENTRY();
  if (ctl->done) return;
  const T alpha = (T)ctl->alpha;
  double v[2] = {0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const T rr = r[i] - alpha * q[i];
    r[i] = rr;
    v[0] += (double)rr * (double)rr;
    v[1] += (double)rr * (double)rr / (double)diag[i];
  }
  double t[2];
  if (grid_sum<2>(v, partials, ticket, t)) red_finish<2>(red, CTL_CG_R, ctl, t);
}

// ---- AMG-preconditioned variant: z = M^-1 r comes from amg_apply
template <class T>
__global__ void k_cg_p2(int n, const T* __restrict__ z, T* __restrict__ pd, T* __restrict__ x, const KCtl* ctl) {
  PDL_ENTRY();
  if (ctl->done) return;
  const T beta = (T)ctl->beta, alpha = (T)ctl->alpha;
  const bool first = ctl->it == 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (first) { pd[i] = z[i]; continue; }
    const T po = pd[i];
    x[i] += alpha * po;
    pd[i] = z[i] + beta * po;
  }
}
template <class T>
__global__ void k_cg_r2(int n, const T* __restrict__ q, T* __restrict__ r, double* partials, unsigned* ticket,
                        KCtl* ctl, Red red) {
  PDL_ENTRY();
  if (ctl->done) return;
  const T alpha = (T)ctl->alpha;
  double v[1] = {0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const T rr = r[i] - alpha * q[i];
    r[i] = rr;
    v[0] += (double)rr * (double)rr;
  }
  double t[1];
  if (grid_sum<1>(v, partials, ticket, t)) red_finish<1>(red, CTL_CG_R2, ctl, t);
}
// r -= alpha q, partial r.r (-> check), fused with the AMG level-0
// pre-smoothing from zero x0 = r * il1 in the hierarchy's type P (the same
// expression as k_amg_pre, so the cycle is bitwise unchanged)
template <class T, class P>
__global__ void k_cg_r2x(int n, const T* __restrict__ q, T* __restrict__ r, const P* __restrict__ il1,
                         P* __restrict__ x0, double* partials, unsigned* ticket, KCtl* ctl, Red red) {
  PDL_ENTRY();
  if (ctl->done) return;
  const T alpha = (T)ctl->alpha;
  double v[1] = {0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const T rr = r[i] - alpha * q[i];
    r[i] = rr;
    x0[i] = (P)((P)rr * il1[i]);
    v[0] += (double)rr * (double)rr;
  }
  double t[1];
  if (grid_sum<1>(v, partials, ticket, t)) red_finish<1>(red, CTL_CG_R2, ctl, t);
}
template <class T>
__global__ void k_cg_dot(int n, const T* __restrict__ a, const T* __restrict__ b, double* partials, unsigned* ticket,
                         KCtl* ctl, Red red, int kind) {
  PDL_ENTRY();
  if (ctl->done) return;
  double v[1] = {0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[0] += (double)a[i] * (double)b[i];
  double t[1];
  if (grid_sum<1>(v, partials, ticket, t)) red_finish<1>(red, kind, ctl, t);
}

// the deferred x update of the final iteration
template <class T>
__global__ void k_cg_final(int n, const T* __restrict__ pd, T* __restrict__ x, const KCtl* ctl) {
  PDL_ENTRY();
  if (!ctl->half) return;
  const T alpha = (T)ctl->alpha;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] += alpha * pd[i];
}

// ============================================================ BiCGStab (NC components)
// Right-preconditioned (Jacobi) van der Vorst BiCGStab, the NC components
// (3 velocity components, or 1 transported scalar) advanced together over one
// coefficient stream; each component keeps its own scalars and stops
// independently.  The reductions always carry 3 component slots (zeros for
// k >= NC: those components start with b = 0 and are done from the start).
__device__ __forceinline__ bool all_done(const KCtl* c) { return c[0].done && c[1].done && c[2].done; }

// Gather of an NC-vector: NC scalar loads (measured on C5: dev.cuh's
// two-load ld3 made k_bi_t slower here, 0.53 against 0.64 of the roofline)
template <class T, int NC>
__device__ __forceinline__ void ldv(const T* __restrict__ p, int64_t i, T (&o)[3]) {
#pragma unroll
  for (int k = 0; k < NC; ++k) o[k] = p[NC * i + k];
}

// The BiCGStab vectors are kept SCALED by the Jacobi preconditioner
// D^-1 = 1 / diag (round 2): r~ = D^-1 r, v~ = D^-1 v and y = D^-1 p
// replace r, v, p, so the two matrix applies gather one (v: y) or two
// (t: r~, v~) NC-vectors per neighbour and no 1/diag:
//   p update    y = r~ + beta (y - omega v~)             (= D^-1 (r + beta (p - omega v)))
//   v = A y,    v~ = D^-1 v,  alpha = rho / (rh, v)
//   z = r~ - alpha v~ (= D^-1 s, formed on the fly), t = A z, s = D z
//   x += alpha y + omega z,   r = s - omega t,  r~ = D^-1 r
// The dot products use the unscaled r, v, s, t (the scalars of the
// textbook recurrence); the shadow residual rh stays unscaled.
template <class T, int NC>
__global__ void __launch_bounds__(kThreads) k_bi_init(DevMesh<T> M, const T* __restrict__ diag,
    const T* __restrict__ dinv, const T* __restrict__ coef, const T* __restrict__ b, const T* __restrict__ x,
    T* __restrict__ rs, T* __restrict__ rh, T* __restrict__ y, T* __restrict__ vs, double* partials, unsigned* ticket,
    KCtl* ctl, Red red) {
  PDL_ENTRY();
  double a[6] = {0, 0, 0, 0, 0, 0};
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    T acc[NC];
    const T d = live ? diag[row] : T(0);
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = live ? d * x[NC * (int64_t)row + k] : T(0);
    sell_apply<T, NC>(M, s, lane, coef, x, acc);
    if (live) {
      const T di = dinv[row];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int64_t i = NC * (int64_t)row + k;
        const T rr = b[i] - acc[k];
        rs[i] = rr * di; rh[i] = rr; y[i] = T(0); vs[i] = T(0);
        a[k] += (double)b[i] * (double)b[i];
        a[3 + k] += (double)rr * (double)rr;
      }
    }
  }
  double t[6];
  if (grid_sum<6>(a, partials, ticket, t)) red_finish<6>(red, CTL_BI_INIT, ctl, t);
}

// 1 / diag for own + ghost rows (the Jacobi preconditioner applied as a product)
template <class T>
__global__ void k_recip(int n, const T* __restrict__ d, T* __restrict__ di) {
  PDL_ENTRY();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) di[i] = T(1) / d[i];
}

// Per iteration (4 kernels): y update | v = A y, v~, rh.v -> alpha |
// z = r~ - alpha v~ on the fly, t = A z, t.s, t.t, s.s -> half-step check,
// omega | x, r~ update, rh.r, r.r -> rho, check.

// y = r~ + beta (y - omega v~)
template <class T, int NC>
__global__ void k_bi_p(int n, const T* __restrict__ rs, const T* __restrict__ vs, T* __restrict__ y, const KCtl* ctl) {
  PDL_ENTRY();
  if (all_done(ctl)) return;
  T beta[3], om[3];
  bool act[3];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    act[k] = !ctl[k].done;
    beta[k] = (T)((ctl[k].rho / ctl[k].rho_old) * (ctl[k].alpha / ctl[k].omega));
    om[k] = (T)ctl[k].omega;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (!act[k]) continue;
      const int64_t j = NC * (int64_t)i + k;
      y[j] = rs[j] + beta[k] * (y[j] - om[k] * vs[j]);
    }
  }
}

// v = A y; v~ = v / diag; partial (rh, v) -> alpha
template <class T, int NC, int KBV, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_bi_v(DevMesh<T> M, const T* __restrict__ diag,
    const T* __restrict__ dinv, const T* __restrict__ coef, const T* __restrict__ y, const T* __restrict__ rh,
    T* __restrict__ vs, double* partials, unsigned* ticket, KCtl* ctl, Red red) {
  PDL_ENTRY();
  if (all_done(ctl)) return;
  double a[3] = {0, 0, 0};
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    T acc[3];
    const T d = live ? diag[row] : T(0);
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = live ? d * y[NC * (int64_t)row + k] : T(0);
    const int len = __ldg(&M.ms_len[s]);
    const int base = __ldg(&M.ms_ptr[s]) + lane;
    for (int j = 0; j < len; j += KBV) {
      T c[KBV], yn[KBV][3];
      int nn[KBV];
#pragma unroll
      for (int u = 0; u < KBV; ++u) {
        const bool ok = j + u < len;
        c[u] = ok ? __ldg(&coef[base + 32 * (j + u)]) : T(0);
        nn[u] = ok ? __ldg(&M.mnb[base + 32 * (j + u)]) : 0;   // past the row's end: 0 * y_0
      }
#pragma unroll
      for (int u = 0; u < KBV; ++u) ldv<T, NC>(y, nn[u], yn[u]);
#pragma unroll
      for (int u = 0; u < KBV; ++u)
#pragma unroll
        for (int k = 0; k < NC; ++k) acc[k] += c[u] * yn[u][k];
    }
    if (live) {
      const T di = dinv[row];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int64_t i = NC * (int64_t)row + k;
        vs[i] = acc[k] * di;
        a[k] += (double)rh[i] * (double)acc[k];
      }
    }
  }
  double t[3];
  if (grid_sum<3>(a, partials, ticket, t)) red_finish<3>(red, CTL_BI_V, ctl, t);
}

// z = r~ - alpha v~ (own row and, on the fly, every neighbour); t = A z;
// s = diag z; partials (t, s), (t, t), (s, s) -> half-step check, omega
template <class T, int NC, int KBT, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_bi_t(DevMesh<T> M, const T* __restrict__ diag,
    const T* __restrict__ coef, const T* __restrict__ rs, const T* __restrict__ vs, T* __restrict__ tv,
    double* partials, unsigned* ticket, KCtl* ctl, Red red) {
  PDL_ENTRY();
  if (all_done(ctl)) return;
  T al[3];
#pragma unroll
  for (int k = 0; k < NC; ++k) al[k] = (T)ctl[k].alpha;
  double a[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  SLICE_LOOP(M) {
    const int row = s * 32 + lane;
    const bool live = row < M.n_own;
    T acc[3] = {T(0), T(0), T(0)}, sr[3] = {T(0), T(0), T(0)};
    if (live) {
      const T d = diag[row];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int64_t i = NC * (int64_t)row + k;
        sr[k] = d * (rs[i] - al[k] * vs[i]);
        acc[k] = sr[k];                    // diag * z
      }
    }
    const int len = __ldg(&M.ms_len[s]);
    const int base = __ldg(&M.ms_ptr[s]) + lane;
    for (int j = 0; j < len; j += KBT) {
      T c[KBT], rn[KBT][3], vn[KBT][3];
      int nn[KBT];
#pragma unroll
      for (int u = 0; u < KBT; ++u) {
        const bool ok = j + u < len;
        c[u] = ok ? __ldg(&coef[base + 32 * (j + u)]) : T(0);
        nn[u] = ok ? __ldg(&M.mnb[base + 32 * (j + u)]) : 0;   // past the row's end: 0 * z_0
      }
#pragma unroll
      for (int u = 0; u < KBT; ++u) { ldv<T, NC>(rs, nn[u], rn[u]); ldv<T, NC>(vs, nn[u], vn[u]); }
#pragma unroll
      for (int u = 0; u < KBT; ++u)
#pragma unroll
        for (int k = 0; k < NC; ++k) acc[k] += c[u] * (rn[u][k] - al[k] * vn[u][k]);
    }
    if (live)
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        tv[NC * (int64_t)row + k] = acc[k];
        a[k] += (double)acc[k] * (double)sr[k];
        a[3 + k] += (double)acc[k] * (double)acc[k];
        a[6 + k] += (double)sr[k] * (double)sr[k];
      }
  }
  double t[9];
  if (grid_sum<9>(a, partials, ticket, t)) red_finish<9>(red, CTL_BI_T, ctl, t);
}

// z = r~ - alpha v~; x += alpha y + omega z; r = diag z - omega t, r~ = r / diag;
// partials (rh, r), (r, r)
template <class T, int NC>
__global__ void k_bi_x(int n, const T* __restrict__ diag, const T* __restrict__ dinv, const T* __restrict__ y,
                       const T* __restrict__ vs, const T* __restrict__ tv, const T* __restrict__ rh, T* __restrict__ x,
                       T* __restrict__ rs, double* partials, unsigned* ticket, KCtl* ctl, Red red) {
  PDL_ENTRY();
  if (all_done(ctl)) return;
  T al[3], om[3];
  int mode[3];   // 0 skip, 1 half step, 2 full step
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    mode[k] = ctl[k].done ? 0 : (ctl[k].half ? 1 : 2);
    al[k] = (T)ctl[k].alpha; om[k] = (T)ctl[k].omega;
  }
  double a[6] = {0, 0, 0, 0, 0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const T d = diag[i], di = dinv[i];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int64_t j = NC * (int64_t)i + k;
      if (mode[k] == 1) { x[j] += al[k] * y[j]; continue; }
      if (mode[k] != 2) continue;
      const T z = rs[j] - al[k] * vs[j];
      x[j] += al[k] * y[j] + om[k] * z;
      const T rr = d * z - om[k] * tv[j];
      rs[j] = rr * di;
      a[k] += (double)rh[j] * (double)rr;
      a[3 + k] += (double)rr * (double)rr;
    }
  }
  double t[6];
  if (grid_sum<6>(a, partials, ticket, t)) red_finish<6>(red, CTL_BI_X, ctl, t);
}

// ============================================================ host side
struct SolverBase {
  virtual ~SolverBase() {}
};

template <class T>
struct SolverT : SolverBase {
  dfvm_mesh* m = nullptr;
  DevMesh<T>* M = nullptr;
  std::vector<void*> allocs;
  T *gU = nullptr, *gp = nullptr, *bU = nullptr, *rhsU = nullptr, *udiag = nullptr, *udinv = nullptr, *ucoef = nullptr;
  T* ucoefT = nullptr;          // transposed momentum coefficients (NEXT-3 adjoint apply)
  T *rAU = nullptr, *HbyA = nullptr, *phiHbyA = nullptr, *pcoef = nullptr, *pdiag = nullptr;
  T *prhs0 = nullptr, *prhs = nullptr;
  T *kr = nullptr, *krh = nullptr, *kp = nullptr, *kq = nullptr, *kv = nullptr, *kt = nullptr;
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  KCtl* d_ctl = nullptr;
  KCtl* h_ctl = nullptr;   // pinned
  double* d_cont = nullptr;
  double* h_cont = nullptr;  // pinned
  double* red_local = nullptr;  // [8] this rank's reduction totals (P > 1)
  double* red_all = nullptr;    // [P][8] all-gathered totals
  V4<T>* fdO = nullptr;         // x_f - x_O / x_f - x_N per local internal face (SOU / QUICK)
  V4<T>* fdN = nullptr;
  Amg<T>* amg = nullptr;        // pressure preconditioner (p_precond 1 / 2), built lazily
  bool amg_dirty = true;        // pressure matrix changed since the last Galerkin update
  // AMG side stream: the step's pressure matrix (rAU -> pcoef, pdiag) and
  // the hierarchy values are computed there while the momentum BiCGStab
  // runs on the caller's stream (one rank, no profiling); the first pressure
  // solve of the step waits for side_done
  cudaStream_t side = nullptr;
  cudaEvent_t side_start = nullptr, side_done = nullptr;
  bool side_pending = false;
  T* kz = nullptr;              // preconditioned residual z = M^-1 r
  WKDev* d_wk = nullptr;
  WKDev* h_wk = nullptr;     // pinned
  int* d_wk_ptr = nullptr;
  int* d_wk_faces = nullptr;
  bool assembled = false;
  // device-resident Krylov solves: one CUDA graph per (solver kind, x, b):
  // prologue, a conditional WHILE node whose body is one iteration (the last
  // body kernel sets the condition from the control block), epilogue
  struct LoopGraph { int kind; const void* x; const void* b; cudaGraphExec_t exec; int nl_fixed, nl_body; };
  std::vector<LoopGraph> loops;
  bool loops_off = false;
  // reports of device-resident solves, read back at the next stream sync
  static constexpr int kSlots = 48;
  KCtl* h_slots = nullptr;           // pinned [kSlots][3]
  struct Pending { int slot, nctl; dfvm_solve_report* rep; int nl_fixed, nl_body; };
  std::vector<Pending> pending;
  T* Uold = nullptr;     // start-of-step U and phi (ddtCorr, A-42; allocated on first use)
  T* phiold = nullptr;
  ~SolverT() override {
    if (side_start) cudaEventDestroy(side_start);
    if (side_done) cudaEventDestroy(side_done);
    if (side) cudaStreamDestroy(side);
    cudaDeviceSynchronize();
    for (auto& g : loops) cudaGraphExecDestroy(g.exec);
    if (h_slots) cudaFreeHost(h_slots);
    if (amg) amg_destroy<T>(amg);
    for (void* p : allocs) dev_free(p, nullptr);
    dev_free(d_wk, nullptr);
    dev_free(d_wk_ptr, nullptr);
    dev_free(d_wk_faces, nullptr);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (h_cont) cudaFreeHost(h_cont);
    if (h_wk) cudaFreeHost(h_wk);
  }
  // zero-filled workspace on stream s (the legacy stream at create time,
  // the caller's stream for lazy allocations inside a step)
  template <class U>
  dfvm_status al(U** p, size_t n, cudaStream_t s = nullptr) {
    if (dfvm_status st = dev_alloc_n(p, n, s, true)) return st;
    allocs.push_back((void*)*p);
    return DFVM_OK;
  }
  // face-to-cell displacements for the deferred-correction schemes (O-1 fp64
  // geometry in the renumbered orientation)
  dfvm_status build_face_offsets() {
    if (fdO) return DFVM_OK;
    const HostMesh& H = m->H;
    const Part& P = m->part;
    const size_t F = P.lf_gid.size();
    std::vector<V4<T>> o(std::max<size_t>(F, 1)), n(std::max<size_t>(F, 1));
    for (size_t i = 0; i < F; ++i) {
      const int64_t k = P.lf_gid[i];
      const double* xf = &H.xf0[3 * (int64_t)H.fold_of_new[k]];
      const double* xo = &H.xc0[3 * (int64_t)H.old_of_new[H.own[k]]];
      const double* xn = &H.xc0[3 * (int64_t)H.old_of_new[H.nb[k]]];
      o[i] = V4<T>{(T)(xf[0] - xo[0]), (T)(xf[1] - xo[1]), (T)(xf[2] - xo[2]), T(0)};
      n[i] = V4<T>{(T)(xf[0] - xn[0]), (T)(xf[1] - xn[1]), (T)(xf[2] - xn[2]), T(0)};
    }
    dfvm_status st;
    if ((st = al(&fdO, o.size())) || (st = al(&fdN, n.size()))) return st;
    DFVM_CUDA(cudaMemcpy(fdO, o.data(), o.size() * sizeof(V4<T>), cudaMemcpyHostToDevice));
    DFVM_CUDA(cudaMemcpy(fdN, n.data(), n.size() * sizeof(V4<T>), cudaMemcpyHostToDevice));
    DFVM_CUDA(cudaStreamSynchronize(nullptr));
    return DFVM_OK;
  }
  dfvm_status init(dfvm_mesh* mm, DevMesh<T>* MM) {
    m = mm; M = MM;
    const size_t nc = M->n_cells, no = M->n_own, nf = (size_t)M->F + M->B + M->E;
    dfvm_status st;
    if ((st = al(&gU, 9 * nc)) || (st = al(&gp, 3 * nc)) || (st = al(&bU, 3 * no)) || (st = al(&rhsU, 3 * no)) ||
        (st = al(&udiag, nc)) || (st = al(&udinv, nc)) || (st = al(&ucoef, (size_t)M->n_minc)) ||
        (st = al(&ucoefT, (size_t)M->n_minc)) || (st = al(&rAU, nc)) ||
        (st = al(&HbyA, 3 * nc)) || (st = al(&phiHbyA, nf)) || (st = al(&pcoef, (size_t)M->n_minc)) ||
        (st = al(&pdiag, nc)) || (st = al(&prhs0, no)) || (st = al(&prhs, no)) || (st = al(&kr, 3 * nc)) ||
        (st = al(&krh, 3 * nc)) || (st = al(&kp, 3 * nc)) || (st = al(&kq, 3 * nc)) || (st = al(&kv, 3 * nc)) ||
        (st = al(&kt, 3 * nc)) || (st = al(&kz, nc)) ||
        (st = al(&partials, (size_t)kMaxBlocks * 16)) || (st = al(&ticket, 4)) || (st = al(&d_ctl, 4)) ||
        (st = al(&d_cont, 8)) || (st = al(&red_local, 128)) || (st = al(&red_all, (size_t)128 * mm->part.P)))
      return st;
    DFVM_CUDA(cudaMallocHost(&h_ctl, 4 * sizeof(KCtl)));
    DFVM_CUDA(cudaMallocHost(&h_slots, (size_t)kSlots * 3 * sizeof(KCtl)));
    DFVM_CUDA(cudaMallocHost(&h_cont, 4 * sizeof(double)));
    DFVM_CUDA(cudaStreamSynchronize(nullptr));   // zero-fills complete before any use on the caller's stream
    return DFVM_OK;
  }
};

}  // namespace dfvm

using namespace dfvm;

struct dfvm_solver {
  dfvm_mesh* m = nullptr;
  dfvm_bcs* b = nullptr;
  dfvm_piso_opts o{};
  std::unique_ptr<SolverBase> impl;
  int ref_row = -1;
  bool fixed_p = false;
  int kcorr = 1;
  // Windkessel outlets (host description)
  struct WK { int patch; double Rp, C, Rd, pc; int scheme; };
  std::vector<WK> wk;
  bool wk_dirty = true;
  int n_launch = 0;
  double t = 0;   // solver time t^n (advanced by dt per PISO step; time-varying BCs use t^n + dt, A-41)
  // live kernel timing (CUDA events on the launching stream): class 0 = the
  // PCG SpMV kernel, class 1 = one full PCG iteration (3 kernels)
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  double t_ms[4] = {0, 0, 0, 0};
  int64_t t_n[4] = {0, 0, 0, 0};
  // per-kernel profile (dfvm_solver_profile; prof.h)
  Prof prof;
  Prof* pr() { return prof.on ? &prof : nullptr; }
  ~dfvm_solver() { for (auto e : ev) cudaEventDestroy(e); }
};

namespace dfvm {

// time scheme -> theta (Table 1, reading A-40)
static double theta_of(const dfvm_piso_opts& o) {
  return o.time_scheme == DFVM_TIME_CRANK_NICOLSON ? 0.5 : o.time_scheme == DFVM_TIME_FORWARD_EULER ? 0.0 : 1.0;
}

static bool solver_has_fixed_p(const dfvm_solver* S) {
  const HostMesh& H = S->m->H;
  for (size_t p = 0; p < H.pkind.size(); ++p)
    if (H.pkind[p] != DFVM_PATCH_EMPTY && S->b->set[1][p] &&
        (S->b->spec[1][p].kind == DFVM_BC_FIXED_VALUE || S->b->spec[1][p].kind == DFVM_BC_WINDKESSEL))
      return true;
  return false;
}

template <class T>
static dfvm_status sync_wk(dfvm_solver* S, SolverT<T>& X, cudaStream_t st) {
  if (!S->wk_dirty) return DFVM_OK;
  const Part& P = S->m->part;
  const HostMesh& H = S->m->H;
  const int n = (int)S->wk.size();
  if (X.d_wk) {
    dev_free(X.d_wk, st); dev_free(X.d_wk_ptr, st); dev_free(X.d_wk_faces, st);
    X.d_wk = nullptr; X.d_wk_ptr = nullptr; X.d_wk_faces = nullptr;
  }
  if (X.h_wk) { cudaFreeHost(X.h_wk); X.h_wk = nullptr; }
  if (n) {
    std::vector<int> ptr(n + 1, 0), faces;
    for (int o = 0; o < n; ++o) {
      for (int64_t b = 0; b < P.n_lb; ++b)
        if (H.bpatch[P.lb_gid[b] - H.F] == S->wk[o].patch) faces.push_back((int)b);
      ptr[o + 1] = (int)faces.size();
    }
    dfvm_status e;
    if ((e = dev_alloc_n(&X.d_wk, n, st, false)) || (e = dev_alloc_n(&X.d_wk_ptr, n + 1, st, false)) ||
        (e = dev_alloc_n(&X.d_wk_faces, faces.size(), st, false)))
      return e;
    DFVM_CUDA(cudaMallocHost(&X.h_wk, n * sizeof(WKDev)));
    for (int o = 0; o < n; ++o) {
      const auto& w = S->wk[o];
      X.h_wk[o] = WKDev{w.Rp, w.C, w.Rd, w.pc, w.pc, 0.0, 0.0, w.scheme, w.patch};
    }
    DFVM_CUDA(cudaMemcpyAsync(X.d_wk, X.h_wk, n * sizeof(WKDev), cudaMemcpyHostToDevice, st));
    DFVM_CUDA(cudaMemcpyAsync(X.d_wk_ptr, ptr.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
    if (!faces.empty())
      DFVM_CUDA(cudaMemcpyAsync(X.d_wk_faces, faces.data(), faces.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    DFVM_CUDA(cudaStreamSynchronize(st));
  }
  S->wk_dirty = false;
  return DFVM_OK;
}

static void fill_report(const KCtl& c, dfvm_solve_report* r) {
  r->it = c.it; r->res0 = c.res0; r->res = c.res; r->converged = c.converged;
}

constexpr int kChunk = 8;

dfvm_status allgather_f64(dfvm_mesh* m, const double* local, double* gathered, int n, cudaStream_t s);

// cross-rank completion of a reduction: all-gather of the per-rank totals
// then the rank-order sum + control step (k_finalize); no-op on one rank
template <class T>
static dfvm_status fin(dfvm_solver* S, SolverT<T>& X, int kind, int nv, cudaStream_t st) {
  if (S->m->part.P == 1) return DFVM_OK;
  if (dfvm_status e = allgather_f64(S->m, X.red_local, X.red_all, nv, st)) return e;
  PLAUNCH(S->pr(), "k_finalize", -1, 0, st, (k_finalize<<<1, 1, 0, st>>>(kind, nv, X.red_all, S->m->part.P, X.d_ctl)));
  S->n_launch++;
  return DFVM_OK;
}

// ---------------------------------------------------------------- solves
// Each Krylov solve is a prologue (initial residual, first preconditioner
// application), an iteration body and an epilogue (the deferred last x
// update, x = 0 for b = 0).  Two drivers run them:
//  * device-resident (one rank, a non-legacy stream, no profiling): the solve
//    is ONE CUDA graph — prologue, a conditional WHILE node whose body is one
//    iteration ending in k_loop_cond (continue while the control block is not
//    done), epilogue — captured on first use per (kind, x, b) and replayed;
//    no host synchronisation and no launch after convergence.  The control
//    block is copied to a pinned report slot and read at the next stream
//    synchronisation (the end of the step, or of the standalone call);
//  * host-chunked (several ranks with host-side transports, the legacy
//    stream, profiling, DFVM_GRAPHS=0): kChunk iterations enqueued per host
//    round trip, every kernel exiting early on the done flag.
enum LoopKind { LOOP_CG = 0, LOOP_CG_AMG = 1, LOOP_BICGSTAB = 2, LOOP_BICGSTAB1 = 3 };

__global__ void k_loop_cond(cudaGraphConditionalHandle h, const KCtl* ctl, int nc) {
  PDL_ENTRY();
  int go = 0;
  for (int k = 0; k < nc; ++k) go |= !ctl[k].done;
  cudaGraphSetConditional(h, go ? 1u : 0u);
}

template <class T>
__global__ void k_zero_if(int n, int nc, T* __restrict__ x, const KCtl* ctl) {
  PDL_ENTRY();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int k = 0; k < nc; ++k)
      if (ctl[k].zero_x) x[(int64_t)nc * i + k] = T(0);
}

template <class T>
static bool use_device_loops(dfvm_solver* S, SolverT<T>& X, cudaStream_t st) {
  if (X.loops_off) return false;
  const char* g = getenv("DFVM_GRAPHS");
  if (g && g[0] == '0') { X.loops_off = true; return false; }
  return S->m->part.P == 1 && st != nullptr && !S->pr() && !S->timing;
}

// Programmatic dependent launch inside a captured graph: every edge between
// two kernel nodes becomes a programmatic one, so the downstream kernel's
// blocks are scheduled as soon as the upstream kernel's blocks have all begun
// (DFVM_PDL=2, default; the launch-completion port) or have all finished
// (DFVM_PDL=1, the programmatic port: only the launch itself overlaps),
// instead of after the upstream grid has drained and flushed.  Correctness
// rests on PDL_ENTRY (dev.cuh): every kernel waits for its dependencies'
// completion and memory before it touches anything.  DFVM_PDL=0: ordinary
// edges.  Returns the number of edges converted.
static int make_programmatic(cudaGraph_t g) {
  const int mode = [] { const char* e = getenv("DFVM_PDL"); return e ? atoi(e) : 2; }();
  if (mode <= 0) return 0;
  size_t ne = 0;
  if (cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne) != cudaSuccess || ne == 0) return 0;
  std::vector<cudaGraphNode_t> from(ne), to(ne);
  std::vector<cudaGraphEdgeData> ed(ne);
  if (cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne) != cudaSuccess) return 0;
  int n = 0;
  for (size_t k = 0; k < ne; ++k) {
    cudaGraphNodeType ta, tb;
    if (cudaGraphNodeGetType(from[k], &ta) != cudaSuccess || cudaGraphNodeGetType(to[k], &tb) != cudaSuccess) continue;
    if (ta != cudaGraphNodeTypeKernel || tb != cudaGraphNodeTypeKernel) continue;
    if (ed[k].type != cudaGraphDependencyTypeDefault || ed[k].from_port != 0) continue;
    cudaGraphEdgeData pe = {};
    pe.type = cudaGraphDependencyTypeProgrammatic;
    pe.from_port = mode == 1 ? cudaGraphKernelNodePortProgrammatic : cudaGraphKernelNodePortLaunchCompletion;
    if (cudaGraphRemoveDependencies_v2(g, &from[k], &to[k], &ed[k], 1) != cudaSuccess) continue;
    if (cudaGraphAddDependencies_v2(g, &from[k], &to[k], &pe, 1) != cudaSuccess) {
      cudaGraphAddDependencies_v2(g, &from[k], &to[k], &ed[k], 1);   // keep the ordinary edge
      continue;
    }
    ++n;
  }
  cudaGetLastError();
  return n;
}

template <class T, class Pro, class Body, class Epi>
static dfvm_status device_loop(dfvm_solver* S, SolverT<T>& X, int kind, const void* x, const void* b, int nctl,
                               dfvm_solve_report* rep, cudaStream_t st, Pro pro, Body body, Epi epi) {
  typename SolverT<T>::LoopGraph* L = nullptr;
  for (auto& g : X.loops)
    if (g.kind == kind && g.x == x && g.b == b) L = &g;
  if (!L) {
    cudaGraph_t g = nullptr, bg = nullptr;
    cudaGraphExec_t ex = nullptr;
    cudaGraphConditionalHandle h;
    int nl = 0, nb = 0;
    DFVM_CUDA(cudaGraphCreate(&g, 0));
    DFVM_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    DFVM_CUDA(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    dfvm_status ce = pro(&nl);
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaGraph_t cg = nullptr;
    cudaGraphNode_t cn = nullptr;
    cudaError_t err = cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (err == cudaSuccess) err = cudaGraphAddNode(&cn, g, deps, nd, &cp);
    if (err == cudaSuccess) err = cudaStreamUpdateCaptureDependencies(st, &cn, 1, cudaStreamSetCaptureDependencies);
    if (err == cudaSuccess && !ce) ce = epi(&nl);
    cudaError_t e2 = cudaStreamEndCapture(st, &g);
    if (err == cudaSuccess) err = e2;
    if (err == cudaSuccess && !ce) {
      bg = cp.conditional.phGraph_out[0];
      err = cudaStreamBeginCaptureToGraph(st, bg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      if (err == cudaSuccess) {
        ce = body(&nb);
        k_loop_cond<<<1, 1, 0, st>>>(h, X.d_ctl, nctl);
        ++nb;
        e2 = cudaStreamEndCapture(st, &bg);
        if (err == cudaSuccess) err = e2;
      }
    }
    if (err == cudaSuccess && !ce) {
      make_programmatic(g);
      make_programmatic(bg);
      err = cudaGraphInstantiate(&ex, g, 0);
    }
    if (g) cudaGraphDestroy(g);
    if (ce) return ce;
    if (err != cudaSuccess) return cuda_error(err, "device-resident Krylov graph");
    X.loops.push_back({kind, x, b, ex, nl, nb});
    L = &X.loops.back();
  }
  DFVM_CUDA(cudaGraphLaunch(L->exec, st));
  const int slot = (int)X.pending.size();
  if (slot >= SolverT<T>::kSlots) { set_error(DFVM_E_INVALID_ARG, "too many pending solves"); return DFVM_E_INVALID_ARG; }
  DFVM_CUDA(cudaMemcpyAsync(X.h_slots + 3 * slot, X.d_ctl, nctl * sizeof(KCtl), cudaMemcpyDeviceToHost, st));
  X.pending.push_back({slot, nctl, rep, L->nl_fixed, L->nl_body});
  return DFVM_OK;
}

static dfvm_status solve_status(const KCtl* c, int nctl) {
  dfvm_status res = DFVM_OK;
  for (int k = 0; k < nctl; ++k) {
    if (c[k].status == DFVM_E_BREAKDOWN) res = DFVM_E_BREAKDOWN;
    else if (!c[k].converged && res == DFVM_OK) res = DFVM_E_NOT_CONVERGED;
  }
  return res;
}

// after a stream synchronisation: reports, launch counts and the worst status
// of the device-resident solves enqueued since the last one
template <class T>
static dfvm_status resolve_pending(dfvm_solver* S, SolverT<T>& X) {
  dfvm_status res = DFVM_OK;
  for (const auto& p : X.pending) {
    const KCtl* c = X.h_slots + 3 * p.slot;
    int iters = 0;
    for (int k = 0; k < p.nctl; ++k) {
      if (p.rep) fill_report(c[k], &p.rep[k]);
      iters = std::max(iters, c[k].it);
    }
    S->n_launch += p.nl_fixed + (iters + 1) * p.nl_body;
    const dfvm_status st = solve_status(c, p.nctl);
    if (st == DFVM_E_BREAKDOWN || (st == DFVM_E_NOT_CONVERGED && res == DFVM_OK)) res = st;
  }
  X.pending.clear();
  return res;
}

// host-chunked driver: prologue, then chunks of kChunk iterations with one
// control-block read-back each, then the epilogue
struct NoHarvest { void operator()(int, bool) const {} };

template <class T, class Pro, class Body, class Epi, class Harvest = NoHarvest>
static dfvm_status chunk_loop(dfvm_solver* S, SolverT<T>& X, int nctl, dfvm_solve_report* rep, cudaStream_t st,
                              Pro pro, Body body, Epi epi, Harvest harvest = Harvest()) {
  Prof* pr = S->pr();
  dfvm_status e;
  if ((e = pro(&S->n_launch))) return e;
  int it_prof = 0;
  const bool prof_graph = pr && S->m->part.P == 1 && st != nullptr;
  auto iters = [&]() { int i = 0; for (int k = 0; k < nctl; ++k) i = std::max(i, X.h_ctl[k].it); return i; };
  auto all_done = [&]() { for (int k = 0; k < nctl; ++k) if (!X.h_ctl[k].done) return false; return true; };
  for (;;) {
    // profile mode: one iteration per captured chunk, so no launch after
    // convergence is timed (the device-resident loop makes none either)
    const int nchunk = pr ? 1 : kChunk;
    auto chunk = [&](int* nl) -> dfvm_status {
      for (int k = 0; k < nchunk; ++k) {
        if (pr) { pr->iter = k; pr->post = 0; }
        dfvm_status e3 = body(nl);
        if (e3) return e3;
      }
      return DFVM_OK;
    };
    if (prof_graph) {
      // profile mode: this chunk captured afresh with its event pairs as
      // graph nodes and replayed once (no host gap inside an event pair)
      cudaGraph_t g = nullptr;
      cudaGraphExec_t gx = nullptr;
      int nl = 0;
      pr->cut();
      DFVM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      const dfvm_status ce = chunk(&nl);
      DFVM_CUDA(cudaStreamEndCapture(st, &g));
      pr->cut();
      if (ce) { cudaGraphDestroy(g); return ce; }
      DFVM_CUDA(cudaGraphInstantiate(&gx, g, 0));
      cudaGraphDestroy(g);
      DFVM_CUDA(cudaGraphLaunch(gx, st));
      DFVM_CUDA(cudaStreamSynchronize(st));
      cudaGraphExecDestroy(gx);
      S->n_launch += nl;
    } else if ((e = chunk(&S->n_launch))) {
      return e;
    }
    DFVM_CUDA(cudaMemcpyAsync(X.h_ctl, X.d_ctl, nctl * sizeof(KCtl), cudaMemcpyDeviceToHost, st));
    DFVM_CUDA(cudaStreamSynchronize(st));
    harvest(iters() - it_prof, all_done());
    if (pr) {
      pr->harvest(iters() - it_prof, nctl == 1 && X.h_ctl[0].done != 0);
      pr->iter = -1; pr->post = 0;
    }
    it_prof = iters();
    if (all_done()) break;
  }
  DFVM_CUDA(cudaGetLastError());
  if ((e = epi(&S->n_launch))) return e;
  for (int k = 0; k < nctl; ++k)
    if (rep) fill_report(X.h_ctl[k], &rep[k]);
  return solve_status(X.h_ctl, nctl);
}

template <class T>
static dfvm_status run_cg_amg(dfvm_solver* S, SolverT<T>& X, const T* b, T* x, double tol, double rel_tol,
                              int maxit, dfvm_solve_report* rep, cudaStream_t st);

// Jacobi PCG on (pdiag, pcoef): x warm start, b rhs.  The x update of
// iteration k is deferred into the p update of iteration k+1 (x is never read
// inside the loop); k_cg_final applies the last pending one.
template <class T>
static dfvm_status run_cg(dfvm_solver* S, SolverT<T>& X, const T* b, T* x, double tol, double rel_tol, int maxit,
                          dfvm_solve_report* rep, cudaStream_t st) {
  if (S->o.p_precond >= 1) return run_cg_amg(S, X, b, x, tol, rel_tol, maxit, rep, st);
  DevMesh<T>& M = *X.M;
  dfvm_mesh* m = S->m;
  const Red red{m->part.P, X.red_local};
  const int gs = grid_slices(k_cg_spmv<T>, M.n_slices), ge = grid_for(M.n_own);
  const int gp = grid_rows(k_cg_p<T>, M.n_own), gr = grid_rows(k_cg_r<T>, M.n_own);
  Prof* pr = S->pr();
  const double v = sizeof(T), N = M.n_own, Z = (double)M.nnz;
  KCtl init{};
  init.tol = tol; init.rel_tol = rel_tol; init.maxit = maxit;
  DFVM_CUDA(cudaMemcpyAsync(X.d_ctl, &init, sizeof(KCtl), cudaMemcpyHostToDevice, st));
  if (S->timing && S->ev.size() < 4 * kChunk)
    while (S->ev.size() < 4 * kChunk) {
      cudaEvent_t ev;
      DFVM_CUDA(cudaEventCreate(&ev));
      S->ev.push_back(ev);
    }
  int k_ev = 0;
  auto pro = [&](int* nl) -> dfvm_status {
    dfvm_status e;
    if ((e = halo_exchange(m, x, 1, st))) return e;
    PLAUNCH(pr, "k_cg_init", -1, 4 * N + Z * (4 + v) + 4 * v * N, st,
            (k_cg_init<T><<<grid_slices(k_cg_init<T>, M.n_slices), kThreads, 0, st>>>(M, X.pdiag, X.pcoef, b, x,
                                                                                     X.kr, X.partials, X.ticket,
                                                                                     X.d_ctl, red)));
    ++*nl;
    return fin(S, X, CTL_CG_INIT, 3, st);
  };
  auto body = [&](int* nl) -> dfvm_status {
    dfvm_status e;
    const int k = k_ev++ % kChunk;
    if (S->timing) record_event(S->ev[4 * k], st);
    PLAUNCH(pr, "k_cg_p", -1, 6 * v * N, st, (k_cg_p<T><<<gp, kThreads, 0, st>>>(M.n_own, X.kr, X.pdiag, X.kp, x, X.d_ctl)));
    if ((e = halo_exchange(m, X.kp, 1, st))) return e;
    if (S->timing) record_event(S->ev[4 * k + 1], st);
    PLAUNCH(pr, "k_cg_spmv", -1, 4 * N + Z * (4 + v) + 3 * v * N, st,
            (k_cg_spmv<T><<<gs, kThreads, 0, st>>>(M, X.pdiag, X.pcoef, X.kp, X.kq, X.partials, X.ticket, X.d_ctl, red)));
    if (S->timing) record_event(S->ev[4 * k + 2], st);
    if ((e = fin(S, X, CTL_CG_SPMV, 1, st))) return e;
    PLAUNCH(pr, "k_cg_r", -1, 4 * v * N, st,
            (k_cg_r<T><<<gr, kThreads, 0, st>>>(M.n_own, X.kq, X.pdiag, X.kr, X.partials, X.ticket, X.d_ctl, red)));
    if ((e = fin(S, X, CTL_CG_R, 2, st))) return e;
    if (S->timing) record_event(S->ev[4 * k + 3], st);
    *nl += 3;
    return DFVM_OK;
  };
  auto epi = [&](int* nl) -> dfvm_status {
    PLAUNCH(pr, "k_cg_final", -1, 3 * v * N, st, (k_cg_final<T><<<ge, kThreads, 0, st>>>(M.n_own, X.kp, x, X.d_ctl)));
    k_zero_if<T><<<ge, kThreads, 0, st>>>(M.n_own, 1, x, X.d_ctl);
    *nl += 2;
    return DFVM_OK;
  };
  if (use_device_loops(S, X, st)) return device_loop(S, X, LOOP_CG, x, b, 1, rep, st, pro, body, epi);
  // live timing (dfvm_solver_set_timing): the SpMV and whole iterations of
  // the iterations that ran in each chunk
  auto harvest = [&](int ran, bool) {
    if (!S->timing) return;
    for (int k = 0; k < kChunk && k < ran; ++k) {
      float a = 0, b2 = 0;
      cudaEventElapsedTime(&a, S->ev[4 * k + 1], S->ev[4 * k + 2]);
      cudaEventElapsedTime(&b2, S->ev[4 * k], S->ev[4 * k + 3]);
      S->t_ms[0] += a; S->t_n[0]++;
      S->t_ms[1] += b2; S->t_n[1]++;
    }
  };
  return chunk_loop(S, X, 1, rep, st, pro, body, epi, harvest);
}

// PCG preconditioned by one AMG cycle (amg.cu).  Same
// stopping rule, same deferred x update; per iteration:
//   p update (z + beta p) | halo(p) | SpMV + p.q -> alpha | r update + r.r ->
//   check, fused with the level-0 pre-smoothing | z = M^-1 r, r.z folded into
//   the level-0 post-smoother -> beta.
template <class T>
static dfvm_status run_cg_amg(dfvm_solver* S, SolverT<T>& X, const T* b, T* x, double tol, double rel_tol,
                              int maxit, dfvm_solve_report* rep, cudaStream_t st) {
  DevMesh<T>& M = *X.M;
  dfvm_mesh* m = S->m;
  dfvm_status e;
  if (!X.amg && (e = amg_create<T>(m, M, S->o.p_precond == 2, &X.amg, st))) return e;
  Prof* pr = S->pr();
  const double v = sizeof(T), N = M.n_own, Z = (double)M.nnz;
  if (X.amg_dirty) {
    if ((e = amg_update<T>(X.amg, X.pcoef, X.pdiag, st, &S->n_launch, pr))) return e;
    X.amg_dirty = false;
  }
  const Red red{m->part.P, X.red_local};
  const int* done = &X.d_ctl->done;
  const int gs = grid_slices(k_cg_spmv<T>, M.n_slices), ge = grid_for(M.n_own);
  KCtl init{};
  init.tol = tol; init.rel_tol = rel_tol; init.maxit = maxit;
  DFVM_CUDA(cudaMemcpyAsync(X.d_ctl, &init, sizeof(KCtl), cudaMemcpyHostToDevice, st));
  const KDot dot0{X.partials, X.ticket, X.d_ctl, red, CTL_CG_RZ0}, dot1{X.partials, X.ticket, X.d_ctl, red, CTL_CG_RZ};
  void* x0f = nullptr;
  const void* il1f = nullptr;
  int pbf = 0;
  amg_level0_pre<T>(X.amg, &x0f, &il1f, &pbf);
  if (S->timing && S->ev.size() < 8 * kChunk)
    while (S->ev.size() < 8 * kChunk) {
      cudaEvent_t ev;
      DFVM_CUDA(cudaEventCreate(&ev));
      S->ev.push_back(ev);
    }
  int k_ev = 0;
  auto pro = [&](int* nl) -> dfvm_status {
    dfvm_status e2;
    if ((e2 = halo_exchange(m, x, 1, st))) return e2;
    PLAUNCH(pr, "k_cg_init", -1, 4 * N + Z * (4 + v) + 4 * v * N, st,
            (k_cg_init<T><<<grid_slices(k_cg_init<T>, M.n_slices), kThreads, 0, st>>>(M, X.pdiag, X.pcoef, b, x,
                                                                                     X.kr, X.partials, X.ticket,
                                                                                     X.d_ctl, red)));
    ++*nl;
    if ((e2 = fin(S, X, CTL_CG_INIT, 3, st))) return e2;
    // r.z is folded into the level-0 post-smoother when the cycle has one
    // (k_amg_smooth_dot), else a separate k_cg_dot
    bool dd = false;
    if ((e2 = amg_apply<T>(X.amg, X.kr, X.kz, done, st, nl, nullptr, pr, &dot0, false, &dd))) return e2;
    if (!dd) {
      PLAUNCH(pr, "k_cg_dot", -1, 2 * v * N, st,
              (k_cg_dot<T><<<ge, kThreads, 0, st>>>(M.n_own, X.kr, X.kz, X.partials, X.ticket, X.d_ctl, red, CTL_CG_RZ0)));
      ++*nl;
    }
    return fin(S, X, CTL_CG_RZ0, 1, st);
  };
  auto body = [&](int* nl) -> dfvm_status {
    dfvm_status e2;
    const int k = k_ev++ % kChunk;
    if (S->timing) record_event(S->ev[4 * k], st);
    PLAUNCH(pr, "k_cg_p2", -1, 5 * v * N, st, (k_cg_p2<T><<<ge, kThreads, 0, st>>>(M.n_own, X.kz, X.kp, x, X.d_ctl)));
    if ((e2 = halo_exchange(m, X.kp, 1, st))) return e2;
    if (S->timing) record_event(S->ev[4 * k + 1], st);
    PLAUNCH(pr, "k_cg_spmv", -1, 4 * N + Z * (4 + v) + 3 * v * N, st,
            (k_cg_spmv<T><<<gs, kThreads, 0, st>>>(M, X.pdiag, X.pcoef, X.kp, X.kq, X.partials, X.ticket, X.d_ctl, red)));
    if (S->timing) record_event(S->ev[4 * k + 2], st);
    if ((e2 = fin(S, X, CTL_CG_SPMV, 1, st))) return e2;
    if (pbf == 4) {
      PLAUNCH(pr, "k_cg_r2x", -1, 3 * v * N + 8 * N, st,
              (k_cg_r2x<T, float><<<ge, kThreads, 0, st>>>(M.n_own, X.kq, X.kr, (const float*)il1f, (float*)x0f,
                                                            X.partials, X.ticket, X.d_ctl, red)));
    } else if (pbf == 8) {
      PLAUNCH(pr, "k_cg_r2x", -1, 3 * v * N + 16 * N, st,
              (k_cg_r2x<T, double><<<ge, kThreads, 0, st>>>(M.n_own, X.kq, X.kr, (const double*)il1f, (double*)x0f,
                                                             X.partials, X.ticket, X.d_ctl, red)));
    } else {
      PLAUNCH(pr, "k_cg_r2", -1, 3 * v * N, st,
              (k_cg_r2<T><<<ge, kThreads, 0, st>>>(M.n_own, X.kq, X.kr, X.partials, X.ticket, X.d_ctl, red)));
    }
    if ((e2 = fin(S, X, CTL_CG_R2, 1, st))) return e2;
    if (pr) pr->post = 1;
    bool dd = false;
    if ((e2 = amg_apply<T>(X.amg, X.kr, X.kz, done, st, nl, S->timing ? &S->ev[4 * kChunk + 4 * k] : nullptr, pr,
                           &dot1, pbf != 0, &dd)))
      return e2;
    if (!dd) {
      PLAUNCH(pr, "k_cg_dot", -1, 2 * v * N, st,
              (k_cg_dot<T><<<ge, kThreads, 0, st>>>(M.n_own, X.kr, X.kz, X.partials, X.ticket, X.d_ctl, red, CTL_CG_RZ)));
      ++*nl;
    }
    if ((e2 = fin(S, X, CTL_CG_RZ, 1, st))) return e2;
    if (S->timing) record_event(S->ev[4 * k + 3], st);
    *nl += 3;
    return DFVM_OK;
  };
  auto epi = [&](int* nl) -> dfvm_status {
    PLAUNCH(pr, "k_cg_final", -1, 3 * v * N, st, (k_cg_final<T><<<ge, kThreads, 0, st>>>(M.n_own, X.kp, x, X.d_ctl)));
    k_zero_if<T><<<ge, kThreads, 0, st>>>(M.n_own, 1, x, X.d_ctl);
    *nl += 2;
    return DFVM_OK;
  };
  if (use_device_loops(S, X, st)) return device_loop(S, X, LOOP_CG_AMG, x, b, 1, rep, st, pro, body, epi);
  // live timing: SpMV, whole iteration, and the level-0 AMG kernels (recorded
  // only when the cycle ran: the last iteration of a solve skips it)
  auto harvest = [&](int ran, bool all_done) {
    if (!S->timing) return;
    for (int k = 0; k < kChunk && k < ran; ++k) {
      float a = 0, b2 = 0, c2 = 0, d2 = 0;
      cudaEventElapsedTime(&a, S->ev[4 * k + 1], S->ev[4 * k + 2]);
      cudaEventElapsedTime(&b2, S->ev[4 * k], S->ev[4 * k + 3]);
      S->t_ms[0] += a; S->t_n[0]++;
      S->t_ms[1] += b2; S->t_n[1]++;
      if (k + 1 < ran || !all_done) {
        cudaEvent_t* ea = &S->ev[4 * kChunk + 4 * k];
        if (cudaEventElapsedTime(&c2, ea[0], ea[1]) == cudaSuccess && cudaEventElapsedTime(&d2, ea[2], ea[3]) == cudaSuccess) {
          S->t_ms[2] += c2; S->t_n[2]++;
          S->t_ms[3] += d2; S->t_n[3]++;
        }
      }
    }
    cudaGetLastError();
  };
  return chunk_loop(S, X, 1, rep, st, pro, body, epi, harvest);
}

// 3-component BiCGStab on (udiag, ucoef): x = U (warm start), b = rhsU.
// Right-preconditioned (Jacobi) van der Vorst BiCGStab, the three velocity
// components advanced together over one coefficient stream; each component
// keeps its own scalars and stops independently; vectors kept scaled by
// 1 / diag (see k_bi_init).  Ghosts: x and udiag are exchanged by the caller
// (assemble); y, r~ and v~ are exchanged before the applies that gather them.
template <class T, int NC>
static dfvm_status run_bicgstab(dfvm_solver* S, SolverT<T>& X, const T* b, T* x, double tol, double rel_tol,
                                int maxit, dfvm_solve_report* rep, cudaStream_t st) {
  DevMesh<T>& M = *X.M;
  dfvm_mesh* m = S->m;
  const Red red{m->part.P, X.red_local};
  // k_bi_t: batch 4 at >= 3 blocks/SM (batch 2 at 4 blocks/SM measured equal on C5)
  // batch depth / min blocks per SM: measured on C5 against batch 2 and 1
  // with two-load 3-vector gathers (profiles/r01_bicgstab_variants_c5.txt)
  const int gs = grid_slices(k_bi_v<T, NC, 4, 6>, M.n_slices);
  // DFVM_BI_T=2: k_bi_t in batches of 2 entries at >= 4 blocks/SM (A/B knob)
  const int bi_t_var = [] { const char* e = getenv("DFVM_BI_T"); return e ? atoi(e) : 4; }();
  const int gt = bi_t_var == 2 ? grid_slices(k_bi_t<T, NC, 2, 4>, M.n_slices) : grid_slices(k_bi_t<T, NC, 4, 3>, M.n_slices);
  // (measured on C5: flat [3n] p/x updates and shared-staged own rows in v/t
  // were 26 ms/step slower than these one-thread-per-row kernels)
  const int ge = grid_for(M.n_own);
  Prof* pr = S->pr();
  const double v = sizeof(T), N = M.n_own, Z = (double)M.nnz;
  KCtl init[3] = {};
  for (int k = 0; k < 3; ++k) { init[k].tol = tol; init[k].rel_tol = rel_tol; init[k].maxit = maxit; }
  DFVM_CUDA(cudaMemcpyAsync(X.d_ctl, init, 3 * sizeof(KCtl), cudaMemcpyHostToDevice, st));
  auto pro = [&](int* nl) -> dfvm_status {
    PLAUNCH(pr, "k_recip", -1, 2 * v * M.n_cells, st,
            (k_recip<T><<<grid_for(M.n_cells), kThreads, 0, st>>>(M.n_cells, X.udiag, X.udinv)));
    PLAUNCH(pr, "k_bi_init", -1, 4 * N + Z * (4 + v) + (2 + 6 * NC) * v * N, st,
            (k_bi_init<T, NC><<<grid_slices(k_bi_init<T, NC>, M.n_slices), kThreads, 0, st>>>(M, X.udiag, X.udinv, X.ucoef, b, x, X.kr,
                                                                                     X.krh, X.kp, X.kv, X.partials,
                                                                                     X.ticket, X.d_ctl, red)));
    *nl += 2;
    return fin(S, X, CTL_BI_INIT, 6, st);
  };
  auto body = [&](int* nl) -> dfvm_status {
    dfvm_status e;
    PLAUNCH(pr, "k_bi_p", -1, 4 * NC * v * N, st, (k_bi_p<T, NC><<<ge, kThreads, 0, st>>>(M.n_own, X.kr, X.kv, X.kp, X.d_ctl)));
    if ((e = halo_exchange(m, X.kp, NC, st))) return e;
    PLAUNCH(pr, "k_bi_v", -1, 4 * N + Z * (4 + v) + (2 + 3 * NC) * v * N, st,
            (k_bi_v<T, NC, 4, 6><<<gs, kThreads, 0, st>>>(M, X.udiag, X.udinv, X.ucoef, X.kp, X.krh, X.kv, X.partials,
                                                      X.ticket, X.d_ctl, red)));
    if ((e = fin(S, X, CTL_BI_V, 3, st))) return e;
    if ((e = halo_exchange(m, X.kr, NC, st)) || (e = halo_exchange(m, X.kv, NC, st))) return e;
    PLAUNCH(pr, "k_bi_t", -1, 4 * N + Z * (4 + v) + (1 + 3 * NC) * v * N, st,
            if (bi_t_var == 2) {
              k_bi_t<T, NC, 2, 4><<<gt, kThreads, 0, st>>>(M, X.udiag, X.ucoef, X.kr, X.kv, X.kt, X.partials, X.ticket,
                                                            X.d_ctl, red);
            } else {
              k_bi_t<T, NC, 4, 3><<<gt, kThreads, 0, st>>>(M, X.udiag, X.ucoef, X.kr, X.kv, X.kt, X.partials, X.ticket,
                                                            X.d_ctl, red);
            });
    if ((e = fin(S, X, CTL_BI_T, 9, st))) return e;
    PLAUNCH(pr, "k_bi_x", -1, (2 + 8 * NC) * v * N, st,
            (k_bi_x<T, NC><<<ge, kThreads, 0, st>>>(M.n_own, X.udiag, X.udinv, X.kp, X.kv, X.kt, X.krh, x, X.kr, X.partials,
                                                X.ticket, X.d_ctl, red)));
    if ((e = fin(S, X, CTL_BI_X, 6, st))) return e;
    *nl += 4;
    return DFVM_OK;
  };
  auto epi = [&](int* nl) -> dfvm_status {
    // b = 0 components: x = 0
    k_zero_if<T><<<ge, kThreads, 0, st>>>(M.n_own, NC, x, X.d_ctl);
    ++*nl;
    return DFVM_OK;
  };
  if (use_device_loops(S, X, st))
    return device_loop(S, X, NC == 3 ? LOOP_BICGSTAB : LOOP_BICGSTAB1, x, b, NC, rep, st, pro, body, epi);
  return chunk_loop(S, X, NC, rep, st, pro, body, epi);
}

template <class T>
static dfvm_status assemble(dfvm_solver* S, SolverT<T>& X, const T* U, const T* phi, cudaStream_t st) {
  DevMesh<T>& M = *X.M;
  dfvm_bcs* b = S->b;
  dfvm_status s2;
  if ((s2 = bcs_device(b, 0, st)) || (s2 = bcs_device(b, 1, st))) return s2;
  if ((s2 = halo_exchange(S->m, (void*)U, 3, st))) return s2;
  const int gs = grid_for_slices(M.n_slices);
  Prof* pr = S->pr();
  const double v = sizeof(T), N = M.n_own, F = M.F, Bf = M.B;
  PLAUNCH(pr, "k_grad (U)", -1, 13 * v * N + (16 + 4 * v) * F + (9 + 7 * v) * Bf, st,
          launch_grad<T>(M, U, 3, b->d_kind[0], (const T*)b->d_val[0], X.gU, st));
  S->n_launch++;
  if ((s2 = halo_exchange(S->m, X.gU, 9, st))) return s2;
  PLAUNCH(pr, "k_transport_assemble", -1, 23 * v * N + (16 + 10 * v) * F + (9 + 8 * v) * Bf, st,
          launch_transport_assemble<T, 3>(M.n_slices, st, M, U, phi, X.gU, X.gp, b->d_kind[0], (const T*)b->d_val[0],
                                          (T)S->o.nu, (T)(1.0 / S->o.dt), (T)theta_of(S->o), S->o.convection,
                                          S->kcorr, X.fdO, X.fdN, X.udiag, X.bU, X.rhsU, X.ucoef, X.ucoefT));
  S->n_launch++;
  if ((s2 = halo_exchange(S->m, X.udiag, 1, st))) return s2;   // ghost diag: rAU of the neighbours (k_HbyA ...)
  X.assembled = true;
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

// O-6: one PISO step
template <class T>
static dfvm_status piso(dfvm_solver* S, SolverT<T>& X, T* U, T* p, T* phi, dfvm_step_report* R, cudaStream_t st) {
  DevMesh<T>& M = *X.M;
  dfvm_bcs* b = S->b;
  const dfvm_piso_opts& o = S->o;
  dfvm_status s2;
  S->n_launch = 0;
  X.pending.clear();
  std::memset(R, 0, sizeof(*R));
  if ((s2 = bcs_device(b, 0, st)) || (s2 = bcs_device(b, 1, st))) return s2;
  // time-varying boundary values at the new time level t^{n+1} (A-41)
  if ((s2 = bcs_time(b, 0, S->t + o.dt, st)) || (s2 = bcs_time(b, 1, S->t + o.dt, st))) return s2;
  S->n_launch += (int)!b->wave_patches[0].empty() + (int)!b->wave_patches[1].empty();
  if ((s2 = sync_wk(S, X, st))) return s2;
  const int gs = grid_for_slices(M.n_slices), gf = grid_for((int64_t)M.F + M.B);
  const uint8_t* bkU = b->d_kind[0];
  const T* bvU = (const T*)b->d_val[0];
  const uint8_t* bkp = b->d_kind[1];
  T* bvp = (T*)b->d_val[1];
  Prof* pr = S->pr();
  const double v = sizeof(T), N = M.n_own, F = M.F, Bf = M.B, Z = (double)M.nnz;
  const double grad_s_bytes = 5 * v * N + (16 + 4 * v) * F + (9 + 5 * v) * Bf;
  // grad p^n (predictor source)
  if ((s2 = halo_exchange(S->m, p, 1, st))) return s2;
  PLAUNCH(pr, "k_grad (p)", -1, grad_s_bytes, st, launch_grad<T>(M, p, 1, bkp, bvp, X.gp, st));
  S->n_launch++;
  // 1. momentum assembly from (U^n, phi^n, grad U^n)
  if ((s2 = assemble(S, X, U, phi, st))) return s2;
  if (o.ddt_corr) {   // start-of-step U (with ghosts, exchanged by assemble) and phi for ddtCorr (A-42)
    if (!X.Uold && ((s2 = X.al(&X.Uold, 3 * (size_t)M.n_cells, st)) || (s2 = X.al(&X.phiold, (size_t)M.F + 1, st)))) return s2;
    DFVM_CUDA(cudaMemcpyAsync(X.Uold, U, 3 * (size_t)M.n_cells * sizeof(T), cudaMemcpyDeviceToDevice, st));
    DFVM_CUDA(cudaMemcpyAsync(X.phiold, phi, (size_t)M.F * sizeof(T), cudaMemcpyDeviceToDevice, st));
  }
  // 1b. DFVM_AMG_OVERLAP=1: the step's pressure matrix and AMG values on a
  // low-priority side stream, overlapping the predictor.  Default off:
  // measured on C5 round 2 at 315.5 / 317.1 ms/step against 314.0 / 315.2
  // in the first corrector (profiles/r02_sweep_r2s_overlap.jsonl) — the
  // predictor's one-wave kernels leave the side stream no room until they
  // drain, and the refresh's memory-bound kernels then compete with it
  X.side_pending = false;
  const bool overlap = X.amg && S->m->part.P == 1 && !pr && !S->timing && st != nullptr && [] {
    const char* e = getenv("DFVM_AMG_OVERLAP");
    return e && atoi(e) == 1;
  }();
  if (overlap) {
    if (!X.side) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);   // lo: the lowest priority (greatest value)
      DFVM_CUDA(cudaStreamCreateWithPriority(&X.side, cudaStreamNonBlocking, lo));
      DFVM_CUDA(cudaEventCreateWithFlags(&X.side_start, cudaEventDisableTiming));
      DFVM_CUDA(cudaEventCreateWithFlags(&X.side_done, cudaEventDisableTiming));
    }
    DFVM_CUDA(cudaEventRecord(X.side_start, st));
    DFVM_CUDA(cudaStreamWaitEvent(X.side, X.side_start, 0));
    k_rAU<T><<<grid_for(M.n_own), kThreads, 0, X.side>>>(M.n_own, M.vol, X.udiag, X.rAU);
    k_pcoef<T><<<grid_slices(k_pcoef<T>, M.n_slices), kThreads, 0, X.side>>>(M, X.rAU, X.phiHbyA, bkp, bvp, S->fixed_p ? -1 : S->ref_row,
                                            (T)o.p_ref_value, X.pcoef, X.pdiag, X.prhs0, 1);
    S->n_launch += 2;
    if ((s2 = amg_update<T>(X.amg, X.pcoef, X.pdiag, X.side, &S->n_launch, nullptr))) return s2;
    DFVM_CUDA(cudaEventRecord(X.side_done, X.side));
    X.amg_dirty = false;
    X.side_pending = true;
  }
  // 2. predictor
  dfvm_status res = run_bicgstab<T, 3>(S, X, X.rhsU, U, o.U_tol, o.U_rel_tol, o.U_maxit, R->U, st);
  if (res != DFVM_OK && res != DFVM_E_NOT_CONVERGED) return res;   // breakdown, CUDA / NCCL errors
  const int n_wk = (int)S->wk.size();
  int np = 0;
  for (int corr = 1; corr <= o.n_corr; ++corr) {
    if (X.side_pending) {   // rAU, the pressure matrix and the hierarchy from the side stream
      DFVM_CUDA(cudaStreamWaitEvent(st, X.side_done, 0));
      X.side_pending = false;
    }
    // 3.1 Windkessel
    if (n_wk) {
      PLAUNCH(pr, "k_windkessel", -1, 0, st,
              (k_windkessel<T><<<n_wk, kThreads, 0, st>>>(M, phi, X.d_wk, X.d_wk_ptr, X.d_wk_faces, o.dt, o.rho, bvp,
                                                          Red{S->m->part.P, X.red_local})));
      S->n_launch++;
      if (S->m->part.P > 1) {
        if ((s2 = allgather_f64(S->m, X.red_local, X.red_all, n_wk, st))) return s2;
        k_windkessel_fin<T><<<n_wk, kThreads, 0, st>>>(X.red_all, S->m->part.P, n_wk, X.d_wk, X.d_wk_ptr,
                                                       X.d_wk_faces, o.dt, o.rho, bvp);
        S->n_launch++;
      }
    }
    // 3.2 rAU, HbyA
    if ((s2 = halo_exchange(S->m, U, 3, st))) return s2;
    PLAUNCH(pr, "k_HbyA", -1, 4 * N + Z * (4 + v) + 12 * v * N, st,
            (k_HbyA<T><<<grid_slices(k_HbyA<T>, M.n_slices), kThreads, 0, st>>>(M, X.bU, X.udiag, X.ucoef, U, X.rAU, X.HbyA, overlap ? 0 : 1)));
    S->n_launch++;
    if ((s2 = halo_exchange(S->m, X.HbyA, 3, st)) || (s2 = halo_exchange(S->m, X.rAU, 1, st))) return s2;
    // 3.3 phiHbyA
    PLAUNCH(pr, "k_phiHbyA", -1,
            3 * v * N + (8 + 5 * v) * F + (5 + 8 * v) * Bf + (o.ddt_corr ? 4 * v * N + v * F : 0.0), st,
            (k_phiHbyA<T><<<grid_rows(k_phiHbyA<T>, (int64_t)M.F + M.B), kThreads, 0, st>>>(M, X.HbyA, bkU, bvU, X.phiHbyA, o.ddt_corr ? X.Uold : nullptr,
                                                   X.phiold, X.rAU, (T)(1.0 / o.dt))));
    // 3.4 pressure coefficients
    PLAUNCH(pr, "k_pcoef", -1, 3 * v * N + (16 + 5 * v) * F + (9 + 3 * v) * Bf, st,
            (k_pcoef<T><<<grid_slices(k_pcoef<T>, M.n_slices), kThreads, 0, st>>>(M, X.rAU, X.phiHbyA, bkp, bvp, S->fixed_p ? -1 : S->ref_row,
                                                 (T)o.p_ref_value, X.pcoef, X.pdiag, X.prhs0, overlap ? 2 : 3)));

    // The pressure matrix depends on rAU = V / a_P only (the momentum
    // diagonal of this step's assembly), so it is the same in every corrector
    // of the step: the AMG hierarchy values (Galerkin products, l1
    // diagonals, coarsest inverse) are refreshed once per step, not per
    // corrector (the right-hand side prhs0 changes with phiHbyA).
    if (corr == 1 && !overlap) X.amg_dirty = true;
    S->n_launch += 2;
    // 3.5 non-orthogonal loop
    for (int io = 0; io <= o.n_nonorth; ++io) {
      const T* rhs = X.prhs0;
      if (S->kcorr) {
        // grad p of the current p: the stored gradient is stale after the
        // previous solve (io > 0) or after a Windkessel update of p_b
        if (io > 0 || n_wk > 0) {
          if ((s2 = halo_exchange(S->m, p, 1, st))) return s2;
          PLAUNCH(pr, "k_grad (p)", -1, grad_s_bytes, st, launch_grad<T>(M, p, 1, bkp, bvp, X.gp, st));
          S->n_launch++;
        }
        if ((s2 = halo_exchange(S->m, X.gp, 3, st))) return s2;
        PLAUNCH(pr, "k_prhs", -1, 6 * v * N + (16 + 5 * v) * F, st,
                (k_prhs<T><<<grid_slices(k_prhs<T>, M.n_slices), kThreads, 0, st>>>(M, X.rAU, X.gp, X.prhs0, X.prhs)));
        S->n_launch++;
        rhs = X.prhs;
      }
      const bool final_corr = corr == o.n_corr && io == o.n_nonorth;
      s2 = run_cg(S, X, rhs, p, o.p_tol, final_corr ? o.p_rel_tol_final : o.p_rel_tol, o.p_maxit,
                  np < 16 ? &R->p[np] : nullptr, st);
      np++;
      if (s2 != DFVM_OK && s2 != DFVM_E_NOT_CONVERGED) return s2;   // breakdown, CUDA / NCCL errors
      if (s2 == DFVM_E_NOT_CONVERGED) res = s2;
      if (io == o.n_nonorth) {
        if ((s2 = halo_exchange(S->m, p, 1, st))) return s2;
        PLAUNCH(pr, "k_fluxcorr", -1, 5 * v * N + (8 + 7 * v) * F + (5 + 4 * v) * Bf, st,
                (k_fluxcorr<T><<<grid_rows(k_fluxcorr<T>, (int64_t)M.F + M.B), kThreads, 0, st>>>(M, X.phiHbyA, p, X.rAU, X.gp, bkp, bvp, S->kcorr, phi)));
        S->n_launch++;
      }
    }
    // 3.6 velocity correction (also refreshes grad p)
    PLAUNCH(pr, "k_Ucorr", -1, 12 * v * N + (16 + 4 * v) * F + (9 + 4 * v) * Bf, st,
            (k_Ucorr<T><<<grid_slices(k_Ucorr<T>, M.n_slices), kThreads, 0, st>>>(M, p, bkp, bvp, X.HbyA, X.rAU, U, X.gp)));
    S->n_launch++;
  }
  R->n_p = np;
  // 4. continuity + non-finite + Windkessel commit
  PLAUNCH(pr, "k_continuity", -1, 4 * v * N + (16 + v) * F + (8 + v) * Bf, st,
          (k_continuity<T><<<grid_slices(k_continuity<T>, M.n_slices), kThreads, 0, st>>>(M, phi, U, p, X.partials, X.ticket, X.d_cont, X.d_wk, n_wk,
                                                    Red{S->m->part.P, X.red_local})));
  S->n_launch++;
  if (S->m->part.P > 1) {
    if ((s2 = allgather_f64(S->m, X.red_local, X.red_all, 3, st))) return s2;
    k_continuity_fin<<<1, 1, 0, st>>>(X.red_all, S->m->part.P, X.d_cont, X.d_wk, n_wk);
    S->n_launch++;
  }
  DFVM_CUDA(cudaMemcpyAsync(X.h_cont, X.d_cont, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (n_wk) DFVM_CUDA(cudaMemcpyAsync(X.h_wk, X.d_wk, n_wk * sizeof(WKDev), cudaMemcpyDeviceToHost, st));
  DFVM_CUDA(cudaStreamSynchronize(st));
  DFVM_CUDA(cudaGetLastError());
  if (pr) pr->harvest();
  {   // device-resident solves of this step: reports and status
    const dfvm_status ps = resolve_pending(S, X);
    if (ps == DFVM_E_BREAKDOWN) {
      R->gpu_launches = S->n_launch;
      count_launch(S->n_launch);
      set_error(DFVM_E_BREAKDOWN, "Krylov breakdown in the PISO step");
      return DFVM_E_BREAKDOWN;
    }
    if (ps == DFVM_E_NOT_CONVERGED) res = ps;
  }
  R->cont_err_max = X.h_cont[0];
  R->cont_err_sum = X.h_cont[1];
  R->nonfinite = X.h_cont[2] > 0;
  R->n_outlets = n_wk;
  for (int i = 0; i < n_wk && i < 64; ++i) {
    R->Q[i] = X.h_wk[i].Q; R->p_o[i] = X.h_wk[i].p_o;
    S->wk[i].pc = X.h_wk[i].pc_n;
  }
  R->gpu_launches = S->n_launch;
  count_launch(S->n_launch);
  S->t += o.dt;
  if (R->nonfinite) { set_error(DFVM_E_NONFINITE, "non-finite U or p after the PISO step"); return DFVM_E_NONFINITE; }
  if (o.cont_tol > 0 && !(R->cont_err_max <= o.cont_tol)) {
    set_error(DFVM_E_CONTINUITY, "continuity violated after the PISO step: max_c |sum_f s phi_f| = " +
              std::to_string(R->cont_err_max) + " > cont_tol " + std::to_string(o.cont_tol));
    return DFVM_E_CONTINUITY;
  }
  return res;
}

}  // namespace dfvm

namespace dfvm {

// One implicit-Euler step of passive-scalar transport (NEXT-1 workload,
// PAPER.md §3.1.2): d x/dt + div(phi x) - div(Gamma grad x) = 0
// with the face flux phi fixed, field 's' boundary conditions and the
// solver's convection scheme (upwind / central / SOU / QUICK deferred
// correction); BiCGStab from x^n.
template <class T>
static dfvm_status transport_step_t(dfvm_solver* S, SolverT<T>& X, T* x, const T* phi, double gamma,
                                    dfvm_solve_report* rep, cudaStream_t st) {
  DevMesh<T>& M = *X.M;
  dfvm_bcs* b = S->b;
  dfvm_status e;
  if ((e = bcs_device(b, 2, st))) return e;
  S->n_launch = 0;
  X.pending.clear();
  if ((e = halo_exchange(S->m, x, 1, st))) return e;
  launch_grad<T>(M, x, 1, b->d_kind[2], (const T*)b->d_val[2], X.gp, st);
  if ((e = halo_exchange(S->m, X.gp, 3, st))) return e;
  const int gs = grid_for_slices(M.n_slices), ge = grid_for(M.n_own);
  launch_transport_assemble<T, 1>(M.n_slices, st, M, x, phi, X.gp, nullptr, b->d_kind[2], (const T*)b->d_val[2], (T)gamma,
                                  (T)(1.0 / S->o.dt), (T)theta_of(S->o), S->o.convection, S->kcorr, X.fdO, X.fdN,
                                  X.udiag, X.prhs0, X.prhs, X.ucoef, X.ucoefT);
  if ((e = halo_exchange(S->m, X.udiag, 1, st))) return e;
  S->n_launch += 2;
  X.assembled = true;
  // one-component BiCGStab directly on x (halo-exchanged above) and b = prhs
  dfvm_solve_report r1[1];
  dfvm_status res = run_bicgstab<T, 1>(S, X, X.prhs, x, S->o.U_tol, S->o.U_rel_tol, S->o.U_maxit, r1, st);
  DFVM_CUDA(cudaStreamSynchronize(st));
  DFVM_CUDA(cudaGetLastError());
  if (!X.pending.empty()) res = resolve_pending(S, X);
  count_launch(S->n_launch);
  if (rep) *rep = r1[0];
  return res;
}

}  // namespace dfvm

extern "C" {

dfvm_status dfvm_solver_create(dfvm_mesh* m, dfvm_bcs* b, const dfvm_piso_opts* opts, dfvm_solver** out) {
  if (!m || !b || !opts || !out || b->m != m) { set_error(DFVM_E_INVALID_ARG, "NULL or mismatched argument"); return DFVM_E_INVALID_ARG; }
  if (!(opts->dt > 0) || !(opts->nu >= 0) || opts->n_corr < 1 || opts->n_corr > 8 || opts->n_nonorth < 0 ||
      (opts->n_corr * (opts->n_nonorth + 1)) > 16 || opts->p_maxit < 1 || opts->U_maxit < 1 || !(opts->rho > 0) ||
      opts->p_precond < 0 || opts->p_precond > 2 || opts->convection < 0 || opts->convection > 3 ||
      opts->time_scheme < DFVM_TIME_BACKWARD_EULER || opts->time_scheme > DFVM_TIME_FORWARD_EULER || opts->ddt_corr < 0 || opts->ddt_corr > 1 ||
      !(opts->cont_tol >= 0)) {
    set_error(DFVM_E_INVALID_ARG, "invalid PISO options");
    return DFVM_E_INVALID_ARG;
  }
  if (opts->p_ref_cell < 0 || opts->p_ref_cell >= m->H.N) { set_error(DFVM_E_INVALID_ARG, "p_ref_cell out of range", opts->p_ref_cell); return DFVM_E_INVALID_ARG; }
  cudaSetDevice(m->device);
  std::unique_ptr<dfvm_solver> S(new dfvm_solver());
  S->m = m; S->b = b; S->o = *opts;
  const int32_t gid = m->H.new_of_old[opts->p_ref_cell];
  S->ref_row = (gid >= m->part.lo && gid < m->part.hi) ? (int)(gid - m->part.lo) : -1;
  S->kcorr = m->H.nonorth != DFVM_NONORTH_NONE;
  dfvm_status st;
  if (m->precision == DFVM_F64) {
    auto* X = new SolverT<double>();
    S->impl.reset(X);
    st = X->init(m, &m->d64);
    if (!st && opts->convection >= 2) st = X->build_face_offsets();
  } else {
    auto* X = new SolverT<float>();
    S->impl.reset(X);
    st = X->init(m, &m->d32);
    if (!st && opts->convection >= 2) st = X->build_face_offsets();
  }
  if (st) return st;
  *out = S.release();
  return DFVM_OK;
}

dfvm_status dfvm_solver_set_timing(dfvm_solver* s, int32_t on) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  s->timing = on != 0;
  for (int i = 0; i < 4; ++i) { s->t_ms[i] = 0; s->t_n[i] = 0; }
  return DFVM_OK;
}

dfvm_status dfvm_solver_amg_levels(const dfvm_solver* s, int32_t* n_levels, int64_t* sizes, int64_t* nnz) {
  if (!s || !n_levels) { set_error(DFVM_E_INVALID_ARG, "NULL argument"); return DFVM_E_INVALID_ARG; }
  int lv[32] = {0};
  int64_t nz[32] = {0};
  int n = 0;
  if (s->m->precision == DFVM_F64) {
    auto* X = static_cast<SolverT<double>*>(s->impl.get());
    if (X->amg) { n = amg_levels<double>(X->amg, lv); amg_level_nnz<double>(X->amg, nz); }
  } else {
    auto* X = static_cast<SolverT<float>*>(s->impl.get());
    if (X->amg) { n = amg_levels<float>(X->amg, lv); amg_level_nnz<float>(X->amg, nz); }
  }
  *n_levels = n;
  if (sizes) for (int i = 0; i < n; ++i) sizes[i] = lv[i];
  if (nnz) for (int i = 0; i < n; ++i) nnz[i] = nz[i];
  return DFVM_OK;
}

dfvm_status dfvm_solver_profile(dfvm_solver* s, int32_t on) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  s->prof.clear();
  s->prof.on = on != 0;
  return DFVM_OK;
}

dfvm_status dfvm_solver_profile_get(const dfvm_solver* s, dfvm_kernel_stat* out, int32_t cap, int32_t* n) {
  if (!s || !n || (cap > 0 && !out)) { set_error(DFVM_E_INVALID_ARG, "NULL argument"); return DFVM_E_INVALID_ARG; }
  const auto& st = s->prof.stats;
  *n = (int32_t)st.size();
  for (int32_t i = 0; i < cap && i < (int32_t)st.size(); ++i) {
    std::memset(&out[i], 0, sizeof(out[i]));
    std::strncpy(out[i].name, st[i].name, sizeof(out[i].name) - 1);
    out[i].level = st[i].lvl;
    out[i].launches = st[i].n;
    out[i].ms = st[i].ms;
    out[i].alg_bytes = st[i].bytes;
  }
  return DFVM_OK;
}

dfvm_status dfvm_solver_get_timing(const dfvm_solver* s, double* ms, int64_t* count) {
  if (!s || !ms || !count) { set_error(DFVM_E_INVALID_ARG, "NULL argument"); return DFVM_E_INVALID_ARG; }
  for (int i = 0; i < 4; ++i) { ms[i] = s->t_ms[i]; count[i] = s->t_n[i]; }
  return DFVM_OK;
}

dfvm_status dfvm_solver_destroy(dfvm_solver* s) {
  delete s;
  return DFVM_OK;
}

dfvm_status dfvm_windkessel_update(double pc, double Q, double dt, double Rp, double C, double Rd, int32_t scheme,
                                   double* pc_new, double* p_o) {
  if (!(Rp >= 0) || !(C > 0) || !(Rd > 0) || !(dt > 0) || scheme < 0 || scheme > 2 || !pc_new || !p_o) {
    set_error(DFVM_E_INVALID_WK_PARAMS, "Windkessel needs Rp >= 0, C > 0, Rd > 0, dt > 0, scheme 0..2", scheme);
    return DFVM_E_INVALID_WK_PARAMS;
  }
  double p;
  if (scheme == 0) { const double e = std::exp(-dt / (Rd * C)); p = pc * e + Rd * Q * (1.0 - e); }
  else if (scheme == 1) p = pc + dt * (Q - pc / Rd) / C;
  else p = (pc + dt * Q / C) / (1.0 + dt / (Rd * C));
  *pc_new = p;
  *p_o = p + Rp * Q;
  return DFVM_OK;
}

dfvm_status dfvm_windkessel_set(dfvm_solver* s, int32_t patch, double Rp, double C, double Rd, double pc0,
                                int32_t scheme) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  if (!(Rp >= 0) || !(C > 0) || !(Rd > 0) || scheme < 0 || scheme > 2) {
    set_error(DFVM_E_INVALID_WK_PARAMS, "Windkessel needs Rp >= 0, C > 0, Rd > 0, scheme 0..2", patch);
    return DFVM_E_INVALID_WK_PARAMS;
  }
  if (patch < 0 || patch >= (int32_t)s->m->H.pkind.size() || s->m->H.pkind[patch] == DFVM_PATCH_EMPTY) {
    set_error(DFVM_E_INVALID_ARG, "bad Windkessel patch", patch);
    return DFVM_E_INVALID_ARG;
  }
  if (s->wk.size() >= 64) { set_error(DFVM_E_INVALID_ARG, "at most 64 Windkessel outlets"); return DFVM_E_INVALID_ARG; }
  bool found = false;
  for (auto& w : s->wk)
    if (w.patch == patch) { w = {patch, Rp, C, Rd, pc0, scheme}; found = true; }
  if (!found) s->wk.push_back({patch, Rp, C, Rd, pc0, scheme});
  dfvm_bc_desc d{};
  d.kind = DFVM_BC_WINDKESSEL;
  dfvm_bcs_set(s->b, patch, 'p', &d);
  s->wk_dirty = true;
  return DFVM_OK;
}

dfvm_status dfvm_windkessel_state(const dfvm_solver* s, int32_t patch, double* pc) {
  if (!s || !pc) { set_error(DFVM_E_INVALID_ARG, "NULL argument"); return DFVM_E_INVALID_ARG; }
  for (auto& w : s->wk)
    if (w.patch == patch) { *pc = w.pc; return DFVM_OK; }
  set_error(DFVM_E_INVALID_ARG, "patch has no Windkessel model", patch);
  return DFVM_E_INVALID_ARG;
}

static dfvm_status check_f(const dfvm_field* f, const dfvm_mesh* m, bool cells, int nc, const char* what) {
  if (!f || f->m != m || (cells ? f->loc != DFVM_CELLS : f->loc == DFVM_CELLS) || f->n_comp != nc) {
    set_error(DFVM_E_INVALID_ARG, std::string("field '") + what + "' has the wrong mesh, location or components");
    return DFVM_E_INVALID_ARG;
  }
  return DFVM_OK;
}

dfvm_status dfvm_transport_step(dfvm_solver* s, dfvm_field* x, const dfvm_field* phi, double gamma,
                                dfvm_solve_report* rep, dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(x, s->m, true, 1, "x")) || (st = check_f(phi, s->m, false, 1, "phi"))) return st;
  if (!(gamma >= 0)) { set_error(DFVM_E_INVALID_ARG, "diffusivity must be >= 0"); return DFVM_E_INVALID_ARG; }
  cudaSetDevice(s->m->device);
  cudaStream_t cs = (cudaStream_t)stream;
  if (s->m->precision == DFVM_F64)
    return transport_step_t<double>(s, *static_cast<SolverT<double>*>(s->impl.get()), (double*)x->ptr,
                                    (const double*)phi->ptr, gamma, rep, cs);
  return transport_step_t<float>(s, *static_cast<SolverT<float>*>(s->impl.get()), (float*)x->ptr,
                                 (const float*)phi->ptr, gamma, rep, cs);
}

dfvm_status dfvm_piso_step(dfvm_solver* s, dfvm_field* U, dfvm_field* p, dfvm_field* phi, dfvm_step_report* rep,
                           dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(U, s->m, true, 3, "U")) || (st = check_f(p, s->m, true, 1, "p")) ||
      (st = check_f(phi, s->m, false, 1, "phi")))
    return st;
  cudaSetDevice(s->m->device);
  s->fixed_p = solver_has_fixed_p(s);
  dfvm_step_report local;
  dfvm_step_report* R = rep ? rep : &local;
  cudaStream_t cs = (cudaStream_t)stream;
  if (s->m->precision == DFVM_F64)
    return piso<double>(s, *static_cast<SolverT<double>*>(s->impl.get()), (double*)U->ptr, (double*)p->ptr,
                        (double*)phi->ptr, R, cs);
  return piso<float>(s, *static_cast<SolverT<float>*>(s->impl.get()), (float*)U->ptr, (float*)p->ptr,
                     (float*)phi->ptr, R, cs);
}

}  // extern "C"

template <class T>
static dfvm_status pressure_solve_t(dfvm_solver* s, SolverT<T>& X, const T* rAU, const T* rhs, T* p, double tol,
                                    double rel_tol, int maxit, dfvm_solve_report* rep, cudaStream_t st,
                                    bool adjoint = false) {
  DevMesh<T>& M = *X.M;
  dfvm_status s2;
  if ((s2 = bcs_device(s->b, 1, st))) return s2;
  if ((s2 = halo_exchange(s->m, (void*)rAU, 1, st))) return s2;
  // pressure coefficients from rAU: with phiHbyA = 0, prhs0 = sum_b c_b p_b + the
  // gauge term (A-12) at the reference row; the caller's rhs already holds every
  // other term, so only the gauge term is added to it (k_add_at).
  DFVM_CUDA(cudaMemsetAsync(X.phiHbyA, 0, ((size_t)M.F + M.B + M.E) * sizeof(T), st));
  const int ref = s->fixed_p ? -1 : s->ref_row;
  k_pcoef<T><<<grid_for_slices(M.n_slices), kThreads, 0, st>>>(M, rAU, X.phiHbyA, s->b->d_kind[1],
      (const T*)s->b->d_val[1], ref, (T)s->o.p_ref_value, X.pcoef, X.pdiag, X.prhs0);
  X.amg_dirty = true;
  DFVM_CUDA(cudaMemcpyAsync(X.prhs, rhs, (size_t)M.n_own * sizeof(T), cudaMemcpyDeviceToDevice, st));
  // adjoint system A^T lambda = g: the gauge changes the matrix only (its
  // right-hand-side term belongs to the forward system)
  const bool add_ref = ref >= 0 && !adjoint;
  if (add_ref) k_add_at<T><<<1, 1, 0, st>>>(X.prhs, X.prhs0, ref);
  count_launch(1 + add_ref);
  s->n_launch = 0;
  X.pending.clear();
  dfvm_status r = run_cg(s, X, X.prhs, p, tol, rel_tol, maxit, rep, st);
  DFVM_CUDA(cudaStreamSynchronize(st));
  if (!X.pending.empty() && r == DFVM_OK) r = resolve_pending(s, X);
  count_launch(s->n_launch);
  return r;
}

extern "C" {

dfvm_status dfvm_pressure_solve(dfvm_solver* s, const dfvm_field* rAU, const dfvm_field* rhs, dfvm_field* p,
                                double tol, double rel_tol, int32_t maxit, dfvm_solve_report* rep,
                                dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(rAU, s->m, true, 1, "rAU")) || (st = check_f(rhs, s->m, true, 1, "rhs")) ||
      (st = check_f(p, s->m, true, 1, "p")))
    return st;
  cudaSetDevice(s->m->device);
  s->fixed_p = solver_has_fixed_p(s);
  cudaStream_t cs = (cudaStream_t)stream;
  if (s->m->precision == DFVM_F64)
    return pressure_solve_t<double>(s, *static_cast<SolverT<double>*>(s->impl.get()), (const double*)rAU->ptr,
                                    (const double*)rhs->ptr, (double*)p->ptr, tol, rel_tol, maxit, rep, cs);
  return pressure_solve_t<float>(s, *static_cast<SolverT<float>*>(s->impl.get()), (const float*)rAU->ptr,
                                 (const float*)rhs->ptr, (float*)p->ptr, tol, rel_tol, maxit, rep, cs);
}

dfvm_status dfvm_momentum_assemble(dfvm_solver* s, const dfvm_field* U, const dfvm_field* phi, dfvm_field* diag,
                                   dfvm_field* b, dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(U, s->m, true, 3, "U")) || (st = check_f(phi, s->m, false, 1, "phi")) ||
      (st = check_f(diag, s->m, true, 1, "diag")) || (st = check_f(b, s->m, true, 3, "b")))
    return st;
  cudaSetDevice(s->m->device);
  cudaStream_t cs = (cudaStream_t)stream;
  s->n_launch = 0;
  if (s->m->precision == DFVM_F64) {
    auto& X = *static_cast<SolverT<double>*>(s->impl.get());
    DFVM_CUDA(cudaMemsetAsync(X.gp, 0, (size_t)X.M->n_cells * 3 * sizeof(double), cs));
    if ((st = assemble<double>(s, X, (const double*)U->ptr, (const double*)phi->ptr, cs))) return st;
    DFVM_CUDA(cudaMemcpyAsync(diag->ptr, X.udiag, (size_t)X.M->n_own * sizeof(double), cudaMemcpyDeviceToDevice, cs));
    DFVM_CUDA(cudaMemcpyAsync(b->ptr, X.bU, (size_t)X.M->n_own * 3 * sizeof(double), cudaMemcpyDeviceToDevice, cs));
  } else {
    auto& X = *static_cast<SolverT<float>*>(s->impl.get());
    DFVM_CUDA(cudaMemsetAsync(X.gp, 0, (size_t)X.M->n_cells * 3 * sizeof(float), cs));
    if ((st = assemble<float>(s, X, (const float*)U->ptr, (const float*)phi->ptr, cs))) return st;
    DFVM_CUDA(cudaMemcpyAsync(diag->ptr, X.udiag, (size_t)X.M->n_own * sizeof(float), cudaMemcpyDeviceToDevice, cs));
    DFVM_CUDA(cudaMemcpyAsync(b->ptr, X.bU, (size_t)X.M->n_own * 3 * sizeof(float), cudaMemcpyDeviceToDevice, cs));
  }
  count_launch(s->n_launch);
  return DFVM_OK;
}

// ---- NEXT-3: adjoint apply / adjoint pressure solve / pressure VJP
dfvm_status dfvm_momentum_apply_transpose(dfvm_solver* s, const dfvm_field* x, dfvm_field* y, dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(x, s->m, true, 3, "x")) || (st = check_f(y, s->m, true, 3, "y"))) return st;
  cudaSetDevice(s->m->device);
  cudaStream_t cs = (cudaStream_t)stream;
  if ((st = halo_exchange(s->m, x->ptr, 3, cs))) return st;
  if (s->m->precision == DFVM_F64) {
    auto& X = *static_cast<SolverT<double>*>(s->impl.get());
    if (!X.assembled) { set_error(DFVM_E_INVALID_ARG, "momentum matrix not assembled"); return DFVM_E_INVALID_ARG; }
    k_apply<double, 3><<<grid_for_slices(X.M->n_slices), kThreads, 0, cs>>>(*X.M, X.udiag, X.ucoefT, (const double*)x->ptr, (double*)y->ptr);
  } else {
    auto& X = *static_cast<SolverT<float>*>(s->impl.get());
    if (!X.assembled) { set_error(DFVM_E_INVALID_ARG, "momentum matrix not assembled"); return DFVM_E_INVALID_ARG; }
    k_apply<float, 3><<<grid_for_slices(X.M->n_slices), kThreads, 0, cs>>>(*X.M, X.udiag, X.ucoefT, (const float*)x->ptr, (float*)y->ptr);
  }
  count_launch();
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

dfvm_status dfvm_pressure_solve_adjoint(dfvm_solver* s, const dfvm_field* rAU, const dfvm_field* g, dfvm_field* lambda,
                                        double tol, double rel_tol, int32_t maxit, dfvm_solve_report* rep,
                                        dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(rAU, s->m, true, 1, "rAU")) || (st = check_f(g, s->m, true, 1, "g")) ||
      (st = check_f(lambda, s->m, true, 1, "lambda")))
    return st;
  cudaSetDevice(s->m->device);
  s->fixed_p = solver_has_fixed_p(s);
  cudaStream_t cs = (cudaStream_t)stream;
  if (s->m->precision == DFVM_F64)
    return pressure_solve_t<double>(s, *static_cast<SolverT<double>*>(s->impl.get()), (const double*)rAU->ptr,
                                    (const double*)g->ptr, (double*)lambda->ptr, tol, rel_tol, maxit, rep, cs, true);
  return pressure_solve_t<float>(s, *static_cast<SolverT<float>*>(s->impl.get()), (const float*)rAU->ptr,
                                 (const float*)g->ptr, (float*)lambda->ptr, tol, rel_tol, maxit, rep, cs, true);
}

dfvm_status dfvm_pressure_vjp(dfvm_solver* s, const dfvm_field* p, const dfvm_field* lambda, dfvm_field* grad,
                              dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(p, s->m, true, 1, "p")) || (st = check_f(lambda, s->m, true, 1, "lambda")) ||
      (st = check_f(grad, s->m, true, 1, "grad")))
    return st;
  cudaSetDevice(s->m->device);
  s->fixed_p = solver_has_fixed_p(s);
  cudaStream_t cs = (cudaStream_t)stream;
  if ((st = bcs_device(s->b, 1, cs))) return st;
  if ((st = halo_exchange(s->m, p->ptr, 1, cs)) || (st = halo_exchange(s->m, lambda->ptr, 1, cs))) return st;
  const int ref_orig = s->fixed_p ? -1 : (int)s->o.p_ref_cell;
  if (s->m->precision == DFVM_F64) {
    auto& X = *static_cast<SolverT<double>*>(s->impl.get());
    k_pvjp<double><<<grid_for_slices(X.M->n_slices), kThreads, 0, cs>>>(*X.M, (const double*)p->ptr,
        (const double*)lambda->ptr, s->b->d_kind[1], s->m->d_cell_orig, ref_orig, s->o.p_ref_value, (double*)grad->ptr);
  } else {
    auto& X = *static_cast<SolverT<float>*>(s->impl.get());
    k_pvjp<float><<<grid_for_slices(X.M->n_slices), kThreads, 0, cs>>>(*X.M, (const float*)p->ptr,
        (const float*)lambda->ptr, s->b->d_kind[1], s->m->d_cell_orig, ref_orig, (float)s->o.p_ref_value, (float*)grad->ptr);
  }
  count_launch();
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

dfvm_status dfvm_momentum_apply(dfvm_solver* s, const dfvm_field* x, dfvm_field* y, dfvm_stream stream) {
  if (!s) { set_error(DFVM_E_INVALID_ARG, "NULL solver"); return DFVM_E_INVALID_ARG; }
  dfvm_status st;
  if ((st = check_f(x, s->m, true, 3, "x")) || (st = check_f(y, s->m, true, 3, "y"))) return st;
  cudaSetDevice(s->m->device);
  cudaStream_t cs = (cudaStream_t)stream;
  if ((st = halo_exchange(s->m, x->ptr, 3, cs))) return st;
  if (s->m->precision == DFVM_F64) {
    auto& X = *static_cast<SolverT<double>*>(s->impl.get());
    if (!X.assembled) { set_error(DFVM_E_INVALID_ARG, "momentum matrix not assembled"); return DFVM_E_INVALID_ARG; }
    k_apply<double, 3><<<grid_for_slices(X.M->n_slices), kThreads, 0, cs>>>(*X.M, X.udiag, X.ucoef, (const double*)x->ptr, (double*)y->ptr);
  } else {
    auto& X = *static_cast<SolverT<float>*>(s->impl.get());
    if (!X.assembled) { set_error(DFVM_E_INVALID_ARG, "momentum matrix not assembled"); return DFVM_E_INVALID_ARG; }
    k_apply<float, 3><<<grid_for_slices(X.M->n_slices), kThreads, 0, cs>>>(*X.M, X.udiag, X.ucoef, (const float*)x->ptr, (float*)y->ptr);
  }
  count_launch();
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

}  // extern "C"
