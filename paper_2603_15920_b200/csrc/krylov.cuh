// krylov.cuh — device control block of the Krylov solvers (PCG / BiCGStab)
// shared by solver.cu and amg.cu (the AMG level-0 post-smoother can fold the
// PCG's r.z reduction into its own pass).
//
// Krylov control runs on the device: every reduction is a deterministic
// two-level sum (block partials in block order, then the last block to
// arrive sums them in a fixed order) and that last block updates the solver
// scalars (alpha, beta, residual, convergence, stagnation) in a device
// control block; every Krylov kernel first checks the control block and
// exits when the solve is done.
#pragma once
#include "dev.cuh"

namespace dfvm {

// -------------------------------------------------------------- control
struct KCtl {
  double bnorm, res0, res, thr, best;
  double rz, alpha, beta;                 // CG
  double rho, rho_old, omega, snorm;       // BiCGStab (alpha shared)
  double tol, rel_tol;
  int it, best_it, maxit, done, converged, status, zero_x, half;
};

struct WKDev {
  double Rp, C, Rd, pc_n, pc_new, Q, p_o;
  int scheme, pad;
};

// stopping rule (A-13, stagnation per A-13''): called by the last block after each residual update
__device__ __forceinline__ void krylov_check(KCtl& c, double res) {
  c.res = res;
  if (res <= c.thr) { c.converged = 1; c.done = 1; return; }
  if (res < c.best) { c.best = res; c.best_it = c.it; }
  else if (c.tol < 1e-12 && c.best <= 1e-8 * c.res0 && c.it - c.best_it >= max(50, c.best_it)) { c.done = 1; c.status = DFVM_E_NOT_CONVERGED; return; }
  if (c.it >= c.maxit) { c.done = 1; c.status = DFVM_E_NOT_CONVERGED; }
}
__device__ __forceinline__ void krylov_start(KCtl& c, double bb, double rr) {
  c.bnorm = sqrt(bb);
  c.res0 = c.res = c.best = sqrt(rr);
  c.thr = fmax(c.tol * c.bnorm, c.rel_tol * c.res0);
  c.it = 0; c.best_it = 0; c.converged = 0; c.status = 0; c.zero_x = 0; c.half = 0; c.done = 0;
  if (c.bnorm == 0.0) { c.zero_x = 1; c.done = 1; c.converged = 1; c.res0 = c.res = 0; return; }
  if (c.res0 <= c.thr) { c.done = 1; c.converged = 1; }
}

// ---- control steps: applied to the global totals t[] of a reduction,
// either by the last block of the reducing kernel (one rank) or by the
// finalize kernel after the cross-rank all-gather (rank-order sum), so every
// rank applies bitwise-identical updates.
enum CtlKind { CTL_CG_INIT = 0, CTL_CG_SPMV, CTL_CG_R, CTL_BI_INIT, CTL_BI_V, CTL_BI_S, CTL_BI_T, CTL_BI_X,
               CTL_CG_R2, CTL_CG_RZ0, CTL_CG_RZ };

static __device__ void ctl_apply(int kind, KCtl* ctl, const double* t) {
  switch (kind) {
    // AMG-preconditioned CG: the residual check uses r.r; r.z comes from a
    // separate reduction after the V-cycle
    case CTL_CG_R2: {
      KCtl& c = *ctl;
      c.it++;
      krylov_check(c, sqrt(t[0]));
      if (c.done) c.half = 1;
      break;
    }
    case CTL_CG_RZ0: ctl->rz = t[0]; ctl->beta = 0.0; break;
    case CTL_CG_RZ: ctl->beta = t[0] / ctl->rz; ctl->rz = t[0]; break;
    case CTL_CG_INIT: {
      KCtl& c = *ctl;
      krylov_start(c, t[0], t[1]);
      c.rz = t[2]; c.beta = 0.0;
      break;
    }
    case CTL_CG_SPMV: {
      KCtl& c = *ctl;
      // breakdown: x already holds x_k (its update was applied by k_cg_p)
      if (!(t[0] > 0)) { c.done = 1; c.status = DFVM_E_BREAKDOWN; c.half = 0; c.it++; break; }
      c.alpha = c.rz / t[0];
      break;
    }
    case CTL_CG_R: {
      KCtl& c = *ctl;
      c.it++;
      krylov_check(c, sqrt(t[0]));
      if (c.done) c.half = 1;          // x += alpha pd still pending
      else { c.beta = t[1] / c.rz; c.rz = t[1]; }
      break;
    }
    case CTL_BI_INIT:
      for (int k = 0; k < 3; ++k) {
        KCtl& c = ctl[k];
        krylov_start(c, t[k], t[3 + k]);
        c.rho_old = 1; c.alpha = 1; c.omega = 1; c.rho = t[3 + k];
        if (!c.done && c.rho == 0.0) { c.done = 1; c.status = DFVM_E_BREAKDOWN; }
      }
      break;
    case CTL_BI_V:
      for (int k = 0; k < 3; ++k) {
        KCtl& c = ctl[k];
        if (c.done) continue;
        c.it++;
        if (t[k] == 0.0) { c.done = 1; c.status = DFVM_E_BREAKDOWN; continue; }
        c.alpha = c.rho / t[k];
      }
      break;
    case CTL_BI_S:
      for (int k = 0; k < 3; ++k) {
        KCtl& c = ctl[k];
        if (c.done) continue;
        c.snorm = sqrt(t[k]);
        if (c.snorm <= c.thr) c.half = 1;
      }
      break;
    case CTL_BI_T:   // t[0..2] = t.s, t[3..5] = t.t, t[6..8] = s.s (s formed inside k_bi_t)
      for (int k = 0; k < 3; ++k) {
        KCtl& c = ctl[k];
        if (c.done) continue;
        c.snorm = sqrt(t[6 + k]);
        if (c.snorm <= c.thr) { c.half = 1; continue; }
        if (t[3 + k] == 0.0) { c.done = 1; c.status = DFVM_E_BREAKDOWN; continue; }
        c.omega = t[k] / t[3 + k];
      }
      break;
    case CTL_BI_X:
      for (int k = 0; k < 3; ++k) {
        KCtl& c = ctl[k];
        if (c.done) continue;
        if (c.half) { c.res = c.snorm; c.converged = 1; c.done = 1; continue; }
        krylov_check(c, sqrt(t[3 + k]));
        if (c.done) continue;
        if (c.omega == 0.0) { c.done = 1; c.status = DFVM_E_BREAKDOWN; continue; }
        c.rho_old = c.rho;
        c.rho = t[k];
        if (c.rho == 0.0) { c.done = 1; c.status = DFVM_E_BREAKDOWN; }
      }
      break;
  }
}

// cross-rank reduction target: with one rank the last block applies the
// control step itself; with several it stores the rank's totals in `local`
// and the host enqueues all-gather + k_finalize.
struct Red {
  int nranks;
  double* local;
};
template <int NV>
__device__ __forceinline__ void red_finish(const Red& red, int kind, KCtl* ctl, const double (&t)[NV]) {
  if (red.nranks == 1) { ctl_apply(kind, ctl, t); return; }
#pragma unroll
  for (int i = 0; i < NV; ++i) red.local[i] = t[i];
}
static __global__ void k_finalize(int kind, int nv, const double* __restrict__ all, int P, KCtl* ctl) {
  PDL_ENTRY();
  // the reducing kernel exited early (and produced no totals) when the solve
  // was already done; init kernels always run
  if (kind == CTL_CG_SPMV || kind == CTL_CG_R || kind == CTL_CG_R2 || kind == CTL_CG_RZ0 || kind == CTL_CG_RZ) {
    if (ctl->done) return;
  }
  else if (kind != CTL_CG_INIT && kind != CTL_BI_INIT) { if (ctl[0].done && ctl[1].done && ctl[2].done) return; }
  double t[16];
  for (int i = 0; i < nv; ++i) {
    double s = 0;
    for (int r = 0; r < P; ++r) s += all[r * nv + i];   // fixed rank order
    t[i] = s;
  }
  ctl_apply(kind, ctl, t);
}


// A reduction folded into another kernel's pass (e.g. r.z in the AMG level-0
// post-smoother): where its partials go and which control step it drives.
struct KDot {
  double* partials;
  unsigned* ticket;
  KCtl* ctl;
  Red red;
  int kind;
};

}  // namespace dfvm
