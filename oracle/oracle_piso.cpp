// oracle/oracle_piso.cpp — O-5 momentum LDU, O-6 PISO step, O-7 linear
// solvers, O-8 Windkessel, and the steady Poisson pin (E1).
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain loops in the paper's order;
// readings of SURVEY.md §8(c) are named where the paper is silent.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

namespace orc {

static double dotv(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// --------------------------------------------------------------- O-7
// Stopping rule shared by CG and BiCGStab (A-13): b = 0 -> x = 0 with 0
// iterations; otherwise stop when ||r||_2 <= max(tol ||b||_2,
// rel_tol ||r_0||_2), or at maxit.  In parity mode only (tol < 1e-12, a
// request at round-off level) also on stagnation: no new minimum of ||r||_2
// for max(50, best_it) iterations once the best residual is at the round-off
// plateau, best <= 1e-8 ||r_0||_2 (A-13'').  (||r||_2 of CG is not monotone:
// it can rise for > 50 iterations early in a solve, so the test is neither
// applied to throughput-mode solves nor before the residual has dropped.)
static double threshold(double bnorm, double res0, double tol, double rel_tol) {
  double a = tol * bnorm, b = rel_tol * res0;
  return a > b ? a : b;
}

// Textbook Jacobi-preconditioned CG ("conjugate gradient"; A-14 Jacobi).
SolveReport cg(const Mesh& m, const LDU& A, const double* b, double* x, double tol, double rel_tol, int maxit) {
  SolveReport rep;
  const int64_t N = m.N;
  std::vector<double> bb(b, b + N), r(N), z(N), p(N), q(N);
  const double bnorm = std::sqrt(dotv(bb, bb));
  if (bnorm == 0.0) {
    for (int64_t i = 0; i < N; ++i) x[i] = 0;
    rep.converged = 1; return rep;
  }
  ldu_apply(m, A, x, q.data());
  for (int64_t i = 0; i < N; ++i) r[i] = b[i] - q[i];
  rep.res0 = rep.res = std::sqrt(dotv(r, r));
  const double thr = threshold(bnorm, rep.res0, tol, rel_tol);
  if (rep.res0 <= thr) { rep.converged = 1; return rep; }
  for (int64_t i = 0; i < N; ++i) { z[i] = r[i] / A.diag[i]; p[i] = z[i]; }
  double rz = dotv(r, z);
  double best = rep.res0; int best_it = 0;
  for (int it = 1; it <= maxit; ++it) {
    ldu_apply(m, A, p.data(), q.data());
    const double pq = dotv(p, q);
    if (!(pq > 0)) { rep.status = E_BREAKDOWN; rep.it = it; return rep; }
    const double alpha = rz / pq;
    for (int64_t i = 0; i < N; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
    rep.res = std::sqrt(dotv(r, r));
    rep.it = it;
    if (rep.res <= thr) { rep.converged = 1; return rep; }
    if (rep.res < best) { best = rep.res; best_it = it; }
    else if (tol < 1e-12 && best <= 1e-8 * rep.res0 && it - best_it >= std::max(50, best_it)) break;  // stagnation, parity mode (A-13)
    for (int64_t i = 0; i < N; ++i) z[i] = r[i] / A.diag[i];
    const double rz_new = dotv(r, z);
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int64_t i = 0; i < N; ++i) p[i] = z[i] + beta * p[i];
  }
  rep.status = E_NOT_CONVERGED;
  return rep;
}

// van der Vorst BiCGStab, right Jacobi preconditioning ("BiCGStab").
SolveReport bicgstab(const Mesh& m, const LDU& A, const double* b, double* x, double tol, double rel_tol, int maxit) {
  SolveReport rep;
  const int64_t N = m.N;
  std::vector<double> bb(b, b + N), r(N), rh(N), p(N, 0), v(N, 0), y(N), s(N), zz(N), t(N);
  const double bnorm = std::sqrt(dotv(bb, bb));
  if (bnorm == 0.0) {
    for (int64_t i = 0; i < N; ++i) x[i] = 0;
    rep.converged = 1; return rep;
  }
  ldu_apply(m, A, x, t.data());
  for (int64_t i = 0; i < N; ++i) { r[i] = b[i] - t[i]; rh[i] = r[i]; }
  rep.res0 = rep.res = std::sqrt(dotv(r, r));
  const double thr = threshold(bnorm, rep.res0, tol, rel_tol);
  if (rep.res0 <= thr) { rep.converged = 1; return rep; }
  double rho_old = 1, alpha = 1, omega = 1;
  double best = rep.res0; int best_it = 0;
  for (int it = 1; it <= maxit; ++it) {
    rep.it = it;
    const double rho = dotv(rh, r);
    if (rho == 0.0) { rep.status = E_BREAKDOWN; return rep; }
    const double beta = (rho / rho_old) * (alpha / omega);
    for (int64_t i = 0; i < N; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
    for (int64_t i = 0; i < N; ++i) y[i] = p[i] / A.diag[i];
    ldu_apply(m, A, y.data(), v.data());
    const double rv = dotv(rh, v);
    if (rv == 0.0) { rep.status = E_BREAKDOWN; return rep; }
    alpha = rho / rv;
    for (int64_t i = 0; i < N; ++i) s[i] = r[i] - alpha * v[i];
    const double snorm = std::sqrt(dotv(s, s));
    if (snorm <= thr) {
      for (int64_t i = 0; i < N; ++i) x[i] += alpha * y[i];
      rep.res = snorm; rep.converged = 1; return rep;
    }
    for (int64_t i = 0; i < N; ++i) zz[i] = s[i] / A.diag[i];
    ldu_apply(m, A, zz.data(), t.data());
    const double tt = dotv(t, t);
    if (tt == 0.0) { rep.status = E_BREAKDOWN; return rep; }
    omega = dotv(t, s) / tt;
    for (int64_t i = 0; i < N; ++i) { x[i] += alpha * y[i] + omega * zz[i]; r[i] = s[i] - omega * t[i]; }
    rep.res = std::sqrt(dotv(r, r));
    if (rep.res <= thr) { rep.converged = 1; return rep; }
    if (omega == 0.0) { rep.status = E_BREAKDOWN; return rep; }
    if (rep.res < best) { best = rep.res; best_it = it; }
    else if (tol < 1e-12 && best <= 1e-8 * rep.res0 && it - best_it >= std::max(50, best_it)) break;
    rho_old = rho;
  }
  rep.status = E_NOT_CONVERGED;
  return rep;
}

// Dense LU with partial pivoting (the "direct mode" pin of O-7).
SolveReport dense_solve(const Mesh& m, const LDU& A, const double* b, double* x) {
  SolveReport rep;
  const int64_t N = m.N;
  std::vector<double> M((size_t)N * N, 0.0), rhs(b, b + N);
  for (int64_t c = 0; c < N; ++c) M[c * N + c] = A.diag[c];
  for (int64_t f = 0; f < m.F; ++f) {
    M[(int64_t)m.owner[f] * N + m.neigh[f]] += A.upper[f];
    M[(int64_t)m.neigh[f] * N + m.owner[f]] += A.lower[f];
  }
  for (int64_t k = 0; k < N; ++k) {
    int64_t piv = k;
    double best = std::fabs(M[k * N + k]);
    for (int64_t i = k + 1; i < N; ++i)
      if (std::fabs(M[i * N + k]) > best) { best = std::fabs(M[i * N + k]); piv = i; }
    if (best == 0.0) { rep.status = E_BREAKDOWN; return rep; }
    if (piv != k) {
      for (int64_t j = 0; j < N; ++j) std::swap(M[k * N + j], M[piv * N + j]);
      std::swap(rhs[k], rhs[piv]);
    }
    for (int64_t i = k + 1; i < N; ++i) {
      const double l = M[i * N + k] / M[k * N + k];
      if (l == 0.0) continue;
      for (int64_t j = k; j < N; ++j) M[i * N + j] -= l * M[k * N + j];
      rhs[i] -= l * rhs[k];
    }
  }
  for (int64_t i = N - 1; i >= 0; --i) {
    double s = rhs[i];
    for (int64_t j = i + 1; j < N; ++j) s -= M[i * N + j] * x[j];
    x[i] = s / M[i * N + i];
  }
  rep.converged = 1;
  return rep;
}

// --------------------------------------------------------------- O-8
// Windkessel RCR update (eq:windkessel_discrete P:420-425, and the FE / BE
// alternatives named at P:425): returns p_c^{n+1}; p_o = p_c^{n+1} + R_p Q.
static int windkessel(double pc, double Q, double dt, double Rp, double Cc, double Rd, int scheme,
                      double* pc_new, double* po) {
  if (!(Rp >= 0) || !(Cc > 0) || !(Rd > 0) || !(dt > 0) || scheme < 0 || scheme > 2) {
    set_error(E_INVALID_WK_PARAMS, "Windkessel needs Rp >= 0, C > 0, Rd > 0, dt > 0", scheme);
    return E_INVALID_WK_PARAMS;
  }
  double p;
  if (scheme == 0) {
    const double e = std::exp(-dt / (Rd * Cc));
    p = pc * e + Rd * Q * (1.0 - e);
  } else if (scheme == 1) {
    p = pc + dt * (Q - pc / Rd) / Cc;               // forward Euler of eq:windkessel_ode_a
  } else {
    p = (pc + dt * Q / Cc) / (1.0 + dt / (Rd * Cc)); // backward Euler
  }
  *pc_new = p;
  *po = p + Rp * Q;
  return OK;
}

// --------------------------------------------------------------- solver
struct Opts {
  double nu, dt, rho;
  double theta;                       // time scheme (Table 1): 1 backward Euler, 0.5 Crank-Nicolson, 0 forward Euler
  int n_corr, n_nonorth, convection;  // convection 0 upwind, 1 central
  int ddt_corr;                       // OpenFOAM ddtCorr Rhie-Chow term in phiHbyA (reading A-42), 0 off
  int64_t p_ref_cell;
  double p_ref_value;
  int direct;
  double p_tol, p_rel_tol, p_rel_tol_final; int p_maxit;
  double U_tol, U_rel_tol; int U_maxit;
};

struct WK { int patch; double Rp, C, Rd, pc; int scheme; };

struct Report {
  SolveReport U[3];
  SolveReport p[16];
  int n_p;
  double cont_err_max, cont_err_sum;
  int n_outlets;
  double Q[64], p_o[64];
  int nonfinite;
};

struct Solver {
  const Mesh* m;
  BCs* b;
  Opts o;
  std::vector<WK> wk;
  double t = 0;
};

static SolveReport solve(const Solver& S, const LDU& A, const double* rhs, double* x,
                         bool sym, double tol, double rel_tol, int maxit) {
  if (S.o.direct) return dense_solve(*S.m, A, rhs, x);
  return sym ? cg(*S.m, A, rhs, x, tol, rel_tol, maxit)
             : bicgstab(*S.m, A, rhs, x, tol, rel_tol, maxit);
}

// O-5: transport LDU for the momentum (ncomp 3, field 'U', diffusivity nu)
// or a passive scalar (ncomp 1, field 's', diffusivity Gamma) from
// (x^n, phi^n, grad x^n) — eq:fvm_momentum P:157-168, eq:conv_face_flux
// P:174-181, eq:upwind P:185-191 (tie -> owner, A-17), central = linear
// weight (A-7), eq:diff_ortho / eq:nonortho_flux with the explicit
// correction from grad x^n (A-16), implicit Euler (A-11).
// Convection 2 (SOU) / 3 (QUICK): upwind implicit part plus the explicit
// deferred correction m_f (x_f^HO - x_f^U) (eq:deferred_correction
// P:193-199), SOU x_f^HO = x_C + (grad x)_C . d_Cf (eq:sou P:200-206), QUICK
// x_f^HO = x_C + 1/2 [(grad x)_C . d_Cf + (x_D - x_C)(d_Cf . d_CD)/|d_CD|^2]
// (SPEC.md:233 reading), C the upwind and D the downwind cell; the
// correction leaves the owner row (b_O -= c) and enters the neighbour row.
// Time scheme (Table 1, reading A-40): the theta method on the spatial
// operator A_s (convection + diffusion; b_s its explicit sources),
//   (V/dt + theta A_s) x* = V/dt x^n + b_s - (1 - theta) A_s x^n,
// theta = 1 backward Euler (A-11), 1/2 Crank-Nicolson, 0 forward Euler.
static void assemble_transport(const Solver& S, int nc, int fi, double diffusivity, const double* U,
                               const double* phi, LDU& M, std::vector<double>& bvec) {
  const Mesh& m = *S.m;
  const BCs& b = *S.b;
  const double nu = diffusivity, dt = S.o.dt;
  const int conv = S.o.convection;
  const int64_t N = m.N;
  M.diag.assign(N, 0); M.lower.assign(m.F, 0); M.upper.assign(m.F, 0);
  bvec.assign((size_t)nc * N, 0);
  std::vector<double> G((size_t)3 * nc * N);
  grad(m, b, fi, nc, U, G.data());
  auto lambda = [&](int64_t f, double md) { return conv == 1 ? m.w[f] : (md >= 0 ? 1.0 : 0.0); };
  // spatial part: cell-wise accumulation in ascending face order into
  // M.diag (= diag of A_s) and bvec (= b_s); the time term and theta after
  for (int64_t f = 0; f < m.F; ++f) {
    const double md = phi[f];
    const double lam = lambda(f, md);
    const double nd = nu * m.delta[f];
    M.upper[f] = (1.0 - lam) * md - nd;
    M.lower[f] = -lam * md - nd;
  }
  for (int64_t c = 0; c < N; ++c) {
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f < m.F) {
        const int64_t O = m.owner[f], Nn = m.neigh[f];
        const double md = phi[f];
        const double lam = lambda(f, md);
        const double nd = nu * m.delta[f];
        const double w = m.w[f];
        double corr[3] = {0, 0, 0};
        for (int k = 0; k < nc; ++k) {
          double s2 = 0;
          for (int l = 0; l < 3; ++l)
            s2 += m.kf[3 * f + l] * (w * G[(size_t)3 * nc * O + 3 * k + l] + (1.0 - w) * G[(size_t)3 * nc * Nn + 3 * k + l]);
          corr[k] = nu * s2;
        }
        double dc[3] = {0, 0, 0};   // deferred convection correction
        if (conv >= 2) {
          const int64_t Cc = md >= 0 ? O : Nn, D = md >= 0 ? Nn : O;
          double dCf[3], dCD[3];
          for (int l = 0; l < 3; ++l) { dCf[l] = m.xf[3 * f + l] - m.xc[3 * Cc + l]; dCD[l] = m.xc[3 * D + l] - m.xc[3 * Cc + l]; }
          const double fCD = (dCf[0] * dCD[0] + dCf[1] * dCD[1] + dCf[2] * dCD[2]) /
                             (dCD[0] * dCD[0] + dCD[1] * dCD[1] + dCD[2] * dCD[2]);
          for (int k = 0; k < nc; ++k) {
            const double* Gc = &G[(size_t)3 * nc * Cc + 3 * k];
            const double gd = Gc[0] * dCf[0] + Gc[1] * dCf[1] + Gc[2] * dCf[2];
            const double xC = U[(size_t)nc * Cc + k], xD = U[(size_t)nc * D + k];
            const double hi = conv == 2 ? xC + gd : xC + 0.5 * (gd + (xD - xC) * fCD);
            dc[k] = md * (hi - xC);
          }
        }
        if (O == c) {
          M.diag[c] += lam * md + nd;
          for (int k = 0; k < nc; ++k) bvec[(size_t)nc * c + k] += corr[k] - dc[k];
        } else {
          M.diag[c] += -(1.0 - lam) * md + nd;
          for (int k = 0; k < nc; ++k) bvec[(size_t)nc * c + k] += -corr[k] + dc[k];
        }
      } else {
        const int p = m.face_patch[f - m.F];
        if (m.pkind[p] == PK_EMPTY) continue;
        const double mb = phi[f];
        if (is_fixed(b, fi, p)) {
          double Ub[3];
          boundary_value(m, b, fi, nc, U, f, Ub);
          const double nd = nu * m.delta_b[f - m.F];
          M.diag[c] += nd;
          for (int k = 0; k < nc; ++k) bvec[(size_t)nc * c + k] += -mb * Ub[k] + nd * Ub[k];
        } else {
          M.diag[c] += mb;  // zeroGradient: outflow m_b x_O
        }
      }
    }
  }
  // time term and theta weighting: b = V/dt x^n + b_s - (1 - theta) (A_s x^n),
  // diag = V/dt + theta diag_s, off-diagonals theta a_s
  const double th = S.o.theta;
  for (int64_t c = 0; c < N; ++c) {
    const double vdt = m.V[c] / dt;
    for (int k = 0; k < nc; ++k) {
      double ax = M.diag[c] * U[(size_t)nc * c + k];
      for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
        const int64_t f = m.cface[i];
        if (f >= m.F) continue;
        if (m.owner[f] == c) ax += M.upper[f] * U[(size_t)nc * m.neigh[f] + k];
        else ax += M.lower[f] * U[(size_t)nc * m.owner[f] + k];
      }
      bvec[(size_t)nc * c + k] = vdt * U[(size_t)nc * c + k] + bvec[(size_t)nc * c + k] - (1.0 - th) * ax;
    }
  }
  for (int64_t c = 0; c < N; ++c) M.diag[c] = m.V[c] / dt + th * M.diag[c];
  for (int64_t f = 0; f < m.F; ++f) { M.upper[f] *= th; M.lower[f] *= th; }
}

static void assemble_momentum(const Solver& S, const double* U, const double* phi, LDU& M,
                              std::vector<double>& bvec) {
  assemble_transport(S, 3, 0, S.o.nu, U, phi, M, bvec);
}

// H_c(U) = b_c - sum_nb a_{c,nb} U_nb (eq:Ap_H P:333-335, pressure excluded)
static void H_op(const Solver& S, const LDU& M, const std::vector<double>& bvec, const double* U,
                 double* H) {
  const Mesh& m = *S.m;
  for (int64_t c = 0; c < m.N; ++c) {
    double acc[3] = {bvec[3 * c], bvec[3 * c + 1], bvec[3 * c + 2]};
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f >= m.F) continue;
      if (m.owner[f] == c) for (int k = 0; k < 3; ++k) acc[k] -= M.upper[f] * U[3 * (int64_t)m.neigh[f] + k];
      else for (int k = 0; k < 3; ++k) acc[k] -= M.lower[f] * U[3 * (int64_t)m.owner[f] + k];
    }
    for (int k = 0; k < 3; ++k) H[3 * c + k] = acc[k];
  }
}

static bool has_fixed_p(const Solver& S) {
  const Mesh& m = *S.m;
  for (size_t p = 0; p < m.pkind.size(); ++p)
    if (m.pkind[p] != PK_EMPTY && is_fixed(*S.b, 1, p)) return true;
  return false;
}

// Pressure matrix (eq:pressure_poisson LHS P:337-340; weight = interpolated
// rAU, A-8): (A p)_c = sum_f c_f (p_c - p_nb) + sum_{b fixed p} c_b p_c.
static void pressure_matrix(const Solver& S, const double* rAU, LDU& A, std::vector<double>& cf,
                            std::vector<double>& cb) {
  const Mesh& m = *S.m;
  A.diag.assign(m.N, 0); A.lower.assign(m.F, 0); A.upper.assign(m.F, 0);
  cf.assign(m.F, 0); cb.assign(m.NF - m.F, 0);
  for (int64_t f = 0; f < m.F; ++f) {
    const double w = m.w[f];
    cf[f] = (w * rAU[m.owner[f]] + (1.0 - w) * rAU[m.neigh[f]]) * m.delta[f];
    A.lower[f] = A.upper[f] = -cf[f];
  }
  for (int64_t f = m.F; f < m.NF; ++f) {
    const int p = m.face_patch[f - m.F];
    if (m.pkind[p] != PK_EMPTY && is_fixed(*S.b, 1, p)) cb[f - m.F] = rAU[m.owner[f]] * m.delta_b[f - m.F];
  }
  for (int64_t c = 0; c < m.N; ++c) {
    double acc = 0;
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      acc += f < m.F ? cf[f] : cb[f - m.F];
    }
    A.diag[c] = acc;
  }
}

// O-6 step 3.3: phiHbyA = interp(HbyA) . S on internal faces; boundary
// faces HbyA_b . S_b with HbyA_b = U_b on fixed-value U, HbyA_O on
// zeroGradient; empty faces 0.  Step 3.3', the optional ddtCorr (A-42,
// OpenFOAM's Euler ddtCorr), on internal faces:
//   phiHbyA += rAU_f c_f (phi^n - U^n_f . S) / dt,
//   c_f = 1 - min(|phi^n - U^n_f . S| / (|phi^n| + 1e-15), 1),
// U^n_f, rAU_f the w-interpolates of the start-of-step U and of rAU.
static void phi_hbya(const Solver& S, const double* HbyA, const double* rAU, const double* Un, const double* phin,
                     std::vector<double>& fv, double* phiHbyA) {
  const Mesh& m = *S.m;
  fv.assign((size_t)3 * m.NF, 0.0);
  interpolate(m, *S.b, 0, 3, HbyA, fv.data());
  for (int64_t f = 0; f < m.NF; ++f) {
    if (f >= m.F && m.is_empty_face(f)) { phiHbyA[f] = 0; continue; }
    phiHbyA[f] = fv[3 * f] * m.Sf[3 * f] + fv[3 * f + 1] * m.Sf[3 * f + 1] + fv[3 * f + 2] * m.Sf[3 * f + 2];
  }
  if (S.o.ddt_corr) {
    for (int64_t f = 0; f < m.F; ++f) {
      const int64_t O = m.owner[f], Nn = m.neigh[f];
      const double w = m.w[f];
      double uS = 0;
      for (int l = 0; l < 3; ++l) uS += (w * Un[3 * O + l] + (1.0 - w) * Un[3 * Nn + l]) * m.Sf[3 * f + l];
      const double d = phin[f] - uS;
      const double c = 1.0 - std::min(std::fabs(d) / (std::fabs(phin[f]) + 1e-15), 1.0);
      const double rf = w * rAU[O] + (1.0 - w) * rAU[Nn];
      phiHbyA[f] += rf * c * d / S.o.dt;
    }
  }
}

// Pressure right-hand side of one non-orthogonal corrector (eq:pressure_poisson
// RHS P:337-339 times -1; the explicit
// non-orthogonal part in the A-9 reading):
//   rhs_c = -D_c(phiHbyA) + sum_{b fixed p} c_b p_b
//           + sum_{f in c} s_cf rAU_f k_f . (grad p)_f,
// rAU_f = w rAU_O + (1 - w) rAU_N, (grad p)_f = w G_O + (1 - w) G_N (A-2),
// G the Gauss gradient of the current p (passed in).  Faces of the cell in
// ascending index.
static void pressure_rhs(const Solver& S, const double* rAU, const double* Dphi, const std::vector<double>& cb,
                         const double* p, const double* Gp, double* rhs) {
  const Mesh& m = *S.m;
  const BCs& b = *S.b;
  for (int64_t c = 0; c < m.N; ++c) {
    double acc = -Dphi[c];
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f < m.F) {
        const int64_t O = m.owner[f], Nn = m.neigh[f];
        const double w = m.w[f];
        const double rf = w * rAU[O] + (1.0 - w) * rAU[Nn];
        double kg = 0;
        for (int l = 0; l < 3; ++l) kg += m.kf[3 * f + l] * (w * Gp[3 * O + l] + (1.0 - w) * Gp[3 * Nn + l]);
        acc += ((O == c) ? 1.0 : -1.0) * rf * kg;
      } else if (cb[f - m.F] != 0.0) {
        double pb;
        boundary_value(m, b, 1, 1, p, f, &pb);
        acc += cb[f - m.F] * pb;
      }
    }
    rhs[c] = acc;
  }
}

// Rhie-Chow flux correction (the A-9 form, no ddtCorr):
//   phi_f = phiHbyA_f - c_f (p_N - p_O) - rAU_f k_f . (grad p)_f,
//   phi_b = phiHbyA_b - c_b (p_b - p_O) on fixed-value p, phiHbyA_b otherwise,
// with the same (grad p)_f as the right-hand side it corrects (so the
// converged flux satisfies sum_f s_cf phi_f = 0 cell by cell).
static void flux_correct(const Solver& S, const double* rAU, const double* phiHbyA, const std::vector<double>& cf,
                         const std::vector<double>& cb, const double* p, const double* Gp, double* phi) {
  const Mesh& m = *S.m;
  const BCs& b = *S.b;
  for (int64_t f = 0; f < m.F; ++f) {
    const int64_t O = m.owner[f], Nn = m.neigh[f];
    const double w = m.w[f];
    const double rf = w * rAU[O] + (1.0 - w) * rAU[Nn];
    double kg = 0;
    for (int l = 0; l < 3; ++l) kg += m.kf[3 * f + l] * (w * Gp[3 * O + l] + (1.0 - w) * Gp[3 * Nn + l]);
    phi[f] = phiHbyA[f] - cf[f] * (p[Nn] - p[O]) - rf * kg;
  }
  for (int64_t f = m.F; f < m.NF; ++f) {
    if (m.is_empty_face(f)) { phi[f] = 0; continue; }
    if (cb[f - m.F] != 0.0) {
      double pb;
      boundary_value(m, b, 1, 1, p, f, &pb);
      phi[f] = phiHbyA[f] - cb[f - m.F] * (pb - p[m.owner[f]]);
    } else {
      phi[f] = phiHbyA[f];
    }
  }
}

// Gauge (A-12, OpenFOAM setReference): A_rr doubled and b_r += A_rr p_ref.
static void apply_reference(const Solver& S, LDU& A, double* rhs) {
  const int64_t r = S.o.p_ref_cell;
  const double d = A.diag[r];
  A.diag[r] = 2.0 * d;
  rhs[r] += d * S.o.p_ref_value;
}

// O-6: one PISO step in icoFoam order.
static int piso_step(Solver& S, double* U, double* p, double* phi, Report& R) {
  const Mesh& m = *S.m;
  BCs& b = *S.b;
  const int64_t N = m.N;
  std::memset(&R, 0, sizeof(R));
  // 0. time-varying boundary values at the new time level t^{n+1} (A-41)
  for (int fi = 0; fi < 2; ++fi)
    for (size_t pt = 0; pt < m.pkind.size(); ++pt)
      if (b.bc[fi][pt].nh >= 0 && b.bc[fi][pt].kind != BC_FIXED && b.bc[fi][pt].kind != BC_PARABOLIC) {
        set_error(E_INVALID_ARG, "time-varying waveform on a patch that is not fixed-value / parabolic", (int64_t)pt);
        return E_INVALID_ARG;
      }
  b.t_eval = S.t + S.o.dt;
  // start-of-step state for the optional ddtCorr term (A-42)
  const std::vector<double> Un(U, U + 3 * N), phin(phi, phi + m.NF);
  // 1. assemble O-5 from (U^n, phi^n, grad U^n)
  LDU M;
  std::vector<double> bvec;
  assemble_momentum(S, U, phi, M, bvec);
  // 2. predictor: M U* = b - V grad p^n, per component (eq:momentum_predictor
  //    P:326-328 made implicit per Table 1, A-6)
  {
    std::vector<double> Gp(3 * N);
    grad(m, b, 1, 1, p, Gp.data());
    std::vector<double> rhs(N), x(N);
    for (int k = 0; k < 3; ++k) {
      for (int64_t c = 0; c < N; ++c) { rhs[c] = bvec[3 * c + k] - m.V[c] * Gp[3 * c + k]; x[c] = U[3 * c + k]; }
      R.U[k] = solve(S, M, rhs.data(), x.data(), false, S.o.U_tol, S.o.U_rel_tol, S.o.U_maxit);
      for (int64_t c = 0; c < N; ++c) U[3 * c + k] = x[c];
    }
  }
  std::vector<double> rAU(N), HbyA(3 * N), H(3 * N), phiHbyA(m.NF), Gp(3 * N), rhs(N), fv(3 * m.NF);
  std::vector<double> pcn(S.wk.size());
  for (size_t i = 0; i < S.wk.size(); ++i) pcn[i] = S.wk[i].pc;
  const bool fixed_p = has_fixed_p(S);
  int np = 0;
  for (int corr = 1; corr <= S.o.n_corr; ++corr) {
    // 3.1 Windkessel (eq:windkessel_Q/discrete P:406-425; A-19 lagged Q,
    //     p_c^{n+1} from the start-of-step p_c^n)
    for (size_t i = 0; i < S.wk.size(); ++i) {
      const WK& w = S.wk[i];
      double Q = 0;
      for (int64_t f = m.pstart[w.patch]; f < m.pstart[w.patch] + m.pn[w.patch]; ++f) Q += phi[f];
      double pc_new, po;
      int st = windkessel(pcn[i], Q, S.o.dt, w.Rp, w.C, w.Rd, w.scheme, &pc_new, &po);
      if (st) return st;
      S.wk[i].pc = pc_new;
      b.wk_value[w.patch] = po / S.o.rho;
      if (i < 64) { R.Q[i] = Q; R.p_o[i] = po; }
    }
    R.n_outlets = (int)S.wk.size();
    // 3.2 rAU = V / a_P; HbyA = H(U) / a_P (A-10: latest U)
    H_op(S, M, bvec, U, H.data());
    for (int64_t c = 0; c < N; ++c) {
      rAU[c] = m.V[c] / M.diag[c];
      for (int k = 0; k < 3; ++k) HbyA[3 * c + k] = H[3 * c + k] / M.diag[c];
    }
    // 3.3 phiHbyA (+ the optional ddtCorr term)
    phi_hbya(S, HbyA.data(), rAU.data(), Un.data(), phin.data(), fv, phiHbyA.data());
    // 3.4 pressure coefficients
    LDU A;
    std::vector<double> cf, cb;
    pressure_matrix(S, rAU.data(), A, cf, cb);
    std::vector<double> Dphi(N);
    div(m, phiHbyA.data(), Dphi.data());
    // 3.5 non-orthogonal loop
    for (int io = 0; io <= S.o.n_nonorth; ++io) {
      grad(m, b, 1, 1, p, Gp.data());
      pressure_rhs(S, rAU.data(), Dphi.data(), cb, p, Gp.data(), rhs.data());
      LDU Ar = A;
      if (!fixed_p) apply_reference(S, Ar, rhs.data());
      const bool final_corr = corr == S.o.n_corr && io == S.o.n_nonorth;
      SolveReport sr = solve(S, Ar, rhs.data(), p, true, S.o.p_tol,
                             final_corr ? S.o.p_rel_tol_final : S.o.p_rel_tol, S.o.p_maxit);
      if (np < 16) R.p[np] = sr;
      np++;
      if (io == S.o.n_nonorth) flux_correct(S, rAU.data(), phiHbyA.data(), cf, cb, p, Gp.data(), phi);
    }
    // 3.6 velocity correction (eq:velocity_correction P:344-346)
    grad(m, b, 1, 1, p, Gp.data());
    for (int64_t c = 0; c < N; ++c)
      for (int k = 0; k < 3; ++k) U[3 * c + k] = HbyA[3 * c + k] - rAU[c] * Gp[3 * c + k];
  }
  R.n_p = np;
  // 4. commit, continuity diagnostic
  S.t += S.o.dt;
  std::vector<double> D(N);
  div(m, phi, D.data());
  double mx = 0, sm = 0;
  for (int64_t c = 0; c < N; ++c) { double a = std::fabs(D[c]); if (a > mx) mx = a; sm += a; }
  R.cont_err_max = mx; R.cont_err_sum = sm;
  int nf = 0;
  for (int64_t i = 0; i < 3 * N; ++i) if (!std::isfinite(U[i])) nf = 1;
  for (int64_t i = 0; i < N; ++i) if (!std::isfinite(p[i])) nf = 1;
  R.nonfinite = nf;
  return nf ? E_NONFINITE : OK;
}

}  // namespace orc

// ====================================================================== C ABI
using namespace orc;

extern "C" {

int orc_windkessel_update(double pc, double Q, double dt, double Rp, double Cc, double Rd, int scheme,
                          double* pc_new, double* po) {
  return windkessel(pc, Q, dt, Rp, Cc, Rd, scheme, pc_new, po);
}

// Generic LDU solves on a mesh's internal-face addressing (solver pins).
// mode: 0 CG, 1 BiCGStab, 2 dense LU.  rep[4] = {it, res0, res, converged}.
int orc_ldu_solve(const void* mp, const double* diag, const double* lower, const double* upper,
                  const double* b, double* x, int mode, double tol, double rel_tol, int maxit, double* rep) {
  const Mesh& m = *(const Mesh*)mp;
  LDU A;
  A.diag.assign(diag, diag + m.N);
  A.lower.assign(lower, lower + m.F);
  A.upper.assign(upper, upper + m.F);
  SolveReport r = mode == 0 ? cg(m, A, b, x, tol, rel_tol, maxit)
                : mode == 1 ? bicgstab(m, A, b, x, tol, rel_tol, maxit)
                            : dense_solve(m, A, b, x);
  rep[0] = r.it; rep[1] = r.res0; rep[2] = r.res; rep[3] = r.converged;
  return r.status;
}
int orc_ldu_apply(const void* mp, const double* diag, const double* lower, const double* upper,
                  const double* x, double* y) {
  const Mesh& m = *(const Mesh*)mp;
  LDU A;
  A.diag.assign(diag, diag + m.N);
  A.lower.assign(lower, lower + m.F);
  A.upper.assign(upper, upper + m.F);
  ldu_apply(m, A, x, y);
  return OK;
}

void* orc_solver_create(const void* mp, void* bp, const double* dopts, const int64_t* iopts) {
  // dopts: nu, dt, rho, p_ref_value, p_tol, p_rel_tol, p_rel_tol_final, U_tol, U_rel_tol, theta
  // iopts: n_corr, n_nonorth, convection, p_ref_cell, direct, p_maxit, U_maxit, ddt_corr
  Solver* S = new Solver();
  S->m = (const Mesh*)mp;
  S->b = (BCs*)bp;
  Opts& o = S->o;
  o.nu = dopts[0]; o.dt = dopts[1]; o.rho = dopts[2]; o.p_ref_value = dopts[3];
  o.p_tol = dopts[4]; o.p_rel_tol = dopts[5]; o.p_rel_tol_final = dopts[6];
  o.U_tol = dopts[7]; o.U_rel_tol = dopts[8]; o.theta = dopts[9];
  o.n_corr = (int)iopts[0]; o.n_nonorth = (int)iopts[1]; o.convection = (int)iopts[2];
  o.p_ref_cell = iopts[3]; o.direct = (int)iopts[4]; o.p_maxit = (int)iopts[5]; o.U_maxit = (int)iopts[6];
  o.ddt_corr = (int)iopts[7];
  return S;
}
void orc_solver_destroy(void* s) { delete (Solver*)s; }

// O-6 step 3.5 pieces on the solver's mesh / p boundary conditions (pins of
// the A-9 reading): rhs of the pressure equation from (rAU, phiHbyA, p), and
// the corrected flux phi from (rAU, phiHbyA, p); (grad p) is the Gauss
// gradient of the given p in both, as in the step.
int orc_pressure_rhs(void* sp, const double* rAU, const double* phiHbyA, const double* p, double* rhs) {
  Solver& S = *(Solver*)sp;
  const Mesh& m = *S.m;
  LDU A;
  std::vector<double> cf, cb, Dphi(m.N), Gp(3 * m.N);
  pressure_matrix(S, rAU, A, cf, cb);
  div(m, phiHbyA, Dphi.data());
  grad(m, *S.b, 1, 1, p, Gp.data());
  pressure_rhs(S, rAU, Dphi.data(), cb, p, Gp.data(), rhs);
  return OK;
}
int orc_phi_hbya(void* sp, const double* HbyA, const double* rAU, const double* Un, const double* phin,
                 double* phiHbyA) {
  Solver& S = *(Solver*)sp;
  std::vector<double> fv;
  phi_hbya(S, HbyA, rAU, Un, phin, fv, phiHbyA);
  return OK;
}
int orc_flux_correct(void* sp, const double* rAU, const double* phiHbyA, const double* p, double* phi) {
  Solver& S = *(Solver*)sp;
  const Mesh& m = *S.m;
  LDU A;
  std::vector<double> cf, cb, Gp(3 * m.N);
  pressure_matrix(S, rAU, A, cf, cb);
  grad(m, *S.b, 1, 1, p, Gp.data());
  flux_correct(S, rAU, phiHbyA, cf, cb, p, Gp.data(), phi);
  return OK;
}

int orc_windkessel_set(void* sp, int32_t patch, double Rp, double Cc, double Rd, double pc0, int scheme) {
  Solver* S = (Solver*)sp;
  if (!(Rp >= 0) || !(Cc > 0) || !(Rd > 0) || scheme < 0 || scheme > 2) {
    set_error(E_INVALID_WK_PARAMS, "Windkessel needs Rp >= 0, C > 0, Rd > 0", patch);
    return E_INVALID_WK_PARAMS;
  }
  for (auto& w : S->wk)
    if (w.patch == patch) { w = {patch, Rp, Cc, Rd, pc0, scheme}; return OK; }
  S->wk.push_back({patch, Rp, Cc, Rd, pc0, scheme});
  S->b->bc[1][patch].kind = BC_WINDKESSEL;
  return OK;
}
double orc_windkessel_pc(const void* sp, int32_t patch) {
  for (auto& w : ((const Solver*)sp)->wk) if (w.patch == patch) return w.pc;
  return NAN;
}

// rep layout (doubles): [0..11] U{it,res0,res,conv}x3, [12] n_p,
// [13..76] p{it,res0,res,conv}x16, [77] cont max, [78] cont sum, [79] n_out,
// [80..143] Q, [144..207] p_o, [208] nonfinite
int orc_piso_step(void* sp, double* U, double* p, double* phi, double* rep) {
  Solver* S = (Solver*)sp;
  for (size_t pt = 0; pt < S->m->pkind.size(); ++pt)
    if (S->m->pkind[pt] != PK_EMPTY && (S->b->bc[0][pt].kind == BC_UNSET || S->b->bc[1][pt].kind == BC_UNSET)) {
      set_error(E_MISSING_BC, "patch without U or p boundary condition", (int64_t)pt);
      return E_MISSING_BC;
    }
  Report R;
  int st = piso_step(*S, U, p, phi, R);
  for (int k = 0; k < 3; ++k) { rep[4 * k] = R.U[k].it; rep[4 * k + 1] = R.U[k].res0; rep[4 * k + 2] = R.U[k].res; rep[4 * k + 3] = R.U[k].converged; }
  rep[12] = R.n_p;
  for (int i = 0; i < 16; ++i) { rep[13 + 4 * i] = R.p[i].it; rep[14 + 4 * i] = R.p[i].res0; rep[15 + 4 * i] = R.p[i].res; rep[16 + 4 * i] = R.p[i].converged; }
  rep[77] = R.cont_err_max; rep[78] = R.cont_err_sum; rep[79] = R.n_outlets;
  for (int i = 0; i < 64; ++i) { rep[80 + i] = R.Q[i]; rep[144 + i] = R.p_o[i]; }
  rep[208] = R.nonfinite;
  return st;
}

// Momentum LDU of O-5 (for operator parity): diag[N], lower[F], upper[F], b[N][3]
int orc_momentum_assemble(void* sp, const double* U, const double* phi, double* diag, double* lower,
                          double* upper, double* b) {
  Solver* S = (Solver*)sp;
  LDU M; std::vector<double> bv;
  assemble_momentum(*S, U, phi, M, bv);
  std::memcpy(diag, M.diag.data(), 8 * M.diag.size());
  std::memcpy(lower, M.lower.data(), 8 * M.lower.size());
  std::memcpy(upper, M.upper.data(), 8 * M.upper.size());
  std::memcpy(b, bv.data(), 8 * bv.size());
  return OK;
}

// One implicit-Euler step of passive-scalar transport (NEXT-1 workload,
// PAPER.md §3.1.2): d(x)/dt + div(phi x) - div(Gamma grad x) = 0
// with the face flux phi fixed, field 's' boundary conditions and the
// solver's convection scheme; BiCGStab (or dense LU in direct mode) from x^n.
int orc_transport_step(void* sp, double* x, const double* phi, double gamma, double* rep) {
  Solver* S = (Solver*)sp;
  LDU M; std::vector<double> bv;
  assemble_transport(*S, 1, 2, gamma, x, phi, M, bv);
  SolveReport r = solve(*S, M, bv.data(), x, false, S->o.U_tol, S->o.U_rel_tol, S->o.U_maxit);
  rep[0] = r.it; rep[1] = r.res0; rep[2] = r.res; rep[3] = r.converged;
  return r.status;
}

// Pressure solve of O-6 step 3.5 on its own: A_p(rAU) p = rhs with the gauge
// of A-12 when no fixed-value p patch exists.  mode 0 CG, 2 dense.
int orc_pressure_solve(void* sp, const double* rAU, const double* rhs_in, double* p, double tol,
                       double rel_tol, int maxit, int mode, double* rep) {
  Solver* S = (Solver*)sp;
  const Mesh& m = *S->m;
  LDU A; std::vector<double> cf, cb;
  pressure_matrix(*S, rAU, A, cf, cb);
  std::vector<double> rhs(rhs_in, rhs_in + m.N);
  if (!has_fixed_p(*S)) apply_reference(*S, A, rhs.data());
  SolveReport r = mode == 2 ? dense_solve(m, A, rhs.data(), p) : cg(m, A, rhs.data(), p, tol, rel_tol, maxit);
  rep[0] = r.it; rep[1] = r.res0; rep[2] = r.res; rep[3] = r.converged;
  return r.status;
}

// ------------------------------------------------------------- NEXT-3
// Adjoint (transposed) LDU apply, written as the definition
// (A^T x)_c = sum_r A_rc x_r over the faces (a scatter, unlike ldu_apply's
// gather): A_ON = upper_f sends x_O to row N, A_NO = lower_f sends x_N to
// row O (the transpose apply behind eq:vjp P:352-358).
int orc_ldu_apply_transpose(const void* mp, const double* diag, const double* lower, const double* upper,
                            const double* x, double* y) {
  const Mesh& m = *(const Mesh*)mp;
  for (int64_t c = 0; c < m.N; ++c) y[c] = diag[c] * x[c];
  for (int64_t f = 0; f < m.F; ++f) {
    const int64_t O = m.owner[f], N = m.neigh[f];
    y[N] += upper[f] * x[O];
    y[O] += lower[f] * x[N];
  }
  return OK;
}

// Adjoint pressure solve of the implicit differentiation (eq:implicit_diff
// P:366-370): (dF/dp)^T lambda = g with F(p) = A_p(rAU) p - rhs, i.e. the
// transposed pressure matrix (gauge of A-12 included), solved "using the same
// iterative solver as the forward pass" (CG; mode 2: dense LU).
int orc_pressure_adjoint(void* sp, const double* rAU, const double* g, double* lambda, double tol, int maxit,
                         int mode, double* rep) {
  Solver* S = (Solver*)sp;
  const Mesh& m = *S->m;
  LDU A; std::vector<double> cf, cb;
  pressure_matrix(*S, rAU, A, cf, cb);
  std::vector<double> rhs(m.N, 0.0);
  if (!has_fixed_p(*S)) apply_reference(*S, A, rhs.data());   // only the matrix part matters here
  LDU At;
  At.diag = A.diag; At.lower = A.upper; At.upper = A.lower;    // transpose: swap the off-diagonal halves
  std::vector<double> gg(g, g + m.N);
  SolveReport r = mode == 2 ? dense_solve(m, At, gg.data(), lambda) : cg(m, At, gg.data(), lambda, tol, 0.0, maxit);
  rep[0] = r.it; rep[1] = r.res0; rep[2] = r.res; rep[3] = r.converged;
  return r.status;
}

// Gradient of L with respect to rAU through a converged pressure solve
// A(rAU) p = rhs(rAU) (implicit function theorem, eq:implicit_diff):
//   dL/dtheta = lambda^T (d rhs/dtheta - (dA/dtheta) p),  A^T lambda = dL/dp.
// Per face coefficient (pressure_matrix): c_f = (w rAU_O + (1-w) rAU_N) delta_f
// enters rows O and N as c_f (p_O - p_N) and (p_N - p_O):
//   dL/dc_f = -(lambda_O - lambda_N) (p_O - p_N);
// a fixed-value boundary face, c_b = rAU_O delta_b, enters row O of A as
// c_b p_O (rhs, which holds its c_b p_b part, is an input of the solve and
// held fixed): dL/dc_b = -lambda_O p_O;
// with the gauge (A-12, no fixed-value p): A_rr -> 2 A_rr and rhs_r += A_rr p_ref,
// so every coefficient in A_rr adds lambda_r (p_ref - p_r).
// Chain rule to rAU: dc_f/drAU_O = w delta_f, dc_f/drAU_N = (1-w) delta_f,
// dc_b/drAU_O = delta_b.  (rhs — divergence, non-orthogonal correction,
// boundary values — is the solve's input and held fixed, as in
// orc_pressure_solve; the gauge's rhs term is part of the solve.)
int orc_pressure_vjp(void* sp, const double* rAU, const double* p, const double* lambda, double* grad) {
  Solver* S = (Solver*)sp;
  const Mesh& m = *S->m;
  BCs& b = *S->b;
  (void)rAU;
  const bool gauge = !has_fixed_p(*S);
  const int64_t r = S->o.p_ref_cell;
  for (int64_t c = 0; c < m.N; ++c) grad[c] = 0.0;
  for (int64_t f = 0; f < m.F; ++f) {
    const int64_t O = m.owner[f], N = m.neigh[f];
    double d = -(lambda[O] - lambda[N]) * (p[O] - p[N]);
    if (gauge && (O == r || N == r)) d += lambda[r] * (S->o.p_ref_value - p[r]);
    grad[O] += d * m.w[f] * m.delta[f];
    grad[N] += d * (1.0 - m.w[f]) * m.delta[f];
  }
  for (int64_t f = m.F; f < m.NF; ++f) {
    const int pt = m.face_patch[f - m.F];
    if (m.pkind[pt] == PK_EMPTY || !is_fixed(b, 1, pt)) continue;
    const int64_t O = m.owner[f];
    grad[O] += -lambda[O] * p[O] * m.delta_b[f - m.F];
  }
  return OK;
}

// Steady Poisson pin (E1, eq:poisson_3d P:445-448) with field 's' BCs:
// sum_f s[delta (phi_N - phi_O) + k . grad phi_f] + sum_b delta_b (phi_b - phi_c) = src_c
// where src_c = f(x_c) V_c (A-33).  Two-point part implicit, correction
// explicit (Picard) until max|dphi| < picard_tol.  Returns Picard sweeps.
int orc_poisson_steady(const void* mp, void* bp, const double* src, double* phi, double picard_tol,
                       int max_picard, int direct, double cg_tol) {
  const Mesh& m = *(const Mesh*)mp;
  BCs& b = *(BCs*)bp;
  const int64_t N = m.N;
  LDU A;
  A.diag.assign(N, 0); A.lower.assign(m.F, 0); A.upper.assign(m.F, 0);
  for (int64_t f = 0; f < m.F; ++f) A.lower[f] = A.upper[f] = -m.delta[f];
  std::vector<double> bfix(N, 0);
  for (int64_t c = 0; c < N; ++c) {
    double acc = 0;
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f < m.F) { acc += m.delta[f]; continue; }
      const int p = m.face_patch[f - m.F];
      if (m.pkind[p] == PK_EMPTY || !is_fixed(b, 2, p)) continue;
      double xb;
      boundary_value(m, b, 2, 1, phi, f, &xb);
      acc += m.delta_b[f - m.F];
      bfix[c] += m.delta_b[f - m.F] * xb;
    }
    A.diag[c] = acc;
  }
  std::vector<double> G(3 * N), rhs(N), old(N);
  int it;
  for (it = 1; it <= max_picard; ++it) {
    grad(m, b, 2, 1, phi, G.data());
    for (int64_t c = 0; c < N; ++c) {
      double corr = 0;
      for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
        const int64_t f = m.cface[i];
        if (f >= m.F) continue;
        const int64_t O = m.owner[f], Nn = m.neigh[f];
        const double w = m.w[f];
        double kg = 0;
        for (int l = 0; l < 3; ++l) kg += m.kf[3 * f + l] * (w * G[3 * O + l] + (1.0 - w) * G[3 * Nn + l]);
        corr += ((O == c) ? 1.0 : -1.0) * kg;
      }
      rhs[c] = -src[c] + corr + bfix[c];
    }
    for (int64_t c = 0; c < N; ++c) old[c] = phi[c];
    if (direct) dense_solve(m, A, rhs.data(), phi);
    else cg(m, A, rhs.data(), phi, cg_tol, 0.0, 100000);
    double mx = 0;
    for (int64_t c = 0; c < N; ++c) mx = std::fmax(mx, std::fabs(phi[c] - old[c]));
    if (mx < picard_tol) break;
  }
  return it;
}

}  // extern "C"
