// oracle/oracle_mesh.cpp — O-0 validation, O-1 geometry, O-2 connectivity,
// O-3 face coefficients, boundary values and the O-4 operators.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  Each function cites the passage
// of /root/reference/PAPER.md ("P:line") or SPEC.md ("S:line") it follows and
// the SURVEY.md §8(c) reading adopted where the paper is silent.
#include "oracle.h"

#include <cmath>
#include <cstring>
#include <string>

namespace orc {

static thread_local int g_err_code = 0;
static thread_local std::string g_err_msg;
static thread_local int64_t g_err_index = -1;

void set_error(int code, const std::string& msg, int64_t index) {
  g_err_code = code; g_err_msg = msg; g_err_index = index;
}

static inline double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static inline void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
static inline double norm3(const double* a) { return std::sqrt(dot3(a, a)); }

// ------------------------------------------------------------------ O-0
// Validate the raw polyMesh.  First failure wins.
static int validate(const int64_t n_points, const int64_t* fo, const int32_t* fp, int64_t nf,
                    const int32_t* owner, const int32_t* neigh, int64_t F,
                    const int32_t* pkind, const int64_t* pstart, const int64_t* pn, int np,
                    int64_t* N_out) {
  // rule 1: vertex indices in range, >= 3 vertices per face
  for (int64_t f = 0; f < nf; ++f) {
    if (fo[f + 1] - fo[f] < 3) { set_error(E_MESH_CONSISTENCY, "face has fewer than 3 vertices", f); return E_MESH_CONSISTENCY; }
    for (int64_t i = fo[f]; i < fo[f + 1]; ++i)
      if (fp[i] < 0 || fp[i] >= n_points) {
        set_error(E_MESH_CONSISTENCY, "face references a point index out of range", f);
        return E_MESH_CONSISTENCY;
      }
  }
  // rule 2: owner/neighbour >= 0, N = 1 + max, every cell has >= 4 faces
  int64_t mx = -1;
  for (int64_t f = 0; f < nf; ++f) {
    if (owner[f] < 0) { set_error(E_MESH_CONSISTENCY, "negative owner index", f); return E_MESH_CONSISTENCY; }
    if (owner[f] > mx) mx = owner[f];
  }
  for (int64_t f = 0; f < F; ++f) {
    if (neigh[f] < 0) { set_error(E_MESH_CONSISTENCY, "negative neighbour index", f); return E_MESH_CONSISTENCY; }
    if (neigh[f] > mx) mx = neigh[f];
  }
  const int64_t N = mx + 1;
  std::vector<int> cnt(N, 0);
  for (int64_t f = 0; f < nf; ++f) cnt[owner[f]]++;
  for (int64_t f = 0; f < F; ++f) cnt[neigh[f]]++;
  for (int64_t c = 0; c < N; ++c)
    if (cnt[c] < 4) { set_error(E_MESH_CONSISTENCY, "cell has fewer than 4 faces", c); return E_MESH_CONSISTENCY; }
  // rule 3: owner < neighbour
  for (int64_t f = 0; f < F; ++f)
    if (!(owner[f] < neigh[f])) { set_error(E_MESH_CONSISTENCY, "internal face with owner >= neighbour", f); return E_MESH_CONSISTENCY; }
  // rule 4: patches tile [F, nf) in order
  int64_t s = F;
  for (int p = 0; p < np; ++p) {
    if (pstart[p] != s || pn[p] < 0) { set_error(E_MESH_CONSISTENCY, "patches do not tile the boundary faces in order", p); return E_MESH_CONSISTENCY; }
    if (pkind[p] < 0 || pkind[p] > 2) { set_error(E_INVALID_ARG, "unknown patch kind", p); return E_INVALID_ARG; }
    s += pn[p];
  }
  if (s != nf) { set_error(E_MESH_CONSISTENCY, "patches do not cover all boundary faces", s); return E_MESH_CONSISTENCY; }
  *N_out = N;
  return OK;
}

// ------------------------------------------------------------------ O-1
// Face area vector and centroid (S_f points out of the owner with
// |S_f| = A_f).  Triangles directly; polygons by the fan about the vertex
// mean with signed sub-triangle weights (reading A-22).
static int face_geometry(const double* P, const int64_t* fo, const int32_t* fp, int64_t f,
                         double* S, double* xf) {
  const int64_t b = fo[f];
  const int m = (int)(fo[f + 1] - b);
  if (m == 3) {
    const double* p0 = P + 3 * (int64_t)fp[b];
    const double* p1 = P + 3 * (int64_t)fp[b + 1];
    const double* p2 = P + 3 * (int64_t)fp[b + 2];
    double a[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
    double c[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
    double n[3];
    cross3(a, c, n);
    for (int d = 0; d < 3; ++d) { S[d] = 0.5 * n[d]; xf[d] = (p0[d] + p1[d] + p2[d]) / 3.0; }
    if (norm3(S) == 0.0) { set_error(E_DEGENERATE_FACE, "face has zero area", f); return E_DEGENERATE_FACE; }
    return OK;
  }
  double xb[3] = {0, 0, 0};
  for (int k = 0; k < m; ++k)
    for (int d = 0; d < 3; ++d) xb[d] += P[3 * (int64_t)fp[b + k] + d];
  for (int d = 0; d < 3; ++d) xb[d] /= m;
  std::vector<double> nk(3 * m), ck(3 * m);
  double Ssum[3] = {0, 0, 0};
  for (int k = 0; k < m; ++k) {
    const double* pk = P + 3 * (int64_t)fp[b + k];
    const double* pk1 = P + 3 * (int64_t)fp[b + (k + 1) % m];
    double e[3] = {pk1[0] - pk[0], pk1[1] - pk[1], pk1[2] - pk[2]};
    double g[3] = {xb[0] - pk[0], xb[1] - pk[1], xb[2] - pk[2]};
    cross3(e, g, &nk[3 * k]);
    for (int d = 0; d < 3; ++d) {
      ck[3 * k + d] = (pk[d] + pk1[d] + xb[d]) / 3.0;
      Ssum[d] += nk[3 * k + d];
    }
  }
  for (int d = 0; d < 3; ++d) S[d] = 0.5 * Ssum[d];
  double A = norm3(S);
  if (A == 0.0) { set_error(E_DEGENERATE_FACE, "face has zero area", f); return E_DEGENERATE_FACE; }
  double Sh[3] = {S[0] / A, S[1] / A, S[2] / A};
  double asum = 0, xs[3] = {0, 0, 0};
  for (int k = 0; k < m; ++k) {
    double a = dot3(&nk[3 * k], Sh);
    asum += a;
    for (int d = 0; d < 3; ++d) xs[d] += a * ck[3 * k + d];
  }
  if (!(asum > 0)) { set_error(E_DEGENERATE_FACE, "face fan weights sum to <= 0", f); return E_DEGENERATE_FACE; }
  for (int d = 0; d < 3; ++d) xf[d] = xs[d] / asum;
  return OK;
}

static int mesh_build(Mesh& m, const double* P, int64_t n_points, const int64_t* fo, const int32_t* fp,
                      int64_t nf, const int32_t* owner, const int32_t* neigh, int64_t F,
                      const int32_t* pkind, const int64_t* pstart, const int64_t* pn, int np, int nonorth) {
  int64_t N = 0;
  int st = validate(n_points, fo, fp, nf, owner, neigh, F, pkind, pstart, pn, np, &N);
  if (st) return st;
  if (nonorth < 0 || nonorth > 3) { set_error(E_INVALID_ARG, "unknown non-orthogonal correction mode", nonorth); return E_INVALID_ARG; }
  m.N = N; m.F = F; m.NF = nf; m.nonorth = nonorth;
  m.owner.assign(owner, owner + nf);
  m.neigh.assign(neigh, neigh + F);
  m.pkind.assign(pkind, pkind + np);
  m.pstart.assign(pstart, pstart + np);
  m.pn.assign(pn, pn + np);
  m.face_patch.assign(nf - F, 0);
  for (int p = 0; p < np; ++p)
    for (int64_t f = pstart[p]; f < pstart[p] + pn[p]; ++f) m.face_patch[f - F] = p;

  // O-2: cell -> faces in ascending face index (scan faces in order)
  m.cptr.assign(N + 1, 0);
  for (int64_t f = 0; f < nf; ++f) m.cptr[owner[f] + 1]++;
  for (int64_t f = 0; f < F; ++f) m.cptr[neigh[f] + 1]++;
  for (int64_t c = 0; c < N; ++c) m.cptr[c + 1] += m.cptr[c];
  m.cface.assign(m.cptr[N], 0);
  {
    std::vector<int64_t> pos(m.cptr.begin(), m.cptr.end() - 1);
    for (int64_t f = 0; f < nf; ++f) {
      m.cface[pos[owner[f]]++] = f;
      if (f < F) m.cface[pos[neigh[f]]++] = f;
    }
  }

  // O-1 face geometry
  m.Sf.assign(3 * nf, 0); m.xf.assign(3 * nf, 0);
  for (int64_t f = 0; f < nf; ++f) {
    st = face_geometry(P, fo, fp, f, &m.Sf[3 * f], &m.xf[3 * f]);
    if (st) return st;
  }
  // O-1 cell geometry: pyramids on the mean of the face centroids
  m.xc.assign(3 * N, 0); m.V.assign(N, 0);
  m.n_bad_pyramids = 0;
  for (int64_t c = 0; c < N; ++c) {
    double xh[3] = {0, 0, 0};
    const int64_t nfc = m.cptr[c + 1] - m.cptr[c];
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i)
      for (int d = 0; d < 3; ++d) xh[d] += m.xf[3 * m.cface[i] + d];
    for (int d = 0; d < 3; ++d) xh[d] /= (double)nfc;
    double v3sum = 0, xs[3] = {0, 0, 0};
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      const double s = (owner[f] == c) ? 1.0 : -1.0;
      const double* S = &m.Sf[3 * f];
      const double* x = &m.xf[3 * f];
      double dxf[3] = {x[0] - xh[0], x[1] - xh[1], x[2] - xh[2]};
      double v3 = s * dot3(S, dxf);
      if (v3 <= 0) m.n_bad_pyramids++;
      v3sum += v3;
      for (int d = 0; d < 3; ++d) xs[d] += v3 * (0.75 * x[d] + 0.25 * xh[d]);
    }
    m.V[c] = v3sum / 3.0;
    if (!(m.V[c] > 0)) { set_error(E_INVERTED_CELL, "cell volume <= 0", c); return E_INVERTED_CELL; }
    for (int d = 0; d < 3; ++d) m.xc[3 * c + d] = xs[d] / v3sum;
  }
  // O-0 rule 5: empty patches only on extruded cells (two parallel empty
  // faces, every other face normal to the empty direction).
  {
    std::vector<int> nempty(N, 0);
    std::vector<int64_t> first_empty(N, -1);
    for (int64_t f = F; f < nf; ++f)
      if (m.is_empty_face(f)) {
        int64_t c = owner[f];
        nempty[c]++;
        if (first_empty[c] < 0) first_empty[c] = f;
      }
    for (int64_t c = 0; c < N; ++c) {
      if (!nempty[c]) continue;
      if (nempty[c] != 2) { set_error(E_MESH_CONSISTENCY, "cell with empty faces must have exactly two", c); return E_MESH_CONSISTENCY; }
      const double* Se = &m.Sf[3 * first_empty[c]];
      double A = norm3(Se), e[3] = {Se[0] / A, Se[1] / A, Se[2] / A};
      for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
        const int64_t f = m.cface[i];
        const double* S = &m.Sf[3 * f];
        double cs = dot3(S, e) / norm3(S);
        if (m.is_empty_face(f)) {
          if (std::fabs(std::fabs(cs) - 1.0) > 1e-12) { set_error(E_MESH_CONSISTENCY, "empty faces of a cell are not parallel", f); return E_MESH_CONSISTENCY; }
        } else if (std::fabs(cs) > 1e-12) {
          set_error(E_MESH_CONSISTENCY, "non-empty face not normal to the empty direction", f);
          return E_MESH_CONSISTENCY;
        }
      }
    }
  }
  // O-3 coefficients (P:229-254 eq:diff_ortho, eq:nonortho_flux; Table 1)
  m.w.assign(F, 0); m.delta.assign(F, 0); m.kf.assign(3 * F, 0);
  m.delta_b.assign(nf - F, 0);
  m.n_clamped = 0;
  for (int64_t f = 0; f < F; ++f) {
    const double* S = &m.Sf[3 * f];
    const double* x = &m.xf[3 * f];
    const double* xO = &m.xc[3 * (int64_t)owner[f]];
    const double* xN = &m.xc[3 * (int64_t)neigh[f]];
    double d[3] = {xN[0] - xO[0], xN[1] - xO[1], xN[2] - xO[2]};
    const double Sd = dot3(S, d);
    if (!(Sd > 0)) { set_error(E_NONCONVEX_PAIR, "S_f . d <= 0 on internal face", f); return E_NONCONVEX_PAIR; }
    // linear-interpolation weight from normal-projected distances (A-1)
    double a[3] = {x[0] - xO[0], x[1] - xO[1], x[2] - xO[2]};
    double bvec[3] = {xN[0] - x[0], xN[1] - x[1], xN[2] - x[2]};
    const double dO = std::fabs(dot3(S, a)), dN = std::fabs(dot3(S, bvec));
    m.w[f] = dN / (dO + dN);
    const double A = norm3(S), dl = norm3(d);
    double dl_ = 0;
    switch (nonorth) {
      case NO_NONE:
        m.delta[f] = A / dl;           // eq:diff_ortho, literal |S|/|d| (A-3), no correction
        break;
      case NO_MINIMUM:
        m.delta[f] = Sd / (dl * dl);   // Delta = (S.d^) d^
        break;
      case NO_ORTHOGONAL:
        m.delta[f] = A / dl;           // Delta = |S| d^
        break;
      default: {                        // over-relaxed Delta = (|S| / |S^.d^|) d^ (A-4 clamp)
        double Shd = Sd / A;
        dl_ = 0.05 * dl;
        if (Shd < dl_) { Shd = dl_; m.n_clamped++; }
        m.delta[f] = A / Shd;
      }
    }
    if (nonorth != NO_NONE)
      for (int k = 0; k < 3; ++k) m.kf[3 * f + k] = S[k] - m.delta[f] * d[k];
  }
  for (int64_t f = F; f < nf; ++f) {
    if (m.is_empty_face(f)) continue;
    const double* S = &m.Sf[3 * f];
    const double* x = &m.xf[3 * f];
    const double* xO = &m.xc[3 * (int64_t)owner[f]];
    double d[3] = {x[0] - xO[0], x[1] - xO[1], x[2] - xO[2]};
    const double A = norm3(S);
    const double Sd = dot3(S, d) / A;
    if (!(Sd > 0)) { set_error(E_NONCONVEX_PAIR, "S_b . d_b <= 0 on boundary face", f); return E_NONCONVEX_PAIR; }
    m.delta_b[f - F] = A / Sd;   // (phi_b - phi_O)|S_b| / (S^_b . d_b)  (A-5)
  }
  return OK;
}

// ------------------------------------------------------------ boundary values
int field_index(char fld) { return fld == 'U' ? 0 : fld == 'p' ? 1 : fld == 's' ? 2 : -1; }

bool is_fixed(const BCs& b, int fi, int64_t p) {
  int k = b.bc[fi][p].kind;
  return k == BC_FIXED || k == BC_PARABOLIC || k == BC_WINDKESSEL;
}

// phi_b (SURVEY.md §8(c) O-4 "Interpolation"): fixedValue -> value, parabolic
// u_b = -U_max (1 - r^2/R^2) n_out (A-18), zeroGradient -> phi_O,
// Windkessel p -> p_o / rho (A-19).
// time-varying inflow multiplier ("time-varying inflow profiles",
// P:582 "pulsatile parabolic velocity profile"; reading A-41: a truncated
// Fourier series of period T, the harmonics summed in ascending k)
double waveform(const BC& bc, double t) {
  double g = bc.wa[0];
  for (int k = 1; k <= bc.nh; ++k) {
    const double w = 2.0 * M_PI * k * t / bc.period;
    g += bc.wa[k] * std::cos(w) + bc.wb[k] * std::sin(w);
  }
  return g;
}

void boundary_value(const Mesh& m, const BCs& b, int fi, int ncomp, const double* x,
                    int64_t f, double* out) {
  const int p = m.face_patch[f - m.F];
  const BC& bc = b.bc[fi][p];
  const int64_t O = m.owner[f];
  switch (bc.kind) {
    case BC_FIXED:
      for (int k = 0; k < ncomp; ++k) out[k] = bc.value[k];
      if (bc.nh >= 0) { const double g = waveform(bc, b.t_eval); for (int k = 0; k < ncomp; ++k) out[k] *= g; }
      break;
    case BC_PARABOLIC: {
      const double* S = &m.Sf[3 * f];
      const double* xb = &m.xf[3 * f];
      double r[3] = {xb[0] - bc.center[0], xb[1] - bc.center[1], xb[2] - bc.center[2]};
      const double rr = dot3(r, r);
      const double A = norm3(S);
      const double mag = bc.u_max * (1.0 - rr / (bc.radius * bc.radius));
      for (int k = 0; k < ncomp; ++k) out[k] = -mag * S[k] / A;
      if (bc.nh >= 0) { const double g = waveform(bc, b.t_eval); for (int k = 0; k < ncomp; ++k) out[k] *= g; }
      break;
    }
    case BC_WINDKESSEL:
      out[0] = b.wk_value[p];
      break;
    default:  // zeroGradient
      for (int k = 0; k < ncomp; ++k) out[k] = x[ncomp * O + k];
  }
}

static int check_bcs(const Mesh& m, const BCs& b, int fi) {
  for (size_t p = 0; p < m.pkind.size(); ++p)
    if (m.pkind[p] != PK_EMPTY && b.bc[fi][p].kind == BC_UNSET) {
      set_error(E_MISSING_BC, "non-empty patch without a boundary condition", (int64_t)p);
      return E_MISSING_BC;
    }
  return OK;
}

// ------------------------------------------------------------------ O-4
// Linear interpolation phi_f = w phi_O + (1 - w) phi_N; boundary
// faces carry phi_b; empty faces are excluded (value 0).
void interpolate(const Mesh& m, const BCs& b, int fi, int ncomp, const double* x, double* xf) {
  for (int64_t f = 0; f < m.F; ++f)
    for (int k = 0; k < ncomp; ++k)
      xf[ncomp * f + k] = m.w[f] * x[ncomp * (int64_t)m.owner[f] + k] +
                          (1.0 - m.w[f]) * x[ncomp * (int64_t)m.neigh[f] + k];
  for (int64_t f = m.F; f < m.NF; ++f) {
    if (m.is_empty_face(f)) { for (int k = 0; k < ncomp; ++k) xf[ncomp * f + k] = 0; continue; }
    boundary_value(m, b, fi, ncomp, x, f, &xf[ncomp * f]);
  }
}

// Gauss-Green gradient from face values (eq:gauss_green P:207-213):
// G_c = (1/V_c) sum_f s_cf phi_f S_f, faces in ascending index, empty faces
// skipped.  g[c][k][l] = d(phi^k)/dx^l.
void grad_from_faces(const Mesh& m, int ncomp, const double* fv, double* g) {
  for (int64_t c = 0; c < m.N; ++c) {
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f >= m.F && m.is_empty_face(f)) continue;
      const double s = (m.owner[f] == c) ? 1.0 : -1.0;
      for (int k = 0; k < ncomp; ++k)
        for (int l = 0; l < 3; ++l) acc[3 * k + l] += s * fv[ncomp * f + k] * m.Sf[3 * f + l];
    }
    for (int k = 0; k < ncomp; ++k)
      for (int l = 0; l < 3; ++l) g[(3 * ncomp) * c + 3 * k + l] = acc[3 * k + l] / m.V[c];
  }
}

void grad(const Mesh& m, const BCs& b, int fi, int ncomp, const double* x, double* g) {
  std::vector<double> fv((size_t)ncomp * m.NF);
  interpolate(m, b, fi, ncomp, x, fv.data());
  grad_from_faces(m, ncomp, fv.data(), g);
}

// Divergence of a face flux, not divided by V (the
// aggregation of eq:aggregate P:297-302 with sigma = +1 owner / -1 neighbour).
void div(const Mesh& m, const double* flux, double* out) {
  for (int64_t c = 0; c < m.N; ++c) {
    double acc = 0;
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f >= m.F && m.is_empty_face(f)) continue;
      acc += ((m.owner[f] == c) ? 1.0 : -1.0) * flux[f];
    }
    out[c] = acc;
  }
}

// Laplacian apply (eq:nonortho_flux P:240-250, with the Gauss gradient of
// P:254 in the correction, w-interpolated to the face, A-2):
//   y_c = sum_f s_cf gamma_f [delta_f (x_N - x_O) + k_f . (grad x)_f]
//       + sum_{b fixed} gamma_O delta_b (x_b - x_c)
// yabs: the same sums of absolute term values (parity scale).
void laplacian(const Mesh& m, const BCs& b, int fi, const double* gamma, const double* x,
               const double* g_in, double* y, double* yabs) {
  std::vector<double> gl;
  const double* G = g_in;
  if (!G) { gl.assign(3 * m.N, 0); grad(m, b, fi, 1, x, gl.data()); G = gl.data(); }
  for (int64_t c = 0; c < m.N; ++c) {
    double acc = 0, aacc = 0;
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f < m.F) {
        const int64_t O = m.owner[f], N = m.neigh[f];
        const double s = (O == c) ? 1.0 : -1.0;
        const double w = m.w[f];
        const double gf = gamma ? w * gamma[O] + (1.0 - w) * gamma[N] : 1.0;
        double corr = 0, acorr = 0;
        for (int l = 0; l < 3; ++l) {
          const double gfl = w * G[3 * O + l] + (1.0 - w) * G[3 * N + l];
          corr += m.kf[3 * f + l] * gfl;
          acorr += std::fabs(m.kf[3 * f + l] * gfl);
        }
        const double q = gf * (m.delta[f] * (x[N] - x[O]) + corr);
        acc += s * q;
        aacc += std::fabs(gf) * (std::fabs(m.delta[f]) * (std::fabs(x[N]) + std::fabs(x[O])) + acorr);
      } else {
        const int p = m.face_patch[f - m.F];
        if (m.pkind[p] == PK_EMPTY || !is_fixed(b, fi, p)) continue;
        double xb;
        boundary_value(m, b, fi, 1, x, f, &xb);
        const double gO = gamma ? gamma[c] : 1.0;
        const double db = m.delta_b[f - m.F];
        acc += gO * db * (xb - x[c]);
        aacc += std::fabs(gO) * db * (std::fabs(xb) + std::fabs(x[c]));
      }
    }
    y[c] = acc;
    if (yabs) yabs[c] = aacc;
  }
}

// y = A x for an LDU matrix, rows accumulated over the row's faces in
// ascending face order.
void ldu_apply(const Mesh& m, const LDU& A, const double* x, double* y) {
  for (int64_t c = 0; c < m.N; ++c) {
    double acc = A.diag[c] * x[c];
    for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
      const int64_t f = m.cface[i];
      if (f >= m.F) continue;
      if (m.owner[f] == c) acc += A.upper[f] * x[m.neigh[f]];
      else acc += A.lower[f] * x[m.owner[f]];
    }
    y[c] = acc;
  }
}

}  // namespace orc

// ====================================================================== C ABI
using namespace orc;

extern "C" {

int orc_last_error_code(void) { return g_err_code; }
const char* orc_last_error_message(void) { return g_err_msg.c_str(); }
int64_t orc_last_error_index(void) { return g_err_index; }

int orc_mesh_create(const double* points, int64_t n_points, const int64_t* face_offsets,
                    const int32_t* face_points, int64_t n_faces, const int32_t* owner,
                    const int32_t* neighbour, int64_t n_internal, const int32_t* patch_kind,
                    const int64_t* patch_start, const int64_t* patch_n, int32_t n_patches,
                    int nonorth, void** out) {
  set_error(0, "", -1);
  Mesh* m = new Mesh();
  int st = mesh_build(*m, points, n_points, face_offsets, face_points, n_faces, owner, neighbour,
                      n_internal, patch_kind, patch_start, patch_n, n_patches, nonorth);
  if (st) { delete m; *out = nullptr; return st; }
  *out = m;
  return OK;
}
void orc_mesh_destroy(void* m) { delete (Mesh*)m; }
void orc_mesh_sizes(const void* mp, int64_t* out) {
  const Mesh* m = (const Mesh*)mp;
  out[0] = m->N; out[1] = m->F; out[2] = m->NF; out[3] = m->n_clamped; out[4] = m->n_bad_pyramids;
}
void orc_mesh_geometry(const void* mp, double* Sf, double* xf, double* xc, double* V) {
  const Mesh* m = (const Mesh*)mp;
  std::memcpy(Sf, m->Sf.data(), m->Sf.size() * 8);
  std::memcpy(xf, m->xf.data(), m->xf.size() * 8);
  std::memcpy(xc, m->xc.data(), m->xc.size() * 8);
  std::memcpy(V, m->V.data(), m->V.size() * 8);
}
void orc_mesh_coeffs(const void* mp, double* w, double* delta, double* k, double* delta_b) {
  const Mesh* m = (const Mesh*)mp;
  std::memcpy(w, m->w.data(), m->w.size() * 8);
  std::memcpy(delta, m->delta.data(), m->delta.size() * 8);
  std::memcpy(k, m->kf.data(), m->kf.size() * 8);
  std::memcpy(delta_b, m->delta_b.data(), m->delta_b.size() * 8);
}

void* orc_bcs_create(const void* mp) {
  const Mesh* m = (const Mesh*)mp;
  BCs* b = new BCs();
  b->m = m;
  for (int i = 0; i < 3; ++i) b->bc[i].assign(m->pkind.size(), BC());
  b->wk_value.assign(m->pkind.size(), 0.0);
  return b;
}
void orc_bcs_destroy(void* b) { delete (BCs*)b; }
// kind: 0 fixedValue, 1 zeroGradient, 2 parabolic, 3 Windkessel
int orc_bcs_set(void* bp, int32_t patch, char fld, int kind, const double* value, double u_max,
                const double* center, double radius) {
  BCs* b = (BCs*)bp;
  int fi = field_index(fld);
  if (fi < 0 || patch < 0 || patch >= (int)b->m->pkind.size() || kind < 0 || kind > 3) {
    set_error(E_INVALID_ARG, "bad bc", patch); return E_INVALID_ARG;
  }
  if ((kind == BC_PARABOLIC && fi != 0) || (kind == BC_WINDKESSEL && fi != 1)) {
    set_error(E_INVALID_ARG, "bc kind not valid for this field", patch); return E_INVALID_ARG;
  }
  BC& c = b->bc[fi][patch];
  c.kind = kind;
  for (int i = 0; i < 3; ++i) { c.value[i] = value ? value[i] : 0; c.center[i] = center ? center[i] : 0; }
  c.u_max = u_max; c.radius = radius;
  return OK;
}
void orc_bcs_set_wk_value(void* bp, int32_t patch, double v) { ((BCs*)bp)->wk_value[patch] = v; }
// time-varying multiplier g(t) of patch's fixed / parabolic value of field fld ('U' or 'p')
int orc_bcs_set_waveform(void* bp, int32_t patch, char fld, double period, int32_t nh, const double* a,
                         const double* bcoef) {
  BCs* b = (BCs*)bp;
  const int fi = field_index(fld);
  if (fi < 0 || fi > 1 || patch < 0 || patch >= (int)b->m->pkind.size() || nh < 0 || nh > 16 || !(period > 0) || !a) {
    set_error(E_INVALID_ARG, "bad waveform", patch); return E_INVALID_ARG;
  }
  BC& c = b->bc[fi][patch];
  c.nh = nh; c.period = period;
  for (int k = 0; k <= 16; ++k) { c.wa[k] = k <= nh ? a[k] : 0; c.wb[k] = (k <= nh && k > 0 && bcoef) ? bcoef[k] : 0; }
  return OK;
}
void orc_bcs_set_time(void* bp, double t) { ((BCs*)bp)->t_eval = t; }

int orc_interpolate(const void* mp, const void* bp, char fld, int ncomp, const double* x, double* xf) {
  const Mesh& m = *(const Mesh*)mp; const BCs& b = *(const BCs*)bp;
  int fi = field_index(fld);
  if (int st = check_bcs(m, b, fi)) return st;
  interpolate(m, b, fi, ncomp, x, xf);
  return OK;
}
int orc_grad(const void* mp, const void* bp, char fld, int ncomp, const double* x, double* g) {
  const Mesh& m = *(const Mesh*)mp; const BCs& b = *(const BCs*)bp;
  int fi = field_index(fld);
  if (int st = check_bcs(m, b, fi)) return st;
  grad(m, b, fi, ncomp, x, g);
  return OK;
}
int orc_grad_faces(const void* mp, int ncomp, const double* fv, double* g) {
  grad_from_faces(*(const Mesh*)mp, ncomp, fv, g);
  return OK;
}
int orc_div(const void* mp, const double* flux, double* out) {
  div(*(const Mesh*)mp, flux, out);
  return OK;
}
int orc_laplacian(const void* mp, const void* bp, char fld, const double* gamma, const double* x,
                  const double* g, double* y, double* yabs) {
  const Mesh& m = *(const Mesh*)mp; const BCs& b = *(const BCs*)bp;
  int fi = field_index(fld);
  if (int st = check_bcs(m, b, fi)) return st;
  laplacian(m, b, fi, gamma, x, g, y, yabs);
  return OK;
}

}  // extern "C"
