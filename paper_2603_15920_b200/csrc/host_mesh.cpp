// host_mesh.cpp — one-time host pipeline of dfvm_mesh_create (SURVEY.md
// §8(a) rows a1-a5): polyMesh validation, fp64 geometry, RCM renumbering,
// face re-sort, cell->face CSR, face coefficients and the block partition
// with its halo lists.  OpenMP-parallel where the work is per face / cell;
// the renumbering itself is the sequential BFS the rules define.
//
// Rules: SURVEY.md §8(c) O-0 (validation), O-1 (geometry), O-3
// (coefficients), O-9 (renumbering, CSR, partition); bit-exact integer maps
// with the independent oracle.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <omp.h>

#include "internal.h"

namespace dfvm {

namespace {

inline double dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// O-1 face area vector and centroid: triangle directly; polygon
// by the fan about the vertex mean, centroid weighted by the signed areas.
int face_geom(const double* P, const int64_t* fo, const int32_t* fp, int64_t f, double* S, double* c) {
  const int64_t b = fo[f];
  const int m = (int)(fo[f + 1] - b);
  if (m == 3) {
    const double* p0 = P + 3 * (int64_t)fp[b];
    const double* p1 = P + 3 * (int64_t)fp[b + 1];
    const double* p2 = P + 3 * (int64_t)fp[b + 2];
    const double u0 = p1[0] - p0[0], u1 = p1[1] - p0[1], u2 = p1[2] - p0[2];
    const double v0 = p2[0] - p0[0], v1 = p2[1] - p0[1], v2 = p2[2] - p0[2];
    S[0] = 0.5 * (u1 * v2 - u2 * v1);
    S[1] = 0.5 * (u2 * v0 - u0 * v2);
    S[2] = 0.5 * (u0 * v1 - u1 * v0);
    for (int d = 0; d < 3; ++d) c[d] = (p0[d] + p1[d] + p2[d]) / 3.0;
    return std::sqrt(dot(S, S)) == 0.0 ? DFVM_E_DEGENERATE_FACE : DFVM_OK;
  }
  double mean[3] = {0, 0, 0};
  for (int i = 0; i < m; ++i)
    for (int d = 0; d < 3; ++d) mean[d] += P[3 * (int64_t)fp[b + i] + d];
  for (int d = 0; d < 3; ++d) mean[d] /= m;
  double nsum[3] = {0, 0, 0};
  double nk[64][3], ck[64][3];
  double* nkp = &nk[0][0];
  double* ckp = &ck[0][0];
  std::vector<double> big;
  if (m > 64) { big.resize(6 * m); nkp = big.data(); ckp = big.data() + 3 * m; }
  for (int i = 0; i < m; ++i) {
    const double* a = P + 3 * (int64_t)fp[b + i];
    const double* e = P + 3 * (int64_t)fp[b + (i + 1) % m];
    const double ex = e[0] - a[0], ey = e[1] - a[1], ez = e[2] - a[2];
    const double gx = mean[0] - a[0], gy = mean[1] - a[1], gz = mean[2] - a[2];
    double* n = nkp + 3 * i;
    n[0] = ey * gz - ez * gy;
    n[1] = ez * gx - ex * gz;
    n[2] = ex * gy - ey * gx;
    for (int d = 0; d < 3; ++d) {
      ckp[3 * i + d] = (a[d] + e[d] + mean[d]) / 3.0;
      nsum[d] += n[d];
    }
  }
  for (int d = 0; d < 3; ++d) S[d] = 0.5 * nsum[d];
  const double A = std::sqrt(dot(S, S));
  if (A == 0.0) return DFVM_E_DEGENERATE_FACE;
  const double sh[3] = {S[0] / A, S[1] / A, S[2] / A};
  double wsum = 0, acc[3] = {0, 0, 0};
  for (int i = 0; i < m; ++i) {
    const double wi = dot(nkp + 3 * i, sh);
    wsum += wi;
    for (int d = 0; d < 3; ++d) acc[d] += wi * ckp[3 * i + d];
  }
  if (!(wsum > 0)) return DFVM_E_DEGENERATE_FACE;
  for (int d = 0; d < 3; ++d) c[d] = acc[d] / wsum;
  return DFVM_OK;
}

}  // namespace

// O-9 steps 1-4: RCM with George-Liu pseudo-peripheral starts.  Key =
// (degree, original id); neighbours expanded in ascending key.
static void rcm_order(int64_t N, const std::vector<int64_t>& aptr, const std::vector<int32_t>& adj,
                      std::vector<int32_t>& new_of_old) {
  std::vector<int32_t> deg(N);
  for (int64_t c = 0; c < N; ++c) deg[c] = (int32_t)(aptr[c + 1] - aptr[c]);
  // cells sorted by key: counting sort on degree, ids ascending within
  int32_t maxdeg = 0;
  for (int64_t c = 0; c < N; ++c) maxdeg = std::max(maxdeg, deg[c]);
  std::vector<int64_t> cnt(maxdeg + 2, 0);
  for (int64_t c = 0; c < N; ++c) cnt[deg[c] + 1]++;
  for (int d = 0; d <= maxdeg; ++d) cnt[d + 1] += cnt[d];
  std::vector<int32_t> by_key(N);
  for (int64_t c = 0; c < N; ++c) by_key[cnt[deg[c]]++] = (int32_t)c;

  std::vector<uint8_t> done(N, 0);
  std::vector<int32_t> mark(N, -1);   // BFS stamp for the level sweeps
  int32_t stamp = 0;
  std::vector<int32_t> order;
  order.reserve(N);
  std::vector<int32_t> cur, nxt;
  auto key_less = [&](int32_t a, int32_t b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; };
  // level sweep from r over not-yet-ordered cells: eccentricity + last level
  auto sweep = [&](int32_t r, std::vector<int32_t>& last) -> int64_t {
    ++stamp;
    cur.assign(1, r);
    mark[r] = stamp;
    int64_t ecc = 0;
    for (;;) {
      nxt.clear();
      for (int32_t c : cur)
        for (int64_t i = aptr[c]; i < aptr[c + 1]; ++i) {
          const int32_t n = adj[i];
          if (!done[n] && mark[n] != stamp) { mark[n] = stamp; nxt.push_back(n); }
        }
      if (nxt.empty()) break;
      ++ecc;
      cur.swap(nxt);
    }
    last = cur;
    return ecc;
  };
  int64_t scan = 0;
  std::vector<int32_t> last, last2;
  while ((int64_t)order.size() < N) {
    while (done[by_key[scan]]) ++scan;
    int32_t r = by_key[scan];
    int64_t er = sweep(r, last);
    for (;;) {
      int32_t x = last[0];
      for (int32_t c : last) if (key_less(c, x)) x = c;
      int64_t ex = sweep(x, last2);
      if (ex > er) { r = x; er = ex; last.swap(last2); } else break;
    }
    // Cuthill-McKee BFS (queue = the order array itself)
    size_t head = order.size();
    order.push_back(r);
    done[r] = 1;
    while (head < order.size()) {
      const int32_t c = order[head++];
      for (int64_t i = aptr[c]; i < aptr[c + 1]; ++i) {
        const int32_t n = adj[i];
        if (!done[n]) { done[n] = 1; order.push_back(n); }
      }
    }
  }
  new_of_old.resize(N);
  for (int64_t k = 0; k < N; ++k) new_of_old[order[k]] = (int32_t)(N - 1 - k);
}

dfvm_status build_host_mesh(HostMesh& H, const double* P, int64_t n_points, const int64_t* fo,
                            const int32_t* fp, int64_t nf, const int32_t* owner, const int32_t* neigh, int64_t F,
                            const dfvm_patch_desc* patches, int32_t np, int nonorth, int rcm) {
  if (nf < 0 || F < 0 || F > nf || np < 0 || !fo || !owner || (F > 0 && !neigh) || (np > 0 && !patches)) {
    set_error(DFVM_E_INVALID_ARG, "invalid mesh array arguments");
    return DFVM_E_INVALID_ARG;
  }
  if (nonorth < 0 || nonorth > 3) { set_error(DFVM_E_INVALID_ARG, "unknown non-orthogonal mode", nonorth); return DFVM_E_INVALID_ARG; }
  // ---- O-0 rule 1: face sizes and vertex range (first failing face wins)
  int64_t bad = -1;
  for (int64_t f = 0; f < nf && bad < 0; ++f) {
    if (fo[f + 1] - fo[f] < 3) { bad = f; break; }
    for (int64_t i = fo[f]; i < fo[f + 1]; ++i)
      if (fp[i] < 0 || fp[i] >= n_points) { bad = f; break; }
  }
  if (bad >= 0) { set_error(DFVM_E_MESH_CONSISTENCY, "face with < 3 vertices or a point index out of range", bad); return DFVM_E_MESH_CONSISTENCY; }
  // ---- rule 2
  int64_t mx = -1;
  for (int64_t f = 0; f < nf; ++f) {
    if (owner[f] < 0) { set_error(DFVM_E_MESH_CONSISTENCY, "negative owner index", f); return DFVM_E_MESH_CONSISTENCY; }
    mx = std::max<int64_t>(mx, owner[f]);
  }
  for (int64_t f = 0; f < F; ++f) {
    if (neigh[f] < 0) { set_error(DFVM_E_MESH_CONSISTENCY, "negative neighbour index", f); return DFVM_E_MESH_CONSISTENCY; }
    mx = std::max<int64_t>(mx, neigh[f]);
  }
  const int64_t N = mx + 1;
  if (N <= 0 || N >= (int64_t)1 << 31 || 2 * F >= (int64_t)1 << 31 || nf >= (int64_t)1 << 31) {
    set_error(DFVM_E_INVALID_ARG, "mesh too large for int32 indices (N, 2F < 2^31)", N);
    return DFVM_E_INVALID_ARG;
  }
  std::vector<int64_t> cptr(N + 1, 0);
  for (int64_t f = 0; f < nf; ++f) cptr[owner[f] + 1]++;
  for (int64_t f = 0; f < F; ++f) cptr[neigh[f] + 1]++;
  for (int64_t c = 0; c < N; ++c)
    if (cptr[c + 1] < 4) { set_error(DFVM_E_MESH_CONSISTENCY, "cell with fewer than 4 faces", c); return DFVM_E_MESH_CONSISTENCY; }
  for (int64_t c = 0; c < N; ++c) cptr[c + 1] += cptr[c];
  // ---- rule 3
  for (int64_t f = 0; f < F; ++f)
    if (owner[f] >= neigh[f]) { set_error(DFVM_E_MESH_CONSISTENCY, "internal face with owner >= neighbour", f); return DFVM_E_MESH_CONSISTENCY; }
  // ---- rule 4
  {
    int64_t s = F;
    for (int p = 0; p < np; ++p) {
      if (patches[p].start_face != s || patches[p].n_faces < 0) { set_error(DFVM_E_MESH_CONSISTENCY, "patches do not tile the boundary faces in order", p); return DFVM_E_MESH_CONSISTENCY; }
      if (patches[p].kind < 0 || patches[p].kind > 2) { set_error(DFVM_E_INVALID_ARG, "unknown patch kind", p); return DFVM_E_INVALID_ARG; }
      s += patches[p].n_faces;
    }
    if (s != nf) { set_error(DFVM_E_MESH_CONSISTENCY, "patches do not cover all boundary faces", s); return DFVM_E_MESH_CONSISTENCY; }
  }
  H.N = N; H.F = F; H.NF = nf; H.nonorth = nonorth;
  H.pkind.resize(np); H.pstart.resize(np); H.pn.resize(np); H.pname.resize(np);
  for (int p = 0; p < np; ++p) {
    H.pkind[p] = patches[p].kind; H.pstart[p] = patches[p].start_face; H.pn[p] = patches[p].n_faces;
    H.pname[p] = patches[p].name ? patches[p].name : "";
  }
  std::vector<int32_t> face_patch(nf - F);
  for (int p = 0; p < np; ++p)
    for (int64_t f = H.pstart[p]; f < H.pstart[p] + H.pn[p]; ++f) face_patch[f - F] = p;
  auto is_empty_old = [&](int64_t f) { return f >= F && H.pkind[face_patch[f - F]] == DFVM_PATCH_EMPTY; };

  // cell -> faces (original numbering, ascending face index)
  std::vector<int64_t> cface(cptr[N]);
  {
    std::vector<int64_t> pos(cptr.begin(), cptr.end() - 1);
    for (int64_t f = 0; f < nf; ++f) {
      cface[pos[owner[f]]++] = f;
      if (f < F) cface[pos[neigh[f]]++] = f;
    }
  }
  // ---- O-1 geometry (original order)
  H.Sf0.assign(3 * nf, 0); H.xf0.assign(3 * nf, 0);
  int64_t bad_face = -1;
#pragma omp parallel for schedule(static) reduction(max : bad_face)
  for (int64_t f = 0; f < nf; ++f)
    if (face_geom(P, fo, fp, f, &H.Sf0[3 * f], &H.xf0[3 * f]) != DFVM_OK) bad_face = std::max(bad_face, f);
  if (bad_face >= 0) {
    for (int64_t f = 0; f < nf; ++f) {  // report the first one
      double S[3], c[3];
      if (face_geom(P, fo, fp, f, S, c) != DFVM_OK) { set_error(DFVM_E_DEGENERATE_FACE, "degenerate face (zero area)", f); break; }
    }
    return DFVM_E_DEGENERATE_FACE;
  }
  H.xc0.assign(3 * N, 0); H.V0.assign(N, 0);
  int64_t bad_cell = -1;
#pragma omp parallel for schedule(static) reduction(max : bad_cell)
  for (int64_t c = 0; c < N; ++c) {
    double xh[3] = {0, 0, 0};
    const int64_t k0 = cptr[c], k1 = cptr[c + 1];
    for (int64_t i = k0; i < k1; ++i)
      for (int d = 0; d < 3; ++d) xh[d] += H.xf0[3 * cface[i] + d];
    for (int d = 0; d < 3; ++d) xh[d] /= (double)(k1 - k0);
    double vs = 0, xs[3] = {0, 0, 0};
    for (int64_t i = k0; i < k1; ++i) {
      const int64_t f = cface[i];
      const double sgn = owner[f] == c ? 1.0 : -1.0;
      const double* S = &H.Sf0[3 * f];
      const double* x = &H.xf0[3 * f];
      const double r[3] = {x[0] - xh[0], x[1] - xh[1], x[2] - xh[2]};
      const double v3 = sgn * dot(S, r);
      vs += v3;
      for (int d = 0; d < 3; ++d) xs[d] += v3 * (0.75 * x[d] + 0.25 * xh[d]);
    }
    H.V0[c] = vs / 3.0;
    if (!(H.V0[c] > 0)) bad_cell = std::max(bad_cell, c);
    for (int d = 0; d < 3; ++d) H.xc0[3 * c + d] = xs[d] / vs;
  }
  if (bad_cell >= 0) {
    for (int64_t c = 0; c < N; ++c)
      if (!(H.V0[c] > 0)) { set_error(DFVM_E_INVERTED_CELL, "cell volume <= 0", c); break; }
    return DFVM_E_INVERTED_CELL;
  }
  // ---- O-0 rule 5: empty faces only on extruded cells
  for (int64_t c = 0; c < N; ++c) {
    int64_t e0 = -1; int ne = 0;
    for (int64_t i = cptr[c]; i < cptr[c + 1]; ++i)
      if (is_empty_old(cface[i])) { if (e0 < 0) e0 = cface[i]; ++ne; }
    if (!ne) continue;
    if (ne != 2) { set_error(DFVM_E_MESH_CONSISTENCY, "a cell with empty faces must have exactly two", c); return DFVM_E_MESH_CONSISTENCY; }
    const double* Se = &H.Sf0[3 * e0];
    const double Ae = std::sqrt(dot(Se, Se));
    for (int64_t i = cptr[c]; i < cptr[c + 1]; ++i) {
      const int64_t f = cface[i];
      const double* S = &H.Sf0[3 * f];
      const double cs = dot(S, Se) / (Ae * std::sqrt(dot(S, S)));
      if (is_empty_old(f) ? std::fabs(std::fabs(cs) - 1.0) > 1e-12 : std::fabs(cs) > 1e-12) {
        set_error(DFVM_E_MESH_CONSISTENCY, "empty patch on a non-extruded cell", f);
        return DFVM_E_MESH_CONSISTENCY;
      }
    }
  }
  // ---- O-9 renumbering
  if (rcm) {
    std::vector<int64_t> aptr(N + 1, 0);
    for (int64_t f = 0; f < F; ++f) { aptr[owner[f] + 1]++; aptr[neigh[f] + 1]++; }
    for (int64_t c = 0; c < N; ++c) aptr[c + 1] += aptr[c];
    std::vector<int32_t> adj(aptr[N]);
    {
      std::vector<int64_t> pos(aptr.begin(), aptr.end() - 1);
      for (int64_t f = 0; f < F; ++f) { adj[pos[owner[f]]++] = neigh[f]; adj[pos[neigh[f]]++] = owner[f]; }
    }
    // collapse duplicates, compact, then order each row by key (degree, id)
    std::vector<int64_t> cptr2(N + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < N; ++c) {
      auto b = adj.begin() + aptr[c], e = adj.begin() + aptr[c + 1];
      std::sort(b, e);
      cptr2[c + 1] = std::unique(b, e) - b;
    }
    for (int64_t c = 0; c < N; ++c) cptr2[c + 1] += cptr2[c];
    std::vector<int32_t> adj2(cptr2[N]);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < N; ++c)
      std::copy(adj.begin() + aptr[c], adj.begin() + aptr[c] + (cptr2[c + 1] - cptr2[c]), adj2.begin() + cptr2[c]);
    adj.clear(); adj.shrink_to_fit();
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < N; ++c)
      std::sort(adj2.begin() + cptr2[c], adj2.begin() + cptr2[c + 1], [&](int32_t a, int32_t b) {
        const int64_t da = cptr2[a + 1] - cptr2[a], db = cptr2[b + 1] - cptr2[b];
        return da != db ? da < db : a < b;
      });
    rcm_order(N, cptr2, adj2, H.new_of_old);
  } else {
    H.new_of_old.resize(N);
    std::iota(H.new_of_old.begin(), H.new_of_old.end(), 0);
  }
  H.old_of_new.resize(N);
  for (int64_t c = 0; c < N; ++c) H.old_of_new[H.new_of_old[c]] = (int32_t)c;
  // ---- O-9 step 5: face re-sort by (a, b, old f); boundary by (new owner, old f)
  H.flip_old.assign(F, 0);
  H.fnew_of_old.assign(nf, 0); H.fold_of_new.assign(nf, 0);
  H.own.assign(F, 0); H.nb.assign(F, 0);
  {
    std::vector<int32_t> a(F), b(F);
    std::vector<int64_t> cnt(N + 1, 0);
    for (int64_t f = 0; f < F; ++f) {
      int32_t x = H.new_of_old[owner[f]], y = H.new_of_old[neigh[f]];
      if (x > y) { std::swap(x, y); H.flip_old[f] = 1; }
      a[f] = x; b[f] = y;
      cnt[x + 1]++;
      H.bw_before = std::max<int64_t>(H.bw_before, (int64_t)neigh[f] - owner[f]);
      H.bw_after = std::max<int64_t>(H.bw_after, (int64_t)y - x);
    }
    for (int64_t c = 0; c < N; ++c) cnt[c + 1] += cnt[c];
    std::vector<int32_t> ord(F);
    {
      std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
      for (int64_t f = 0; f < F; ++f) ord[pos[a[f]]++] = (int32_t)f;   // stable: old f ascending
    }
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t c = 0; c < N; ++c)
      std::sort(ord.begin() + cnt[c], ord.begin() + cnt[c + 1], [&](int32_t u, int32_t v) {
        return b[u] != b[v] ? b[u] < b[v] : u < v;
      });
    for (int64_t k = 0; k < F; ++k) {
      const int32_t f = ord[k];
      H.fnew_of_old[f] = (int32_t)k; H.fold_of_new[k] = f;
      H.own[k] = a[f]; H.nb[k] = b[f];
    }
  }
  H.bown.assign(nf - F, 0); H.bpatch.assign(nf - F, 0);
  for (int p = 0; p < np; ++p) {
    std::vector<std::pair<int32_t, int64_t>> key;
    key.reserve(H.pn[p]);
    for (int64_t f = H.pstart[p]; f < H.pstart[p] + H.pn[p]; ++f) key.push_back({H.new_of_old[owner[f]], f});
    std::sort(key.begin(), key.end());
    for (size_t i = 0; i < key.size(); ++i) {
      const int64_t k = H.pstart[p] + (int64_t)i;
      H.fnew_of_old[key[i].second] = (int32_t)k; H.fold_of_new[k] = (int32_t)key[i].second;
      H.bown[k - F] = key[i].first; H.bpatch[k - F] = p;
    }
  }
  // ---- step 6: CSR of internal incidences, ascending new face index
  H.row_ptr.assign(N + 1, 0);
  for (int64_t k = 0; k < F; ++k) { H.row_ptr[H.own[k] + 1]++; H.row_ptr[H.nb[k] + 1]++; }
  for (int64_t c = 0; c < N; ++c) H.row_ptr[c + 1] += H.row_ptr[c];
  H.inc_face.assign(2 * F, 0); H.inc_nb.assign(2 * F, 0);
  {
    std::vector<int32_t> pos(H.row_ptr.begin(), H.row_ptr.end() - 1);
    for (int64_t k = 0; k < F; ++k) {
      const int32_t o = H.own[k], n = H.nb[k];
      H.inc_face[pos[o]] = (int32_t)k; H.inc_nb[pos[o]++] = n;
      H.inc_face[pos[n]] = (int32_t)((uint32_t)k | 0x80000000u); H.inc_nb[pos[n]++] = o;
    }
  }
  // ---- O-3 face coefficients on the renumbered geometry (flips negate S
  //      exactly; d is taken between the new owner and neighbour)
  H.w.assign(F, 0); H.delta.assign(F, 0); H.k.assign(3 * F, 0); H.delta_b.assign(nf - F, 0);
  int64_t clamped = 0, bad_pair = -1;
#pragma omp parallel for schedule(static) reduction(+ : clamped) reduction(max : bad_pair)
  for (int64_t k = 0; k < F; ++k) {
    const int32_t fo_ = H.fold_of_new[k];
    const double sg = H.flip_old[fo_] ? -1.0 : 1.0;
    const double S[3] = {sg * H.Sf0[3 * fo_], sg * H.Sf0[3 * fo_ + 1], sg * H.Sf0[3 * fo_ + 2]};
    const double* x = &H.xf0[3 * fo_];
    const double* xO = &H.xc0[3 * (int64_t)H.old_of_new[H.own[k]]];
    const double* xN = &H.xc0[3 * (int64_t)H.old_of_new[H.nb[k]]];
    const double d[3] = {xN[0] - xO[0], xN[1] - xO[1], xN[2] - xO[2]};
    const double Sd = dot(S, d);
    if (!(Sd > 0)) { bad_pair = std::max<int64_t>(bad_pair, fo_); continue; }
    const double dOv[3] = {x[0] - xO[0], x[1] - xO[1], x[2] - xO[2]};
    const double dNv[3] = {xN[0] - x[0], xN[1] - x[1], xN[2] - x[2]};
    const double dO = std::fabs(dot(S, dOv)), dN = std::fabs(dot(S, dNv));
    H.w[k] = dN / (dO + dN);
    const double A = std::sqrt(dot(S, S)), L = std::sqrt(dot(d, d));
    double del;
    if (nonorth == DFVM_NONORTH_NONE || nonorth == DFVM_NONORTH_ORTHOGONAL) del = A / L;
    else if (nonorth == DFVM_NONORTH_MINIMUM) del = Sd / (L * L);
    else {
      double proj = Sd / A;
      const double lim = 0.05 * L;
      if (proj < lim) { proj = lim; ++clamped; }
      del = A / proj;
    }
    H.delta[k] = del;
    if (nonorth != DFVM_NONORTH_NONE)
      for (int j = 0; j < 3; ++j) H.k[3 * k + j] = S[j] - del * d[j];
  }
  if (bad_pair >= 0) {
    for (int64_t f = 0; f < F; ++f) {  // first offending face (original numbering)
      const double* S = &H.Sf0[3 * f];
      const double* xO = &H.xc0[3 * (int64_t)owner[f]];
      const double* xN = &H.xc0[3 * (int64_t)neigh[f]];
      const double d[3] = {xN[0] - xO[0], xN[1] - xO[1], xN[2] - xO[2]};
      if (!(dot(S, d) > 0)) { set_error(DFVM_E_NONCONVEX_PAIR, "S_f . d <= 0 on internal face", f); break; }
    }
    return DFVM_E_NONCONVEX_PAIR;
  }
  H.n_clamped = clamped;
  int64_t bad_b = -1;
#pragma omp parallel for schedule(static) reduction(max : bad_b)
  for (int64_t k = F; k < nf; ++k) {
    if (H.pkind[H.bpatch[k - F]] == DFVM_PATCH_EMPTY) continue;
    const int32_t fo_ = H.fold_of_new[k];
    const double* S = &H.Sf0[3 * fo_];
    const double* x = &H.xf0[3 * fo_];
    const double* xO = &H.xc0[3 * (int64_t)H.old_of_new[H.bown[k - F]]];
    const double d[3] = {x[0] - xO[0], x[1] - xO[1], x[2] - xO[2]};
    const double A = std::sqrt(dot(S, S));
    const double proj = dot(S, d) / A;
    if (!(proj > 0)) { bad_b = std::max<int64_t>(bad_b, fo_); continue; }
    H.delta_b[k - F] = A / proj;
  }
  if (bad_b >= 0) { set_error(DFVM_E_NONCONVEX_PAIR, "S_b . d_b <= 0 on boundary face", bad_b); return DFVM_E_NONCONVEX_PAIR; }
  return DFVM_OK;
}

// O-9 step 7: contiguous blocks of the new order; ghosts ordered by
// (peer, new id); send list to q = owned cells adjacent to q, ascending.
void build_part(const HostMesh& H, int P, int rank, Part& T) {
  const int64_t N = H.N;
  T.P = P; T.rank = rank;
  T.lo = (int64_t)rank * N / P;
  T.hi = (int64_t)(rank + 1) * N / P;
  T.n_own = T.hi - T.lo;
  std::vector<std::pair<int32_t, int32_t>> g, s;
  auto part_of = [&](int64_t c) {
    int64_t p = (c * P) / N;                       // candidate, then fix up
    while (p > 0 && c < p * N / P) --p;
    while (p + 1 < P && c >= (p + 1) * N / P) ++p;
    return (int32_t)p;
  };
  for (int64_t c = T.lo; c < T.hi; ++c)
    for (int32_t i = H.row_ptr[c]; i < H.row_ptr[c + 1]; ++i) {
      const int32_t n = H.inc_nb[i];
      if (n < T.lo || n >= T.hi) {
        const int32_t q = part_of(n);
        g.push_back({q, n});
        s.push_back({q, (int32_t)c});
      }
    }
  std::sort(g.begin(), g.end()); g.erase(std::unique(g.begin(), g.end()), g.end());
  std::sort(s.begin(), s.end()); s.erase(std::unique(s.begin(), s.end()), s.end());
  T.ghost_gid.clear(); T.ghost_peer.clear(); T.send_gid.clear(); T.send_peer.clear(); T.peers.clear();
  for (auto& x : g) { T.ghost_peer.push_back(x.first); T.ghost_gid.push_back(x.second); }
  for (auto& x : s) { T.send_peer.push_back(x.first); T.send_gid.push_back(x.second); }
  T.n_ghost = (int64_t)T.ghost_gid.size();
  for (auto& x : g) if (T.peers.empty() || T.peers.back() != x.first) T.peers.push_back(x.first);
  T.peer_ghost_off.assign(T.peers.size() + 1, 0);
  T.peer_send_off.assign(T.peers.size() + 1, 0);
  for (size_t i = 0; i < T.peers.size(); ++i) {
    T.peer_ghost_off[i + 1] = T.peer_ghost_off[i] + std::count(T.ghost_peer.begin(), T.ghost_peer.end(), T.peers[i]);
    T.peer_send_off[i + 1] = T.peer_send_off[i] + std::count(T.send_peer.begin(), T.send_peer.end(), T.peers[i]);
  }
  // local cell numbering
  T.cell_gid.resize(T.n_own + T.n_ghost);
  for (int64_t i = 0; i < T.n_own; ++i) T.cell_gid[i] = (int32_t)(T.lo + i);
  for (int64_t i = 0; i < T.n_ghost; ++i) T.cell_gid[T.n_own + i] = T.ghost_gid[i];
  auto local_of = [&](int32_t gid) -> int32_t {
    if (gid >= T.lo && gid < T.hi) return (int32_t)(gid - T.lo);
    // ghosts are sorted by (peer, gid) == sorted by gid since peers are blocks of gid
    auto it = std::lower_bound(T.ghost_gid.begin(), T.ghost_gid.end(), gid);
    return (int32_t)(T.n_own + (it - T.ghost_gid.begin()));
  };
  // local internal faces: global order, at least one owned endpoint
  T.lf_gid.clear(); T.lf_own.clear(); T.lf_nb.clear();
  if (P == 1) {
    T.lf_gid.resize(H.F); T.lf_own = H.own; T.lf_nb = H.nb;
    std::iota(T.lf_gid.begin(), T.lf_gid.end(), 0);
  } else {
    for (int64_t k = 0; k < H.F; ++k) {
      const bool a = H.own[k] >= T.lo && H.own[k] < T.hi, b = H.nb[k] >= T.lo && H.nb[k] < T.hi;
      if (!a && !b) continue;
      T.lf_gid.push_back((int32_t)k);
      T.lf_own.push_back(local_of(H.own[k]));
      T.lf_nb.push_back(local_of(H.nb[k]));
    }
  }
  // local boundary faces: non-empty (global order) then empty
  T.lb_gid.clear(); T.lb_cell.clear();
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t k = H.F; k < H.NF; ++k) {
      const bool empty = H.pkind[H.bpatch[k - H.F]] == DFVM_PATCH_EMPTY;
      if (empty != (pass == 1)) continue;
      const int32_t o = H.bown[k - H.F];
      if (o < T.lo || o >= T.hi) continue;
      T.lb_gid.push_back((int32_t)k);
      T.lb_cell.push_back((int32_t)(o - T.lo));
      if (pass == 0) T.n_lb++; else T.n_le++;
    }
}

}  // namespace dfvm
