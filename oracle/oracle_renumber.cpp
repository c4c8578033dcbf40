// oracle/oracle_renumber.cpp — O-9: RCM renumbering (George-Liu start),
// face re-sort, cell->face CSR, block partition and halo lists.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  The rules are the exact integer
// specification of SURVEY.md §8(c) O-9 (north_star subsystem (1)); the
// library must reproduce every map bit for bit.
#include "oracle.h"

#include <algorithm>
#include <cstring>
#include <deque>
#include <string>
#include <tuple>

namespace orc {

struct Renum {
  int64_t N = 0, F = 0, NF = 0;
  int P = 1;
  std::vector<int32_t> new_of_old;       // cells
  std::vector<int32_t> face_new_of_old;  // all faces
  std::vector<int8_t> flip_of_old;       // internal faces (by old index)
  std::vector<int32_t> row_ptr;          // [N+1] internal incidences (new numbering)
  std::vector<int32_t> inc_face;         // new face index, bit 31 set when s = -1
  std::vector<int32_t> inc_nb;           // new neighbour id
  std::vector<int32_t> brow_ptr, b_face; // boundary CSR (non-empty boundary faces)
  std::vector<int32_t> part;             // by new id
  // per part: ghosts (new ids, ordered by (peer, new id)), ghost peer,
  // and per peer the send list (new ids)
  std::vector<std::vector<int32_t>> ghost, ghost_peer, send, send_peer;
  int64_t bandwidth_before = 0, bandwidth_after = 0;
};

// O-9 steps 1-4.
static void rcm(const Mesh& m, std::vector<int32_t>& new_of_old) {
  const int64_t N = m.N;
  // adjacency with duplicate pairs collapsed
  std::vector<std::vector<int32_t>> adj(N);
  for (int64_t f = 0; f < m.F; ++f) {
    adj[m.owner[f]].push_back(m.neigh[f]);
    adj[m.neigh[f]].push_back(m.owner[f]);
  }
  for (auto& a : adj) { std::sort(a.begin(), a.end()); a.erase(std::unique(a.begin(), a.end()), a.end()); }
  auto key_less = [&](int32_t a, int32_t b) {
    return adj[a].size() != adj[b].size() ? adj[a].size() < adj[b].size() : a < b;
  };
  // neighbours sorted by key
  for (auto& a : adj) std::sort(a.begin(), a.end(), key_less);
  std::vector<char> placed(N, 0);
  std::vector<int32_t> order;
  order.reserve(N);
  std::vector<int64_t> level(N, -1);
  // BFS levels from r over unplaced cells; returns last level
  auto bfs_levels = [&](int32_t r, std::vector<int32_t>& visited, int64_t& ecc) {
    visited.clear();
    std::vector<int32_t> frontier{r}, next;
    level[r] = 0;
    visited.push_back(r);
    int64_t lv = 0;
    std::vector<int32_t> last = frontier;
    while (!frontier.empty()) {
      next.clear();
      for (int32_t c : frontier)
        for (int32_t nb : adj[c])
          if (!placed[nb] && level[nb] < 0) { level[nb] = lv + 1; next.push_back(nb); visited.push_back(nb); }
      if (next.empty()) break;
      ++lv;
      last = next;
      frontier.swap(next);
    }
    ecc = lv;
    for (int32_t c : visited) level[c] = -1;
    return last;
  };
  int64_t scan = 0;  // smallest-key unplaced search: keys sorted once
  std::vector<int32_t> by_key(N);
  for (int64_t i = 0; i < N; ++i) by_key[i] = (int32_t)i;
  std::sort(by_key.begin(), by_key.end(), key_less);
  std::vector<int32_t> visited;
  while ((int64_t)order.size() < N) {
    while (placed[by_key[scan]]) ++scan;
    int32_t r = by_key[scan];
    // George-Liu pseudo-peripheral start
    int64_t ecc_r;
    std::vector<int32_t> last = bfs_levels(r, visited, ecc_r);
    for (;;) {
      int32_t x = *std::min_element(last.begin(), last.end(), key_less);
      int64_t ecc_x;
      std::vector<int32_t> last_x = bfs_levels(x, visited, ecc_x);
      if (ecc_x > ecc_r) { r = x; ecc_r = ecc_x; last = last_x; }
      else break;
    }
    // Cuthill-McKee BFS
    std::deque<int32_t> q;
    q.push_back(r);
    placed[r] = 1;
    while (!q.empty()) {
      int32_t c = q.front(); q.pop_front();
      order.push_back(c);
      for (int32_t nb : adj[c])
        if (!placed[nb]) { placed[nb] = 1; q.push_back(nb); }
    }
  }
  new_of_old.assign(N, 0);
  for (int64_t k = 0; k < N; ++k) new_of_old[order[N - 1 - k]] = (int32_t)k;
}

static Renum* renumber(const Mesh& m, int P, int use_rcm) {
  Renum* R = new Renum();
  R->N = m.N; R->F = m.F; R->NF = m.NF; R->P = P;
  if (use_rcm) rcm(m, R->new_of_old);
  else { R->new_of_old.resize(m.N); for (int64_t c = 0; c < m.N; ++c) R->new_of_old[c] = (int32_t)c; }
  const auto& nw = R->new_of_old;
  for (int64_t f = 0; f < m.F; ++f) {
    int64_t bw = std::abs((int64_t)m.owner[f] - m.neigh[f]);
    R->bandwidth_before = std::max(R->bandwidth_before, bw);
    R->bandwidth_after = std::max(R->bandwidth_after, (int64_t)std::abs(nw[m.owner[f]] - nw[m.neigh[f]]));
  }
  // step 5: face re-sort
  std::vector<std::tuple<int32_t, int32_t, int64_t>> keys(m.F);
  R->flip_of_old.assign(m.F, 0);
  for (int64_t f = 0; f < m.F; ++f) {
    int32_t a = nw[m.owner[f]], b = nw[m.neigh[f]];
    if (a > b) { std::swap(a, b); R->flip_of_old[f] = 1; }
    keys[f] = std::make_tuple(a, b, f);
  }
  std::sort(keys.begin(), keys.end());
  R->face_new_of_old.assign(m.NF, 0);
  std::vector<int32_t> own_new(m.NF), nb_new(m.F);
  for (int64_t k = 0; k < m.F; ++k) {
    int64_t f = std::get<2>(keys[k]);
    R->face_new_of_old[f] = (int32_t)k;
    own_new[k] = std::get<0>(keys[k]); nb_new[k] = std::get<1>(keys[k]);
  }
  for (size_t p = 0; p < m.pkind.size(); ++p) {
    std::vector<std::pair<int32_t, int64_t>> bk;
    for (int64_t f = m.pstart[p]; f < m.pstart[p] + m.pn[p]; ++f) bk.push_back({nw[m.owner[f]], f});
    std::sort(bk.begin(), bk.end());
    for (size_t i = 0; i < bk.size(); ++i) {
      R->face_new_of_old[bk[i].second] = (int32_t)(m.pstart[p] + (int64_t)i);
      own_new[m.pstart[p] + i] = bk[i].first;
    }
  }
  // step 6: CSR of internal incidences in ascending new face index
  const int64_t N = m.N;
  R->row_ptr.assign(N + 1, 0);
  for (int64_t k = 0; k < m.F; ++k) { R->row_ptr[own_new[k] + 1]++; R->row_ptr[nb_new[k] + 1]++; }
  for (int64_t c = 0; c < N; ++c) R->row_ptr[c + 1] += R->row_ptr[c];
  R->inc_face.assign(2 * m.F, 0); R->inc_nb.assign(2 * m.F, 0);
  {
    std::vector<int32_t> pos(R->row_ptr.begin(), R->row_ptr.end() - 1);
    for (int64_t k = 0; k < m.F; ++k) {
      int32_t o = own_new[k], n = nb_new[k];
      R->inc_face[pos[o]] = (int32_t)k; R->inc_nb[pos[o]++] = n;
      R->inc_face[pos[n]] = (int32_t)((uint32_t)k | 0x80000000u); R->inc_nb[pos[n]++] = o;
    }
  }
  R->brow_ptr.assign(N + 1, 0);
  for (int64_t f = m.F; f < m.NF; ++f)
    if (!m.is_empty_face(f)) R->brow_ptr[own_new[R->face_new_of_old[f]] + 1]++;
  for (int64_t c = 0; c < N; ++c) R->brow_ptr[c + 1] += R->brow_ptr[c];
  R->b_face.assign(R->brow_ptr[N], 0);
  {
    std::vector<int32_t> pos(R->brow_ptr.begin(), R->brow_ptr.end() - 1);
    // boundary faces in ascending new index (via the inverse face map)
    std::vector<int64_t> old_of_new(m.NF);
    for (int64_t f = 0; f < m.NF; ++f) old_of_new[R->face_new_of_old[f]] = f;
    for (int64_t k = m.F; k < m.NF; ++k) {
      int64_t f = old_of_new[k];
      if (m.is_empty_face(f)) continue;
      R->b_face[pos[own_new[k]]++] = (int32_t)k;
    }
  }
  // step 7: partition into P contiguous blocks of the new order
  R->part.assign(N, 0);
  std::vector<int64_t> lo(P + 1);
  for (int p = 0; p <= P; ++p) lo[p] = (int64_t)p * N / P;
  for (int p = 0; p < P; ++p)
    for (int64_t c = lo[p]; c < lo[p + 1]; ++c) R->part[c] = p;
  R->ghost.assign(P, {}); R->ghost_peer.assign(P, {});
  R->send.assign(P, {}); R->send_peer.assign(P, {});
  for (int p = 0; p < P; ++p) {
    std::vector<std::pair<int32_t, int32_t>> g;   // (peer, new id)
    std::vector<std::pair<int32_t, int32_t>> s;   // (peer, new id of owned cell)
    for (int64_t c = lo[p]; c < lo[p + 1]; ++c)
      for (int32_t i = R->row_ptr[c]; i < R->row_ptr[c + 1]; ++i) {
        int32_t nb = R->inc_nb[i];
        int q = R->part[nb];
        if (q != p) { g.push_back({q, nb}); s.push_back({q, (int32_t)c}); }
      }
    std::sort(g.begin(), g.end()); g.erase(std::unique(g.begin(), g.end()), g.end());
    std::sort(s.begin(), s.end()); s.erase(std::unique(s.begin(), s.end()), s.end());
    for (auto& x : g) { R->ghost_peer[p].push_back(x.first); R->ghost[p].push_back(x.second); }
    for (auto& x : s) { R->send_peer[p].push_back(x.first); R->send[p].push_back(x.second); }
  }
  return R;
}

// ------------------------------------------------------------------ O-10
// Partition emulation (the oracle-side check of the
// O-9 partition and halo lists): every part holds only its owned cells
// (ascending new id) and its ghost slice (ghost[p], ordered by (peer, new
// id)); ghost values arrive by an explicit copy from the owning part's send
// list to this part.  Per part, the Gauss gradient of the owned cells and
// then the Laplacian of the owned cells are computed from local data only,
// with the global operators' arithmetic (faces of a cell in ascending
// original index, the same expressions), so the scattered result must equal
// the global apply bit for bit.  A neighbour value that is neither owned nor
// in the ghost slice, or a send list that does not match the receiver's
// ghost slice, is an error (the halo lists are incomplete or misordered).
namespace {
struct PartData {
  int64_t lo = 0, hi = 0;
  std::vector<int32_t> g2l;            // new id -> local index (-1: not local)
  std::vector<double> x, gamma, G;     // local vectors [n_own + n_ghost] (G: x3)
};

// copy the ghost slices of every part from the owners' send lists; nc
// components of the vector selected by `sel`
static int exchange(const Renum& R, std::vector<PartData>& D, int nc, std::vector<double> PartData::*sel) {
  const int P = R.P;
  for (int p = 0; p < P; ++p) {
    const int64_t n_own = D[p].hi - D[p].lo;
    size_t gi = 0;
    for (int q = 0; q < P; ++q) {
      if (q == p) continue;
      // q's send list to p, in order
      std::vector<int32_t> sl;
      for (size_t i = 0; i < R.send[q].size(); ++i)
        if (R.send_peer[q][i] == p) sl.push_back(R.send[q][i]);
      for (size_t i = 0; i < sl.size(); ++i, ++gi) {
        if (gi >= R.ghost[p].size() || R.ghost_peer[p][gi] != q || R.ghost[p][gi] != sl[i]) {
          set_error(E_MESH_CONSISTENCY, "O-10: send list of part " + std::to_string(q) + " does not match the ghost slice of part " +
                    std::to_string(p), sl[i]);
          return E_MESH_CONSISTENCY;
        }
        const int32_t src = D[q].g2l[sl[i]];
        for (int k = 0; k < nc; ++k) (D[p].*sel)[(size_t)nc * (n_own + gi) + k] = (D[q].*sel)[(size_t)nc * src + k];
      }
    }
    if (gi != R.ghost[p].size()) {
      set_error(E_MESH_CONSISTENCY, "O-10: ghost slice of part " + std::to_string(p) + " has cells no peer sends", p);
      return E_MESH_CONSISTENCY;
    }
  }
  return OK;
}
}  // namespace

static int laplacian_parts(const Mesh& m, const BCs& b, int fi, const Renum& R, const double* gamma, const double* x,
                           double* y) {
  const int P = R.P;
  const int64_t N = m.N;
  std::vector<int32_t> old_of_new(N);
  for (int64_t c = 0; c < N; ++c) old_of_new[R.new_of_old[c]] = (int32_t)c;
  std::vector<PartData> D(P);
  for (int p = 0; p < P; ++p) {
    PartData& d = D[p];
    d.lo = (int64_t)p * N / P; d.hi = (int64_t)(p + 1) * N / P;
    const int64_t n_own = d.hi - d.lo, n_loc = n_own + (int64_t)R.ghost[p].size();
    d.g2l.assign(N, -1);
    for (int64_t k = 0; k < n_own; ++k) d.g2l[d.lo + k] = (int32_t)k;
    for (size_t i = 0; i < R.ghost[p].size(); ++i) d.g2l[R.ghost[p][i]] = (int32_t)(n_own + i);
    d.x.assign(n_loc, 0); d.gamma.assign(n_loc, 1.0); d.G.assign(3 * n_loc, 0);
    for (int64_t k = 0; k < n_own; ++k) {          // the initial distribution of the owned values
      d.x[k] = x[old_of_new[d.lo + k]];
      if (gamma) d.gamma[k] = gamma[old_of_new[d.lo + k]];
    }
  }
  int st;
  if ((st = exchange(R, D, 1, &PartData::x))) return st;
  if (gamma && (st = exchange(R, D, 1, &PartData::gamma))) return st;
  auto local = [&](const PartData& d, int64_t old_id, int p) -> int64_t {
    const int32_t l = d.g2l[R.new_of_old[old_id]];
    if (l < 0) set_error(E_MESH_CONSISTENCY, "O-10: part " + std::to_string(p) + " reads a cell it neither owns nor ghosts", old_id);
    return l;
  };
  // boundary value of a scalar field on face f of owned cell with local value xO
  auto bval = [&](int64_t f, double xO) {
    const BC& bc = b.bc[fi][m.face_patch[f - m.F]];
    if (bc.kind == BC_FIXED || bc.kind == BC_PARABOLIC || bc.kind == BC_WINDKESSEL) {
      double v;
      boundary_value(m, b, fi, 1, nullptr, f, &v);
      return v;
    }
    return xO;
  };
  // phase 1: Gauss gradient of the owned cells (grad() = interpolate + grad_from_faces)
  for (int p = 0; p < P; ++p) {
    PartData& d = D[p];
    for (int64_t k = 0; k < d.hi - d.lo; ++k) {
      const int64_t c = old_of_new[d.lo + k];
      double acc[3] = {0, 0, 0};
      for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
        const int64_t f = m.cface[i];
        if (f >= m.F && m.is_empty_face(f)) continue;
        double fv;
        if (f < m.F) {
          const int64_t lO = local(d, m.owner[f], p), lN = local(d, m.neigh[f], p);
          if (lO < 0 || lN < 0) return E_MESH_CONSISTENCY;
          fv = m.w[f] * d.x[lO] + (1.0 - m.w[f]) * d.x[lN];
        } else {
          fv = bval(f, d.x[k]);
        }
        const double s = (m.owner[f] == c) ? 1.0 : -1.0;
        for (int l = 0; l < 3; ++l) acc[l] += s * fv * m.Sf[3 * f + l];
      }
      for (int l = 0; l < 3; ++l) d.G[3 * k + l] = acc[l] / m.V[c];
    }
  }
  if ((st = exchange(R, D, 3, &PartData::G))) return st;
  // phase 2: Laplacian of the owned cells (laplacian() with the gradient given)
  for (int p = 0; p < P; ++p) {
    PartData& d = D[p];
    for (int64_t k = 0; k < d.hi - d.lo; ++k) {
      const int64_t c = old_of_new[d.lo + k];
      double acc = 0;
      for (int64_t i = m.cptr[c]; i < m.cptr[c + 1]; ++i) {
        const int64_t f = m.cface[i];
        if (f < m.F) {
          const int64_t lO = local(d, m.owner[f], p), lN = local(d, m.neigh[f], p);
          if (lO < 0 || lN < 0) return E_MESH_CONSISTENCY;
          const double s = (m.owner[f] == c) ? 1.0 : -1.0;
          const double w = m.w[f];
          const double gf = gamma ? w * d.gamma[lO] + (1.0 - w) * d.gamma[lN] : 1.0;
          double corr = 0;
          for (int l = 0; l < 3; ++l) corr += m.kf[3 * f + l] * (w * d.G[3 * lO + l] + (1.0 - w) * d.G[3 * lN + l]);
          acc += s * (gf * (m.delta[f] * (d.x[lN] - d.x[lO]) + corr));
        } else {
          const int pt = m.face_patch[f - m.F];
          if (m.pkind[pt] == PK_EMPTY || !is_fixed(b, fi, pt)) continue;
          const double xb = bval(f, d.x[k]);
          const double gO = gamma ? d.gamma[k] : 1.0;
          acc += gO * m.delta_b[f - m.F] * (xb - d.x[k]);
        }
      }
      y[c] = acc;
    }
  }
  return OK;
}

}  // namespace orc

using namespace orc;

extern "C" {

void* orc_renumber_create(const void* mp, int n_parts, int use_rcm) {
  return renumber(*(const Mesh*)mp, n_parts, use_rcm);
}
void orc_renumber_destroy(void* r) { delete (Renum*)r; }
// sizes: N, F, NF, I (=2F), nB (non-empty boundary faces), bw_before, bw_after
void orc_renumber_sizes(const void* rp, int64_t* out) {
  const Renum* R = (const Renum*)rp;
  out[0] = R->N; out[1] = R->F; out[2] = R->NF; out[3] = (int64_t)R->inc_face.size();
  out[4] = (int64_t)R->b_face.size(); out[5] = R->bandwidth_before; out[6] = R->bandwidth_after;
}
void orc_renumber_maps(const void* rp, int32_t* cell_new_of_old, int32_t* face_new_of_old, int8_t* flip_of_old,
                       int32_t* row_ptr, int32_t* inc_face, int32_t* inc_nb, int32_t* brow_ptr, int32_t* b_face,
                       int32_t* part) {
  const Renum* R = (const Renum*)rp;
  std::memcpy(cell_new_of_old, R->new_of_old.data(), 4 * R->new_of_old.size());
  std::memcpy(face_new_of_old, R->face_new_of_old.data(), 4 * R->face_new_of_old.size());
  std::memcpy(flip_of_old, R->flip_of_old.data(), R->flip_of_old.size());
  std::memcpy(row_ptr, R->row_ptr.data(), 4 * R->row_ptr.size());
  std::memcpy(inc_face, R->inc_face.data(), 4 * R->inc_face.size());
  std::memcpy(inc_nb, R->inc_nb.data(), 4 * R->inc_nb.size());
  std::memcpy(brow_ptr, R->brow_ptr.data(), 4 * R->brow_ptr.size());
  std::memcpy(b_face, R->b_face.data(), 4 * R->b_face.size());
  std::memcpy(part, R->part.data(), 4 * R->part.size());
}
// per part: out[0] = n_ghost, out[1] = n_send
void orc_renumber_part_sizes(const void* rp, int p, int64_t* out) {
  const Renum* R = (const Renum*)rp;
  out[0] = (int64_t)R->ghost[p].size(); out[1] = (int64_t)R->send[p].size();
}
// O-10: y (original numbering) = Laplacian of x applied part by part (see above)
int orc_laplacian_parts(const void* mp, const void* bp, int fi, const void* rp, const double* gamma, const double* x,
                        double* y) {
  return laplacian_parts(*(const Mesh*)mp, *(const BCs*)bp, fi, *(const Renum*)rp, gamma, x, y);
}
void orc_renumber_part(const void* rp, int p, int32_t* ghost, int32_t* ghost_peer, int32_t* send,
                       int32_t* send_peer) {
  const Renum* R = (const Renum*)rp;
  std::memcpy(ghost, R->ghost[p].data(), 4 * R->ghost[p].size());
  std::memcpy(ghost_peer, R->ghost_peer[p].data(), 4 * R->ghost_peer[p].size());
  std::memcpy(send, R->send[p].data(), 4 * R->send[p].size());
  std::memcpy(send_peer, R->send_peer[p].data(), 4 * R->send_peer[p].size());
}

}  // extern "C"
