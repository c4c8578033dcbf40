// synth/meshgen.cpp — seeded synthetic polyMesh generators.
//
// INPUT TOOLING ONLY. This module produces OpenFOAM-convention raw meshes
// (points, face rings, owner, neighbour, patches) for the tests, smoke() and
// bench.py.  It holds none of the finite-volume method's arithmetic: it never
// computes face area vectors, volumes, weights or any operator.  Both the CPU
// oracle (oracle/) and the CUDA library (paper_2603_15920_b200/) consume its
// output; neither is linked into it.
//
// Mesh recipes follow SURVEY.md §8(d2) (configs C1-C5) and §7 step 1:
//   * box hex slab / cube (cavity C1, Poisson pins),
//   * box tets: alternating 5-tet (global vertex parity) or Kuhn 6-tet,
//   * O-grid circular pipe (central n x n square + 4 ring blocks n x m_r),
//     hex or alternating 5-tet (C2, C5),
//   * voxelised H-tree vascular geometry -> alternating 5-tet (C4),
//   * extruded polygon (Voronoi dual) slab for the cylinder (C3) — the
//     polygons are passed in from Python (scipy Delaunay), this file only
//     assembles the polyMesh.
// Face rings are oriented outward of the owner ("S_f points from
// the owner cell outward"), internal faces precede boundary faces, owner <
// neighbour, and internal faces are in upper-triangular (owner, neighbour)
// order, as OpenFOAM's polyMesh requires.
//
// Cell ids are scrambled with a seeded permutation before the faces are
// ordered, so the renumbering the library performs is measured, not
// inherited.
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <string>
#include <algorithm>
#include <functional>
#include <numeric>

namespace {

// ---------------------------------------------------------------- random
// splitmix64 (order-independent: value depends only on (seed, id)).
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// u(seed, id) in [-1, 1) with 53 random bits.
inline double urand(uint64_t seed, uint64_t id) {
  uint64_t h = splitmix64(seed ^ (id * 0x9E3779B97F4A7C15ull));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

struct Patch { std::string name; int kind; };  // kind: 0 generic, 1 wall, 2 empty

struct Mesh {
  std::vector<double> points;       // [n_p][3]
  std::vector<int64_t> face_offsets;
  std::vector<int32_t> face_points;
  std::vector<int32_t> owner, neighbour;
  std::vector<Patch> patches;
  std::vector<int64_t> patch_start, patch_n;
  int64_t n_cells = 0;
  std::vector<double> meta;        // generator metadata (e.g. pipe radius)
  std::string error;
};

// A cell is a list of vertex ids plus a type that tells how to enumerate its
// faces.  type 0: tet (4 ids), 1: hex (8 ids, VTK order), 2: extruded polygon
// (m bottom ids then m top ids).
struct Cells {
  std::vector<int64_t> ptr{0};
  std::vector<int32_t> v;
  std::vector<uint8_t> type;
  void add(int t, const int32_t* ids, int n) {
    type.push_back((uint8_t)t);
    v.insert(v.end(), ids, ids + n);
    ptr.push_back((int64_t)v.size());
  }
  int64_t size() const { return (int64_t)type.size(); }
  int nfaces(int64_t c) const {
    if (type[c] == 0) return 4;
    if (type[c] == 1) return 6;
    int m = (int)(ptr[c + 1] - ptr[c]) / 2;
    return m + 2;
  }
  // ring of face k of cell c (unoriented: builder orients by geometry)
  int face(int64_t c, int k, int32_t* out) const {
    const int32_t* a = &v[ptr[c]];
    if (type[c] == 0) {
      static const int T[4][3] = {{0, 2, 1}, {0, 1, 3}, {0, 3, 2}, {1, 2, 3}};
      for (int i = 0; i < 3; ++i) out[i] = a[T[k][i]];
      return 3;
    }
    if (type[c] == 1) {
      static const int H[6][4] = {{0, 3, 2, 1}, {4, 5, 6, 7}, {0, 1, 5, 4},
                                  {3, 7, 6, 2}, {0, 4, 7, 3}, {1, 2, 6, 5}};
      for (int i = 0; i < 4; ++i) out[i] = a[H[k][i]];
      return 4;
    }
    int m = (int)(ptr[c + 1] - ptr[c]) / 2;
    if (k == 0) { for (int i = 0; i < m; ++i) out[i] = a[m - 1 - i]; return m; }
    if (k == 1) { for (int i = 0; i < m; ++i) out[i] = a[m + i]; return m; }
    int s = k - 2, s1 = (s + 1) % m;
    out[0] = a[s]; out[1] = a[s1]; out[2] = a[m + s1]; out[3] = a[m + s];
    return 4;
  }
};

// classifier: (face mean point, face Newell normal) -> patch index
using Classifier = std::function<int(const double*, const double*)>;

struct Vec3 { double x, y, z; };

// Newell normal and mean point of a ring (used only to orient rings and
// classify boundary faces; the method's S_f is computed by the consumers).
inline void ring_geom(const std::vector<double>& P, const int32_t* r, int m,
                      double* mean, double* nrm) {
  mean[0] = mean[1] = mean[2] = 0; nrm[0] = nrm[1] = nrm[2] = 0;
  for (int i = 0; i < m; ++i) {
    const double* a = &P[3 * (int64_t)r[i]];
    const double* b = &P[3 * (int64_t)r[(i + 1) % m]];
    mean[0] += a[0]; mean[1] += a[1]; mean[2] += a[2];
    nrm[0] += (a[1] - b[1]) * (a[2] + b[2]);
    nrm[1] += (a[2] - b[2]) * (a[0] + b[0]);
    nrm[2] += (a[0] - b[0]) * (a[1] + b[1]);
  }
  mean[0] /= m; mean[1] /= m; mean[2] /= m;
}

// Seeded permutation of [0, n) (Fisher-Yates on a splitmix64 stream).
std::vector<int32_t> scramble_perm(int64_t n, uint64_t seed) {
  std::vector<int32_t> p(n);
  std::iota(p.begin(), p.end(), 0);
  if (seed == 0) return p;  // seed 0: identity (no scramble)
  uint64_t s = splitmix64(seed);
  for (int64_t i = n - 1; i > 0; --i) {
    s = splitmix64(s);
    int64_t j = (int64_t)(s % (uint64_t)(i + 1));
    std::swap(p[i], p[j]);
  }
  return p;
}

// Assemble a polyMesh from cells: match faces by their three smallest vertex
// ids (bucketed by the smallest), orient rings outward of each cell, scramble
// cell ids, order internal faces by (owner, neighbour) and boundary faces by
// (patch, owner, generation order).
void build(Mesh& M, const Cells& C, const std::vector<Patch>& patches,
           const Classifier& classify, uint64_t scramble_seed) {
  const int64_t N = C.size();
  const int64_t NP = (int64_t)M.points.size() / 3;
  M.n_cells = N;
  M.patches = patches;
  std::vector<int32_t> perm = scramble_perm(N, scramble_seed);  // generated -> scrambled id

  // face instances
  std::vector<int64_t> cfo(N + 1, 0);
  for (int64_t c = 0; c < N; ++c) cfo[c + 1] = cfo[c] + C.nfaces(c);
  const int64_t NI = cfo[N];
  std::vector<int32_t> minv(NI);
  std::vector<uint64_t> key23(NI);   // (second, third smallest)
  std::vector<uint8_t> flipped(N, 0);
  {
    int32_t ring[64];
    std::vector<double> cm(3);
    for (int64_t c = 0; c < N; ++c) {
      // cell mean point for orientation
      double cc[3] = {0, 0, 0};
      int64_t nv = C.ptr[c + 1] - C.ptr[c];
      for (int64_t i = C.ptr[c]; i < C.ptr[c + 1]; ++i)
        for (int d = 0; d < 3; ++d) cc[d] += M.points[3 * (int64_t)C.v[i] + d];
      for (int d = 0; d < 3; ++d) cc[d] /= (double)nv;
      // orientation decided on face 0 (cells are convex; all rings of a
      // cell share the handedness of its vertex ordering)
      int m = C.face(c, 0, ring);
      double mean[3], nrm[3];
      ring_geom(M.points, ring, m, mean, nrm);
      double dot = nrm[0] * (mean[0] - cc[0]) + nrm[1] * (mean[1] - cc[1]) + nrm[2] * (mean[2] - cc[2]);
      flipped[c] = dot < 0;
      for (int k = 0; k < C.nfaces(c); ++k) {
        int mm = C.face(c, k, ring);
        int32_t s[64];
        std::memcpy(s, ring, mm * sizeof(int32_t));
        std::partial_sort(s, s + 3, s + mm);
        minv[cfo[c] + k] = s[0];
        key23[cfo[c] + k] = ((uint64_t)(uint32_t)s[1] << 32) | (uint32_t)s[2];
      }
    }
  }
  // bucket by smallest vertex (counting sort)
  std::vector<int64_t> boff(NP + 1, 0);
  for (int64_t i = 0; i < NI; ++i) boff[minv[i] + 1]++;
  for (int64_t v = 0; v < NP; ++v) boff[v + 1] += boff[v];
  std::vector<int64_t> bidx(NI);
  {
    std::vector<int64_t> pos(boff.begin(), boff.end() - 1);
    for (int64_t i = 0; i < NI; ++i) bidx[pos[minv[i]]++] = i;
  }
  std::vector<int64_t> match(NI, -1);
  for (int64_t v = 0; v < NP; ++v) {
    int64_t b0 = boff[v], b1 = boff[v + 1];
    if (b1 - b0 < 2) continue;
    std::sort(bidx.begin() + b0, bidx.begin() + b1, [&](int64_t a, int64_t b) {
      return key23[a] != key23[b] ? key23[a] < key23[b] : a < b;
    });
    for (int64_t i = b0; i + 1 < b1; ++i) {
      int64_t a = bidx[i], b = bidx[i + 1];
      if (key23[a] == key23[b]) {
        if (match[a] != -1 || match[b] != -1 || (i + 2 < b1 && key23[bidx[i + 2]] == key23[a])) {
          M.error = "non-manifold face (shared by more than two cells)";
          return;
        }
        match[a] = b; match[b] = a; ++i;
      }
    }
  }
  // instance -> cell
  std::vector<int32_t> icell(NI);
  for (int64_t c = 0; c < N; ++c)
    for (int64_t i = cfo[c]; i < cfo[c + 1]; ++i) icell[i] = (int32_t)c;

  // internal faces: owner = smaller scrambled id, use owner's instance
  struct IF { int32_t o, n; int64_t inst; };
  std::vector<IF> inter;
  inter.reserve(NI / 2);
  struct BF { int32_t patch, o; int64_t inst; };
  std::vector<BF> bnd;
  int32_t ring[64];
  for (int64_t i = 0; i < NI; ++i) {
    int32_t ci = perm[icell[i]];
    if (match[i] >= 0) {
      int32_t cj = perm[icell[match[i]]];
      if (ci < cj) inter.push_back({ci, cj, i});
    } else {
      int64_t c = icell[i];
      int k = (int)(i - cfo[c]);
      int m = C.face(c, k, ring);
      if (flipped[c]) std::reverse(ring, ring + m);
      double mean[3], nrm[3];
      ring_geom(M.points, ring, m, mean, nrm);
      int p = classify(mean, nrm);
      if (p < 0 || p >= (int)patches.size()) { M.error = "boundary face not classified"; return; }
      bnd.push_back({p, ci, i});
    }
  }
  // (owner, neighbour) order: counting sort by owner then sort small runs
  {
    std::vector<int64_t> oo(N + 1, 0);
    for (auto& f : inter) oo[f.o + 1]++;
    for (int64_t c = 0; c < N; ++c) oo[c + 1] += oo[c];
    std::vector<IF> tmp(inter.size());
    std::vector<int64_t> pos(oo.begin(), oo.end() - 1);
    for (auto& f : inter) tmp[pos[f.o]++] = f;
    for (int64_t c = 0; c < N; ++c)
      std::sort(tmp.begin() + oo[c], tmp.begin() + oo[c + 1],
                [](const IF& a, const IF& b) { return a.n < b.n; });
    inter.swap(tmp);
  }
  std::stable_sort(bnd.begin(), bnd.end(), [](const BF& a, const BF& b) {
    return a.patch != b.patch ? a.patch < b.patch : a.o < b.o;
  });
  const int64_t F = (int64_t)inter.size(), NB = (int64_t)bnd.size();
  M.face_offsets.assign(1, 0);
  M.face_offsets.reserve(F + NB + 1);
  M.face_points.reserve((F + NB) * 3);
  M.owner.resize(F + NB);
  M.neighbour.resize(F);
  auto emit = [&](int64_t inst) {
    int64_t c = icell[inst];
    int k = (int)(inst - cfo[c]);
    int m = C.face(c, k, ring);
    if (flipped[c]) std::reverse(ring, ring + m);
    M.face_points.insert(M.face_points.end(), ring, ring + m);
    M.face_offsets.push_back((int64_t)M.face_points.size());
  };
  for (int64_t f = 0; f < F; ++f) {
    M.owner[f] = inter[f].o; M.neighbour[f] = inter[f].n; emit(inter[f].inst);
  }
  M.patch_start.assign(patches.size(), 0);
  M.patch_n.assign(patches.size(), 0);
  for (size_t p = 0; p < patches.size(); ++p) M.patch_start[p] = F;
  for (int64_t b = 0; b < NB; ++b) {
    M.owner[F + b] = bnd[b].o; emit(bnd[b].inst);
    M.patch_n[bnd[b].patch]++;
  }
  int64_t s = F;
  for (size_t p = 0; p < patches.size(); ++p) { M.patch_start[p] = s; s += M.patch_n[p]; }
}

// 5-tet split of a hex (VTK corner order) given the parity of corner 0.
// Corner bit pattern (di,dj,dk) per VTK slot.
const int HEX_BITS[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                            {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
int slot_of(int di, int dj, int dk) {
  for (int s = 0; s < 8; ++s)
    if (HEX_BITS[s][0] == di && HEX_BITS[s][1] == dj && HEX_BITS[s][2] == dk) return s;
  return -1;
}
void add_hex_as_5tets(Cells& C, const int32_t* h, int parity0) {
  // even corners: parity0 ^ di ^ dj ^ dk == 0 -> central tet
  int even[4], ne = 0;
  for (int s = 0; s < 8; ++s) {
    int p = parity0 ^ HEX_BITS[s][0] ^ HEX_BITS[s][1] ^ HEX_BITS[s][2];
    if (p == 0) even[ne++] = s;
  }
  int32_t t[4];
  for (int i = 0; i < 4; ++i) t[i] = h[even[i]];
  C.add(0, t, 4);
  for (int s = 0; s < 8; ++s) {
    int p = parity0 ^ HEX_BITS[s][0] ^ HEX_BITS[s][1] ^ HEX_BITS[s][2];
    if (p == 0) continue;
    t[0] = h[s];
    int k = 1;
    for (int d = 0; d < 3; ++d) {
      int b[3] = {HEX_BITS[s][0], HEX_BITS[s][1], HEX_BITS[s][2]};
      b[d] ^= 1;
      t[k++] = h[slot_of(b[0], b[1], b[2])];
    }
    C.add(0, t, 4);
  }
}
// Kuhn / Freudenthal 6-tet split along the 0-6 diagonal.
void add_hex_as_6tets(Cells& C, const int32_t* h) {
  static const int K[6][4] = {{0, 1, 2, 6}, {0, 2, 3, 6}, {0, 3, 7, 6},
                              {0, 7, 4, 6}, {0, 4, 5, 6}, {0, 5, 1, 6}};
  int32_t t[4];
  for (int i = 0; i < 6; ++i) {
    for (int j = 0; j < 4; ++j) t[j] = h[K[i][j]];
    C.add(0, t, 4);
  }
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

typedef struct synth_mesh synth_mesh;

// split: 0 hex, 5 alternating 5-tet, 6 Kuhn 6-tet
// patch_mode: 0 one patch per side (xmin,xmax,ymin,ymax,zmin,zmax, generic)
//             1 cavity (movingWall ymax wall, fixedWalls other x/y sides wall, frontAndBack z empty)
//             2 single patch "boundary" (generic)
//             3 channel slab (inlet xmin, outlet xmax, walls y, frontAndBack z empty)
synth_mesh* synth_box(int nx, int ny, int nz, double lx, double ly, double lz,
                      int split, int patch_mode, double jitter, uint64_t jitter_seed,
                      uint64_t scramble_seed) {
  Mesh* M = new Mesh();
  const int64_t NX = nx + 1, NY = ny + 1, NZ = nz + 1;
  M->points.resize(3 * NX * NY * NZ);
  auto vid = [&](int i, int j, int k) { return (int32_t)((int64_t)k * NX * NY + (int64_t)j * NX + i); };
  const double hx = lx / nx, hy = ly / ny, hz = lz / nz;
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        int64_t v = vid(i, j, k);
        double x = i * hx, y = j * hy, z = k * hz;
        bool interior = i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz;
        if (jitter > 0 && interior) {
          x += jitter * hx * urand(jitter_seed, 3 * (uint64_t)v + 0);
          y += jitter * hy * urand(jitter_seed, 3 * (uint64_t)v + 1);
          z += jitter * hz * urand(jitter_seed, 3 * (uint64_t)v + 2);
        }
        M->points[3 * v + 0] = x; M->points[3 * v + 1] = y; M->points[3 * v + 2] = z;
      }
  Cells C;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int32_t h[8];
        for (int s = 0; s < 8; ++s) h[s] = vid(i + HEX_BITS[s][0], j + HEX_BITS[s][1], k + HEX_BITS[s][2]);
        if (split == 0) C.add(1, h, 8);
        else if (split == 5) add_hex_as_5tets(C, h, (i + j + k) & 1);
        else add_hex_as_6tets(C, h);
      }
  std::vector<Patch> P;
  const double ex = 1e-9 * hx, ey = 1e-9 * hy, ez = 1e-9 * hz;
  Classifier cls;
  if (patch_mode == 1) {
    P = {{"movingWall", 1}, {"fixedWalls", 1}, {"frontAndBack", 2}};
    cls = [=](const double* m, const double*) {
      if (m[2] < ez || m[2] > lz - ez) return 2;
      if (m[1] > ly - ey) return 0;
      return 1;
    };
  } else if (patch_mode == 2) {
    P = {{"boundary", 0}};
    cls = [](const double*, const double*) { return 0; };
  } else if (patch_mode == 3) {
    P = {{"inlet", 0}, {"outlet", 0}, {"walls", 1}, {"frontAndBack", 2}};
    cls = [=](const double* m, const double*) {
      if (m[2] < ez || m[2] > lz - ez) return 3;
      if (m[0] < ex) return 0;
      if (m[0] > lx - ex) return 1;
      return 2;
    };
  } else {
    P = {{"xmin", 0}, {"xmax", 0}, {"ymin", 0}, {"ymax", 0}, {"zmin", 0}, {"zmax", 0}};
    cls = [=](const double* m, const double*) {
      if (m[0] < ex) return 0;
      if (m[0] > lx - ex) return 1;
      if (m[1] < ey) return 2;
      if (m[1] > ly - ey) return 3;
      if (m[2] < ez) return 4;
      return 5;
    };
  }
  build(*M, C, P, cls, scramble_seed);
  M->meta = {lx, ly, lz};
  return (synth_mesh*)M;
}

// O-grid circular pipe along z.
// Central square half-width c = 0.45 R with n x n cells; 4 ring blocks of
// n (tangential) x m_r (radial) cells blending linearly from the square edge
// to the arc; n_z layers over [0, L].  tets != 0: alternating 5-tet split by
// global vertex parity (requires n even).  Patches: inlet (z=0), outlet
// (z=L), wall.
synth_mesh* synth_pipe(int n, int m_r, int n_z, double R, double L, int tets,
                       uint64_t scramble_seed) {
  Mesh* M = new Mesh();
  if (tets && (n % 2)) { M->error = "pipe 5-tet split needs even n"; return (synth_mesh*)M; }
  const double c = 0.45 * R;
  const int64_t nc = (int64_t)(n + 1) * (n + 1);
  const int64_t nl = nc + 4LL * n * m_r;  // vertices per layer
  M->points.resize(3 * nl * (n_z + 1));
  auto central = [&](int i, int j) { return (int64_t)j * (n + 1) + i; };
  // side point of block q at tangential index t (counter-clockwise)
  auto side = [&](int q, int t) -> int64_t {
    switch (q) {
      case 0: return central(n, t);
      case 1: return central(n - t, n);
      case 2: return central(0, n - t);
      default: return central(t, 0);
    }
  };
  auto ring = [&](int q, int r, int t) -> int64_t {
    if (r == 0) return side(q, t);
    if (t == n) { q = (q + 1) & 3; t = 0; }
    return nc + ((int64_t)q * m_r + (r - 1)) * n + t;
  };
  const double PI = 3.14159265358979323846;
  for (int k = 0; k <= n_z; ++k) {
    double z = L * k / n_z;
    double* P = &M->points[3 * (int64_t)k * nl];
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i) {
        int64_t v = central(i, j);
        P[3 * v] = -c + 2 * c * i / n; P[3 * v + 1] = -c + 2 * c * j / n; P[3 * v + 2] = z;
      }
    for (int q = 0; q < 4; ++q)
      for (int r = 1; r <= m_r; ++r)
        for (int t = 0; t < n; ++t) {
          int64_t v = ring(q, r, t), s = side(q, t);
          double th = -PI / 4 + PI / 2 * q + (PI / 2) * t / n;
          double ox = R * std::cos(th), oy = R * std::sin(th);
          double a = (double)r / m_r;
          P[3 * v] = P[3 * s] + a * (ox - P[3 * s]);
          P[3 * v + 1] = P[3 * s + 1] + a * (oy - P[3 * s + 1]);
          P[3 * v + 2] = z;
        }
  }
  Cells C;
  auto emit_hex = [&](const int64_t* q4, int k, int par) {
    int32_t h[8];
    // q4: corners (0,0),(1,0),(1,1),(0,1) of the layer quad
    for (int s = 0; s < 4; ++s) {
      h[s] = (int32_t)(q4[s] + (int64_t)k * nl);
      h[s + 4] = (int32_t)(q4[s] + (int64_t)(k + 1) * nl);
    }
    if (tets) add_hex_as_5tets(C, h, par); else C.add(1, h, 8);
  };
  for (int k = 0; k < n_z; ++k) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        int64_t q4[4] = {central(i, j), central(i + 1, j), central(i + 1, j + 1), central(i, j + 1)};
        emit_hex(q4, k, (i + j + k) & 1);
      }
    for (int q = 0; q < 4; ++q)
      for (int r = 0; r < m_r; ++r)
        for (int t = 0; t < n; ++t) {
          // local axes: bit0 = r, bit1 = t  (parity of corner 0 = r + t + k, n even)
          int64_t q4[4] = {ring(q, r, t), ring(q, r + 1, t), ring(q, r + 1, t + 1), ring(q, r, t + 1)};
          emit_hex(q4, k, (r + t + k) & 1);
        }
  }
  std::vector<Patch> P = {{"inlet", 0}, {"outlet", 0}, {"wall", 1}};
  const double ez = 1e-9 * L / n_z;
  Classifier cls = [=](const double* m, const double* nrm) {
    (void)nrm;
    if (m[2] < ez) return 0;
    if (m[2] > L - ez) return 1;
    return 2;
  };
  build(*M, C, P, cls, scramble_seed);
  M->meta = {R, L, (double)n, (double)m_r, (double)n_z};
  return (synth_mesh*)M;
}

// Voxelised H-tree vascular geometry: root tube along
// x of radius r0 and length l0; each generation halves... see Python docs.
// Capsules are given by the caller (segments + radii); voxels whose centre is
// inside the union are kept; each voxel -> 5 tets by global vertex parity.
// Boundary faces on the domain-box planes listed in `outlet_planes` become
// patches: 0 inlet, 1..n_out outlets (by nearest outlet centre), last = wall.
synth_mesh* synth_voxel_tree(int nx, int ny, int nz, double x0, double y0, double z0, double h,
                             const double* seg, const double* rad, int n_seg,
                             const double* ports, int n_ports, double port_tol,
                             int tets, uint64_t scramble_seed) {
  Mesh* M = new Mesh();
  // inside test per voxel centre
  std::vector<uint8_t> in((int64_t)nx * ny * nz, 0);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        double p[3] = {x0 + (i + 0.5) * h, y0 + (j + 0.5) * h, z0 + (k + 0.5) * h};
        bool inside = false;
        for (int s = 0; s < n_seg && !inside; ++s) {
          const double* a = seg + 6 * s;
          const double* b = a + 3;
          double ab[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
          double ap[3] = {p[0] - a[0], p[1] - a[1], p[2] - a[2]};
          double ll = ab[0] * ab[0] + ab[1] * ab[1] + ab[2] * ab[2];
          double t = ll > 0 ? (ap[0] * ab[0] + ap[1] * ab[1] + ap[2] * ab[2]) / ll : 0;
          // rad > 0: capsule (rounded ends); rad < 0: flat-ended cylinder
          if (rad[s] < 0 && (t < 0 || t > 1)) continue;
          t = std::max(0.0, std::min(1.0, t));
          double d[3] = {ap[0] - t * ab[0], ap[1] - t * ab[1], ap[2] - t * ab[2]};
          inside = d[0] * d[0] + d[1] * d[1] + d[2] * d[2] < rad[s] * rad[s];
        }
        in[((int64_t)k * ny + j) * nx + i] = inside;
      }
  // vertices used by kept voxels
  const int64_t NX = nx + 1, NY = ny + 1;
  auto gv = [&](int i, int j, int k) { return ((int64_t)k * NY + j) * NX + i; };
  std::vector<int32_t> vmap((int64_t)NX * NY * (nz + 1), -1);
  int32_t nv = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        if (!in[((int64_t)k * ny + j) * nx + i]) continue;
        for (int s = 0; s < 8; ++s) {
          int64_t g = gv(i + HEX_BITS[s][0], j + HEX_BITS[s][1], k + HEX_BITS[s][2]);
          if (vmap[g] < 0) vmap[g] = nv++;
        }
      }
  M->points.resize(3 * (int64_t)nv);
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        int32_t v = vmap[gv(i, j, k)];
        if (v < 0) continue;
        M->points[3 * (int64_t)v] = x0 + i * h;
        M->points[3 * (int64_t)v + 1] = y0 + j * h;
        M->points[3 * (int64_t)v + 2] = z0 + k * h;
      }
  Cells C;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        if (!in[((int64_t)k * ny + j) * nx + i]) continue;
        int32_t hh[8];
        for (int s = 0; s < 8; ++s) hh[s] = vmap[gv(i + HEX_BITS[s][0], j + HEX_BITS[s][1], k + HEX_BITS[s][2])];
        if (tets) add_hex_as_5tets(C, hh, (i + j + k) & 1); else C.add(1, hh, 8);
      }
  // ports: each (cx, cy, cz, nx, ny, nz): a boundary face whose normal is
  // parallel to the port axis and whose centre lies within port_tol of the
  // port plane and inside the port disc belongs to that port.
  std::vector<Patch> P;
  P.push_back({"inlet", 0});
  for (int p = 1; p < n_ports; ++p) P.push_back({"outlet" + std::to_string(p - 1), 0});
  P.push_back({"wall", 1});
  std::vector<double> pv(ports, ports + 7 * n_ports);
  Classifier cls = [=](const double* m, const double* nrm) {
    double nn = std::sqrt(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
    for (int p = 0; p < n_ports; ++p) {
      const double* q = &pv[7 * p];
      double d[3] = {m[0] - q[0], m[1] - q[1], m[2] - q[2]};
      double along = d[0] * q[3] + d[1] * q[4] + d[2] * q[5];
      double cosang = (nrm[0] * q[3] + nrm[1] * q[4] + nrm[2] * q[5]) / nn;
      double rr = d[0] * d[0] + d[1] * d[1] + d[2] * d[2] - along * along;
      if (std::fabs(along) < port_tol && std::fabs(cosang) > 0.999 && rr < q[6] * q[6]) return p;
    }
    return n_ports;  // wall
  };
  build(*M, C, P, cls, scramble_seed);
  return (synth_mesh*)M;
}

// Extruded polygon slab: polygons (ring offsets/ids into 2-D points, counter-
// clockwise) extruded over [0, dz] with one layer; patches are decided by the
// caller-supplied per-edge tags of boundary edges: tag_of(edge midpoint) is
// evaluated by a simple rule set: boxes [xmin,xmax]x[ymin,ymax] -> patch id.
// front/back faces go to patch `empty_patch`.
synth_mesh* synth_extrude_polygons(const double* pts2, int64_t n_pts, const int64_t* poly_off,
                                   const int32_t* poly_ids, int64_t n_poly, double dz,
                                   const char* const* patch_names, const int* patch_kinds,
                                   int n_patches, const double* rules, int n_rules,
                                   int empty_patch, uint64_t scramble_seed) {
  Mesh* M = new Mesh();
  M->points.resize(6 * n_pts);
  for (int64_t i = 0; i < n_pts; ++i) {
    M->points[3 * i] = pts2[2 * i]; M->points[3 * i + 1] = pts2[2 * i + 1]; M->points[3 * i + 2] = 0;
    M->points[3 * (n_pts + i)] = pts2[2 * i];
    M->points[3 * (n_pts + i) + 1] = pts2[2 * i + 1];
    M->points[3 * (n_pts + i) + 2] = dz;
  }
  Cells C;
  std::vector<int32_t> buf;
  for (int64_t p = 0; p < n_poly; ++p) {
    int m = (int)(poly_off[p + 1] - poly_off[p]);
    buf.resize(2 * m);
    for (int i = 0; i < m; ++i) {
      buf[i] = poly_ids[poly_off[p] + i];
      buf[m + i] = (int32_t)(poly_ids[poly_off[p] + i] + n_pts);
    }
    C.add(2, buf.data(), 2 * m);
  }
  std::vector<Patch> P;
  for (int i = 0; i < n_patches; ++i) P.push_back({patch_names[i], patch_kinds[i]});
  std::vector<double> rv(rules, rules + 5 * n_rules);
  const double ez = 1e-9 * dz;
  Classifier cls = [=](const double* m, const double*) {
    if (m[2] < ez || m[2] > dz - ez) return empty_patch;
    for (int r = 0; r < n_rules; ++r) {
      const double* q = &rv[5 * r];
      if (m[0] >= q[0] && m[0] <= q[1] && m[1] >= q[2] && m[1] <= q[3]) return (int)q[4];
    }
    return -1;
  };
  build(*M, C, P, cls, scramble_seed);
  M->meta = {dz};
  return (synth_mesh*)M;
}

const char* synth_error(const synth_mesh* m) {
  const Mesh* M = (const Mesh*)m;
  return M->error.empty() ? nullptr : M->error.c_str();
}
void synth_sizes(const synth_mesh* m, int64_t* out /*6*/) {
  const Mesh* M = (const Mesh*)m;
  out[0] = (int64_t)M->points.size() / 3;
  out[1] = (int64_t)M->owner.size();
  out[2] = (int64_t)M->neighbour.size();
  out[3] = (int64_t)M->face_points.size();
  out[4] = (int64_t)M->patches.size();
  out[5] = M->n_cells;
}
void synth_copy(const synth_mesh* m, double* points, int64_t* face_offsets, int32_t* face_points,
                int32_t* owner, int32_t* neighbour, int64_t* patch_start, int64_t* patch_n,
                int32_t* patch_kind) {
  const Mesh* M = (const Mesh*)m;
  std::memcpy(points, M->points.data(), M->points.size() * sizeof(double));
  std::memcpy(face_offsets, M->face_offsets.data(), M->face_offsets.size() * sizeof(int64_t));
  std::memcpy(face_points, M->face_points.data(), M->face_points.size() * sizeof(int32_t));
  std::memcpy(owner, M->owner.data(), M->owner.size() * sizeof(int32_t));
  std::memcpy(neighbour, M->neighbour.data(), M->neighbour.size() * sizeof(int32_t));
  for (size_t p = 0; p < M->patches.size(); ++p) {
    patch_start[p] = M->patch_start[p]; patch_n[p] = M->patch_n[p]; patch_kind[p] = M->patches[p].kind;
  }
}
const char* synth_patch_name(const synth_mesh* m, int p) { return ((const Mesh*)m)->patches[p].name.c_str(); }
void synth_free(synth_mesh* m) { delete (Mesh*)m; }

}  // extern "C"
