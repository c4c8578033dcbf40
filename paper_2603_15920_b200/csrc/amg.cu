// amg.cu — aggregation AMG preconditioner for the pressure PCG (SURVEY.md
// §8(f) NEXT-2: "ILU ... and/or aggregation AMG for the pressure").
//
// Jacobi-PCG on the pressure Laplacian needs O(10^3) iterations on the 50M
// cell pipe (iterations grow with the longest mesh dimension, SURVEY §7 hard
// part 2); the paper's own choice, ILU, is sequential on a GPU.  A
// plain-aggregation V-cycle keeps everything data-parallel and deterministic:
//
//  * hierarchy (host, once per mesh, topology only): greedy aggregation of
//    the owned rows in RCM order (root + its unaggregated neighbours; leftovers
//    join a neighbouring aggregate; isolated rows become singletons), until
//    <= 256 rows (DFVM_AMG_COARSE).  Coarse levels are rank-local (couplings to ghost rows are
//    dropped: the coarse operator is the Galerkin product of the owned block,
//    still SPD).
//  * values (device, whenever the pressure matrix changes): Galerkin
//    A_c = P^T A P with piecewise-constant P, as fixed-order gather sums over
//    precomputed contribution lists (no atomics); l1-Jacobi diagonals
//    d1_i = a_ii + sum_j |a_ij|.
//  * cycle (defaults measured on the C5 pipe): l1-Jacobi
//    pre-smoothing from zero x0 = D1^-1 b, residual, restriction (sum over
//    the aggregate's members), coarse correction scaled by omega = 1.95,
//    prolongation x = x0 + omega x_c[agg], l1-Jacobi post-smoothing (the
//    adjoint of the pre-smoother); a W-cycle (two coarse visits, the second
//    on the residual of the first) on levels <= 4 and a V-cycle below;
//    coarsening stops at <= 256 rows (fp64 hierarchy) or <= 4000 rows (fp32:
//    amg32 and the f32 solver; C5 stops at its 3 330-row level 4), never
//    below 32, and the coarsest level is solved exactly with its dense
//    inverse, refreshed once per step: one-block shared-memory symmetric
//    sweep (fp32 <= 340 rows) or one-block Gauss-Jordan (<= 512 rows), the
//    blocked symmetric sweep in global memory (fp32, <= 4096 rows) or a
//    multi-launch Gauss-Jordan (fp64, <= 4096); a coarsest level beyond the
//    direct bound (coarsening stalled) gets `sweeps` l1-Jacobi sweeps (one
//    block up to 2048 rows, multi-block above).  Adjoint smoothers, a symmetric coarse solve and the W-cycle's
//    2B - BAB keep M^-1 SPD, so CG stays CG.  The converged pressure is
//    preconditioner independent (A-14).
//  * precision: the hierarchy's type P is the solver's T ("amg"), or fp32
//    under an fp64 solver ("amg32": matrix copies, smoother and every level
//    vector in fp32; the PCG itself — residual, dots, x, p — stays fp64).
//    Level 0 reads the PCG residual in T and writes z = M^-1 r in T.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <vector>

#include <cuda_bf16.h>

#include "amg.h"
#include "dev.cuh"
#include "prof.h"
#include "krylov.cuh"

namespace dfvm {

dfvm_status halo_exchange_p(dfvm_mesh* m, void* data, int nc, bool f64, cudaStream_t s);
dfvm_status halo_exchange_lists(dfvm_mesh* m, HaloLists& L, void* data, int nc, bool f64, cudaStream_t s);
dfvm_status allgather_f64(dfvm_mesh* m, const double* local, double* gathered, int n, cudaStream_t s);
bool comm_is_local(const dfvm_comm* c);

constexpr int kCoarseMax = 2048;     // shared-memory capacity of the one-block coarse solve
constexpr int kDirectMax = 512;      // largest coarsest level inverted by one block
constexpr int kDirectBig = 4096;     // largest coarsest level inverted at all (multi-launch Gauss-Jordan above kDirectMax)
constexpr int kMaxLevels = 16;
constexpr int kCsrChunk = 128;       // entries per warp chunk of the CSR-stream coarse kernels (4 per lane)

// Tunables (defaults chosen from B200 measurements on the C5 pipe, DESIGN.md
// §6); overridable through the environment for experiments:
//   DFVM_AMG_COARSE  coarsest-level size bound (rows)   default 256 (fp32: 4000)
//   DFVM_AMG_SWEEPS  l1-Jacobi sweeps of the coarsest solve       default 32
//   DFVM_AMG_CYCLE   'V' or 'W'                                   default W
//   DFVM_AMG_WMAX    deepest level visited twice by the W-cycle   default 4
//                    (deeper levels use V-cycles: the W launch count
//                    doubles per level, and deep levels are launch-bound)
//   DFVM_AMG_OMEGA   coarse-correction scale (symmetric over-correction,
//                    < 2 keeps M SPD with adjoint smoothers)   default 1.95
//   DFVM_AMG_PERM    1: coarse-level SELL storage sorted by row length
//                    within windows of 256 slots (SELL-32-sigma: rows keep
//                    their numbers, the hierarchy is unchanged, padding
//                    shrinks); 0: natural order                  default 0
//                    (C5 round 2: padding 8.4 % on level 1, yet 347.2 ms/step
//                    against 343.1 ms in natural order — the coarse
//                    kernels are bound by their gathers, and the permuted
//                    own-row accesses cost more than the padding saved;
//                    profiles/r02_amg_sweep2_c5.jsonl); results differ from
//                    natural order at round-off (2e-10 on a 38k-cell pipe),
//                    within the parity bound
//                    (round 1 renumbered the aggregates themselves by
//                    length instead: that changed the next aggregation
//                    and cost 0.5 PCG iterations per solve — removed)
//   (round 2 measured and removed a one-cluster "tail" kernel that walked
//   all levels below a size bound with cluster barriers: 0.67 ms per
//   level-3 visit on C5 against ~0.2 ms launched, and slower even from the
//   3,330-row level 4 — 16 SMs cannot hide the gather latency; profiles/
//   r02_bench_c5_tail_variants.txt)
//   DFVM_AMG_FUSED_FROM  coarse levels l >= this run the fused pre-smooth +
//                    residual / prolongation + post-smooth kernels; levels
//                    1 .. this-1 the unfused ones (pre, resid | prolong,
//                    smooth: fewer gathers per entry, one more vector pass;
//                    bitwise identical results)                  default 3
//                    (C5 amg32: 340.3 ms/step against 349.6 ms with every
//                    coarse level fused, 347.2 with level 1 unfused;
//                    profiles/r02_amg_sweep_c5.jsonl)
//   DFVM_AMG_AGGLOM  several ranks: the first coarse level whose rows, summed
//                    over the ranks, are <= this is agglomerated into one
//                    global level replicated on every rank (with the serial
//                    hierarchy below it); the levels above are distributed
//                                                               default 100000
//   DFVM_AMG_DIRECT  coarsest levels with <= this many rows (fp32 default 4096) are solved
//                    exactly with a dense inverse (Gauss-Jordan once per
//                    matrix update, one block), larger ones with
//                    DFVM_AMG_SWEEPS l1-Jacobi sweeps (0: always sweeps)  default 512
struct AmgParams {
  int coarse = 256, sweeps = 32, wmax = 4, direct = kDirectMax, perm = 0;
  int fused_from = 3;   // coarse levels >= this use the fused pre_resid / prolong_smooth kernels
  int agglom = 100000;  // several ranks: agglomerate the first coarse level with <= this many rows in total
  int renum = 0;        // 1: aggregates renumbered by their first member (locality order)
  // 1: coarse levels with one thread per row use the CSR-stream kernels.
  // Default 0 (SELL): measured on C5 round 2 at 334.4 / 336.6 ms/step with
  // CSR-stream against 330.0 / 330.9 (profiles/r02_sweep_r2i_csr.jsonl) —
  // the chunk's serial per-row sums over shared memory and the idle lanes
  // of short chunks cost more than the coalesced, padding-free loads saved
  int csr = 0;
  bool wcycle = true;
  double omega = 1.95;  // C5 amg32 (round 2): 344.0 ms, 11.33 it/solve (1.9: 349.6 ms, 11.58; 1.8: 360.2 ms, 12.17)
  bool env_coarse = false, env_direct = false;
  // fp32 hierarchies (amg32): coarsen only down to <= 4000 rows and solve
  // that level exactly with the blocked dense inverse (C5: the 3 330-row
  // level, no 144-row level below it) — measured on C5 round 2 at 313.4 /
  // 313.4 ms/step and 10.3 PCG iterations per solve, against 324.5 / 327.3
  // ms/step and 11.3 with the W-cycle to a 144-row exact level
  // (profiles/r02_sweep_r2q_lvl4.jsonl); env overrides win
  void fp32_defaults() {
    if (!env_coarse) coarse = 4000;
    if (!env_direct) direct = kDirectBig;
  }
  AmgParams() {
    if (const char* e = getenv("DFVM_AMG_DIRECT")) { direct = std::max(0, std::min(kDirectBig, atoi(e))); env_direct = true; }
    if (const char* e = getenv("DFVM_AMG_PERM")) perm = atoi(e);
    if (const char* e = getenv("DFVM_AMG_OMEGA")) omega = atof(e);
    if (const char* e = getenv("DFVM_AMG_COARSE")) { coarse = std::max(16, std::min(kDirectBig, atoi(e))); env_coarse = true; }
    if (const char* e = getenv("DFVM_AMG_SWEEPS")) sweeps = std::max(1, atoi(e));
    if (const char* e = getenv("DFVM_AMG_CYCLE")) wcycle = (e[0] == 'W' || e[0] == 'w');
    if (const char* e = getenv("DFVM_AMG_WMAX")) wmax = std::max(0, atoi(e));
    if (const char* e = getenv("DFVM_AMG_FUSED_FROM")) fused_from = std::max(1, atoi(e));
    if (const char* e = getenv("DFVM_AMG_AGGLOM")) agglom = std::max(32, atoi(e));
    if (const char* e = getenv("DFVM_AMG_RENUM")) renum = atoi(e);
    if (const char* e = getenv("DFVM_AMG_CSR")) csr = atoi(e);
  }
};

// A level's matrix in SELL-32 storage.  Slot q of slice q / 32 (lane q % 32)
// holds row perm[q] (perm == NULL: row q).  The coarse levels sort the rows of
// each window of 256 slots by length (SELL-32-sigma storage; the rows keep
// their numbers, so the hierarchy and every result are unchanged): much
// less padding than natural order on aggregation levels.
struct SellView {
  const int* ms_ptr;
  const int* ms_len;
  const int* mnb;
  const int* perm;
  const unsigned char* rlen;   // per-slot row length (coarse levels), NULL: the slice length
};
// ------------------------------------------------------------ host setup
namespace {

struct HostLevel {
  int n = 0;
  // SELL-32 of this level's matrix (level 0: the mesh's matrix layout)
  std::vector<int> ms_ptr, ms_len, mnb;
  std::vector<int> perm, slot_of;   // SELL slot -> row and back (empty: identity)
  // CSR view of the real entries: (col, SELL position), owned cols only
  std::vector<int> rp, col, pos;
  // several ranks: ghost rows [n, n + ng) (owner rank, owner-local index),
  // the halo lists, and the CSR of the entries with ghost columns
  int ng = 0;
  std::vector<int> ghost_peer, ghost_key;
  HaloLists halo;
  std::vector<int> grp, gcol, gpos;
  int slot(int r) const { return slot_of.empty() ? r : slot_of[r]; }
};

// entries of owned rows with ghost columns (c >= n)
void sell_to_ghost_csr(HostLevel& L) {
  const int n = L.n;
  L.grp.assign(n + 1, 0);
  L.gcol.clear();
  L.gpos.clear();
  for (int r = 0; r < n; ++r) {
    const int q = L.slot(r), s = q / 32, lane = q % 32;
    for (int j = 0; j < L.ms_len[s]; ++j) {
      const int p = L.ms_ptr[s] + 32 * j + lane;
      const int c = L.mnb[p];
      if (c >= n) { L.gcol.push_back(c); L.gpos.push_back(p); }
    }
    L.grp[r + 1] = (int)L.gcol.size();
  }
}

void sell_to_csr(HostLevel& L, int n_owned_cols) {
  const int n = L.n;
  L.rp.assign(n + 1, 0);
  for (int r = 0; r < n; ++r) {
    const int q = L.slot(r), s = q / 32, lane = q % 32;
    for (int j = 0; j < L.ms_len[s]; ++j) {
      const int c = L.mnb[L.ms_ptr[s] + 32 * j + lane];
      if (c != r && c < n_owned_cols) L.rp[r + 1]++;
    }
  }
  for (int r = 0; r < n; ++r) L.rp[r + 1] += L.rp[r];
  L.col.assign(L.rp[n], 0);
  L.pos.assign(L.rp[n], 0);
  for (int r = 0; r < n; ++r) {
    const int q = L.slot(r), s = q / 32, lane = q % 32;
    int k = L.rp[r];
    for (int j = 0; j < L.ms_len[s]; ++j) {
      const int p = L.ms_ptr[s] + 32 * j + lane;
      const int c = L.mnb[p];
      if (c != r && c < n_owned_cols) { L.col[k] = c; L.pos[k] = p; ++k; }
    }
  }
}

std::vector<int> aggregate(const HostLevel& L, int& nagg) {
  const int n = L.n;
  std::vector<int> agg(n, -1);
  nagg = 0;
  for (int i = 0; i < n; ++i) {          // pass 1: roots with all neighbours free
    if (agg[i] >= 0) continue;
    bool free_nb = true;
    for (int k = L.rp[i]; k < L.rp[i + 1] && free_nb; ++k) free_nb = agg[L.col[k]] < 0;
    if (!free_nb) continue;
    agg[i] = nagg;
    for (int k = L.rp[i]; k < L.rp[i + 1]; ++k) agg[L.col[k]] = nagg;
    ++nagg;
  }
  std::vector<int> a1 = agg;             // pass 2: join a pass-1 neighbour aggregate
  for (int i = 0; i < n; ++i) {
    if (a1[i] >= 0) continue;
    for (int k = L.rp[i]; k < L.rp[i + 1]; ++k)
      if (a1[L.col[k]] >= 0) { agg[i] = a1[L.col[k]]; break; }
  }
  for (int i = 0; i < n; ++i)            // pass 3: leftovers with their free neighbours
    if (agg[i] < 0) {
      agg[i] = nagg;
      for (int k = L.rp[i]; k < L.rp[i + 1]; ++k)
        if (agg[L.col[k]] < 0) agg[L.col[k]] = nagg;
      ++nagg;
    }
  return agg;
}

// Locality order of the aggregates: renumber by their smallest member row, so
// the coarse rows follow the fine (RCM) order — pass-3 leftovers, created
// last, land next to their members instead of at the end (coarse gathers
// stay local).  A monotone map of the fine order: no change to which rows
// are aggregated, but the next level's greedy aggregation sees a different
// row order.
void renumber_by_first_member(std::vector<int>& agg, int nc) {
  std::vector<int> first(nc, INT32_MAX);
  for (int i = 0; i < (int)agg.size(); ++i) first[agg[i]] = std::min(first[agg[i]], i);
  std::vector<int> order(nc);
  for (int I = 0; I < nc; ++I) order[I] = I;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return first[a] < first[b]; });
  std::vector<int> newid(nc);
  for (int k = 0; k < nc; ++k) newid[order[k]] = k;
  for (auto& a : agg) a = newid[a];
}

}  // namespace

template <class P>
struct AmgLevelDev {
  int n = 0, n_slices = 0;
  int64_t n_sell = 0;        // SELL slots (incl. padding)
  int64_t nnz = 0;           // real off-diagonal entries (algorithmic bytes)
  const int *ms_ptr = nullptr, *ms_len = nullptr, *mnb = nullptr;
  const int* perm = nullptr;  // SELL slot -> row (coarse levels, SELL-32-sigma storage), NULL: identity
  const unsigned char* rlen = nullptr;   // per-slot row length (serial coarse levels), NULL: slice length
  SellView sv() const { return SellView{ms_ptr, ms_len, mnb, perm, use_rlen ? rlen : nullptr}; }
  bool use_rlen = false;
  const P* coef = nullptr;   // level 0: the solver's pcoef (P == T) or coef_own (fp32 copy)
  const P* diag = nullptr;   // level 0: the solver's pdiag (P == T) or diag_own
  P* coef_own = nullptr;
  P* diag_own = nullptr;
  P* il1 = nullptr;
  // Galerkin maps of this (coarse) level from the finer level
  int *gal_ptr = nullptr, *gal_idx = nullptr;     // per coarse SELL position
  int *dg_ptr = nullptr, *dg_idx = nullptr;       // per coarse row: internal fine positions
  int *mem_ptr = nullptr, *mem = nullptr;         // per coarse row: fine member rows
  int* agg = nullptr;                             // on the FINE level: fine row -> coarse row
  P *x = nullptr, *b = nullptr, *r = nullptr, *t = nullptr;
  P *e = nullptr, *r2 = nullptr;                  // W-cycle: second-visit solution / rhs
  int n_cells = 0;                                // owned + ghost rows (several ranks)
  // CSR-stream copy of the matrix (serial coarse levels with one thread per
  // row): warp chunks of whole rows with <= kCsrChunk entries (c_ptr: first
  // row per chunk), the real entries of each row in SELL order (c_rp, c_col),
  // their SELL positions (c_pos: c_coef is gathered from coef per update)
  int n_chunk = 0;
  int64_t nnz_csr = 0;
  int *c_ptr = nullptr, *c_rp = nullptr, *c_col = nullptr, *c_pos = nullptr;
  P* c_coef = nullptr;
  int G = 1;                                      // lanes per row of this level's matrix kernels
  int Gr = 1;                                     // lanes per row of the restriction INTO this level
};

// hierarchy stored and cycled in type P
template <class P>
struct AmgH {
  dfvm_mesh* m = nullptr;
  int nlev = 0;
  AmgParams prm;
  Prof* prof = nullptr;             // per-kernel profile of the caller (may be null)
  AmgLevelDev<P> L[kMaxLevels];
  P* ainv = nullptr;                // dense inverse of the coarsest matrix (row-major n x ainv_ld), or NULL
  int ainv_ld = 0;                  // its row stride (n; rounded up to 8 for the blocked fp32 path)
  int64_t inv_refreshes = 0;        // blocked inverse: updates seen (DFVM_AMG_INV_EVERY lags the refresh)
  P* gj_buf = nullptr;              // pivot row / column of the multi-launch Gauss-Jordan
  __nv_bfloat16* ainv16 = nullptr;  // DFVM_AMG_INV16=1: bf16 copy of a large fp32 inverse (half the mat-vec bytes)
  // several ranks: levels 0..ld are distributed (owned aggregates of owned
  // rows, ghost aggregates of the neighbours, a halo per level); level ld+1
  // is the AGGLOMERATION of every rank's level-ld rows into one global
  // level, replicated on every rank together with the serial hierarchy
  // below it (values all-gathered at each update, right-hand sides at each
  // visit)
  bool dist = false;
  HaloLists halos[kMaxLevels];
  int ld = -1;                      // last distributed level (-1: single rank)
  bool agglom = false;
  // depth of level l in the single-rank sense (the agglomerated level is the
  // replicated copy of level ld, so the W-cycle depth rule skips it)
  int depth(int l) const { return (agglom && l > ld) ? l - 1 : l; }
  int Vmax = 0, Nmax = 0;           // padded per-rank value / row counts of the exchanges
  int Vloc = 0;                     // this rank's values
  int* d_pk = nullptr;              // canonical value k of this rank's level-ld rows: >= 0 coef position, < 0 diag -1-i
  int *d_gmap = nullptr, *d_gdmap = nullptr;   // G0 SELL position / row -> index into the gathered values
  int *d_cnt = nullptr, *d_off = nullptr;      // per rank: level-ld rows and their global offset
  int goff = 0;                     // this rank's offset in G0
  double *d_vals = nullptr, *d_vals_all = nullptr, *d_rhs = nullptr, *d_rhs_all = nullptr;
  std::vector<void*> allocs;
  int64_t bytes = 0;
  ~AmgH() {
    if (gj_buf) dev_free(gj_buf, nullptr);
    if (ainv16) dev_free(ainv16, nullptr);
    for (void* p : allocs) dev_free(p, nullptr);
    for (auto& h : halos) { dev_free(h.d_send, nullptr); dev_free(h.d_send_idx, nullptr); }
  }
  // legacy-stream allocations / uploads; amg_create synchronises once after
  // the build, before the caller's stream uses any of them
  template <class U>
  dfvm_status up(U** d, const std::vector<U>& h) {
    if (dfvm_status st = dev_alloc_n(d, h.size(), nullptr, false)) return st;
    if (!h.empty()) DFVM_CUDA(cudaMemcpy(*d, h.data(), h.size() * sizeof(U), cudaMemcpyHostToDevice));
    allocs.push_back((void*)*d);
    bytes += (int64_t)(std::max<size_t>(h.size(), 1) * sizeof(U));
    return DFVM_OK;
  }
  template <class U>
  dfvm_status zalloc(U** d, size_t n) {
    if (dfvm_status st = dev_alloc_n(d, n, nullptr, true)) return st;
    allocs.push_back((void*)*d);
    bytes += (int64_t)(std::max<size_t>(n, 1) * sizeof(U));
    return DFVM_OK;
  }
};

// the solver-facing handle: exactly one of the two hierarchies is built
template <class T>
struct Amg {
  AmgH<T>* same = nullptr;       // "amg": hierarchy in the solver's precision
  AmgH<float>* lo = nullptr;     // "amg32": fp32 hierarchy under an fp64 solver
  ~Amg() { delete same; delete lo; }
};

// Serial coarsening from host level H[lev] (device level A->L[lev] set up):
// aggregation, Galerkin maps, SELL layout, upload, until <= prm.coarse rows
// (or a stall / a level under 32 rows).  lev returns the coarsest index.
template <class P>
static dfvm_status coarsen_serial(AmgH<P>* A, std::vector<HostLevel>& H, int& lev) {
  dfvm_status st;
  // (a level 0 above 256 rows is always coarsened once, so a mesh smaller
  // than the fp32 bound still gets a two-level cycle with an exact coarse
  // solve — C1's 400 cells: 7 PCG iterations against 11.6 with 32 l1-Jacobi
  // sweeps on the single level)
  while ((H[lev].n > A->prm.coarse || (lev == 0 && H[lev].n > 256)) && lev + 1 < kMaxLevels) {
    const HostLevel& F = H[lev];
    int nc = 0;
    std::vector<int> agg = aggregate(F, nc);
    if (A->prm.renum) renumber_by_first_member(agg, nc);
    if (nc >= F.n * 0.85) break;           // coarsening stalled
    // no degenerate tiny level: C5 with DFVM_AMG_COARSE=128 grew an 8-row
    // level under the 144-row one and the PCG needed 1702 iterations per
    // solve; the current level becomes the coarsest (solved exactly)
    if (nc < 32) break;
    // members
    std::vector<int> mem_ptr(nc + 1, 0), mem(F.n);
    for (int i = 0; i < F.n; ++i) mem_ptr[agg[i] + 1]++;
    for (int I = 0; I < nc; ++I) mem_ptr[I + 1] += mem_ptr[I];
    {
      std::vector<int> p(mem_ptr.begin(), mem_ptr.end() - 1);
      for (int i = 0; i < F.n; ++i) mem[p[agg[i]]++] = i;
    }
    // coarse rows: (J, fine position) pairs, sorted; internal -> diag list
    HostLevel C;
    C.n = nc;
    std::vector<int> crow_ptr(nc + 1, 0), ccol, dg_ptr(nc + 1, 0), dg_idx;
    std::vector<std::vector<int>> gal_lists;   // per coarse CSR entry
    std::vector<std::pair<int, int>> buf;
    for (int I = 0; I < nc; ++I) {
      buf.clear();
      for (int q = mem_ptr[I]; q < mem_ptr[I + 1]; ++q) {
        const int i = mem[q];
        for (int k = F.rp[i]; k < F.rp[i + 1]; ++k) buf.push_back({agg[F.col[k]], F.pos[k]});
      }
      std::sort(buf.begin(), buf.end());
      for (size_t k = 0; k < buf.size();) {
        const int J = buf[k].first;
        size_t e = k;
        while (e < buf.size() && buf[e].first == J) ++e;
        if (J == I) {
          for (size_t u = k; u < e; ++u) dg_idx.push_back(buf[u].second);
        } else {
          ccol.push_back(J);
          gal_lists.emplace_back();
          for (size_t u = k; u < e; ++u) gal_lists.back().push_back(buf[u].second);
        }
        k = e;
      }
      crow_ptr[I + 1] = (int)ccol.size();
      dg_ptr[I + 1] = (int)dg_idx.size();
    }
    // coarse SELL-32 layout; with prm.perm the rows of each window of 256
    // slots are stored by decreasing length (SELL-32-sigma storage: the rows
    // keep their numbers, so aggregation below and every result are
    // unchanged, only the padding shrinks)
    const int S = (nc + 31) / 32;
    if (A->prm.perm) {
      C.perm.resize(nc);
      C.slot_of.resize(nc);
      for (int I = 0; I < nc; ++I) C.perm[I] = I;
      constexpr int kSigma = 256;
      for (int w0 = 0; w0 < nc; w0 += kSigma) {
        const int w1 = std::min(nc, w0 + kSigma);
        std::stable_sort(C.perm.begin() + w0, C.perm.begin() + w1, [&](int a, int b) {
          return crow_ptr[a + 1] - crow_ptr[a] > crow_ptr[b + 1] - crow_ptr[b];
        });
      }
      for (int q = 0; q < nc; ++q) C.slot_of[C.perm[q]] = q;
    }
    auto row_at = [&](int q) { return C.perm.empty() ? q : C.perm[q]; };
    C.ms_ptr.assign(S + 1, 0);
    C.ms_len.assign(S, 0);
    for (int s = 0; s < S; ++s) {
      int w = 0;
      for (int q = s * 32; q < std::min(nc, s * 32 + 32); ++q) {
        const int I = row_at(q);
        w = std::max(w, crow_ptr[I + 1] - crow_ptr[I]);
      }
      C.ms_len[s] = w;
      C.ms_ptr[s + 1] = C.ms_ptr[s] + 32 * w;
    }
    C.mnb.assign(C.ms_ptr[S], 0);
    std::vector<int> gal_ptr(C.ms_ptr[S] + 1, 0), gal_idx;
    std::vector<int> slot_entry(C.ms_ptr[S], -1), epos(ccol.size(), -1);
    for (int I = 0; I < nc; ++I) {
      const int q = C.slot(I), s = q / 32, lane = q % 32;
      for (int j = 0; j < C.ms_len[s]; ++j) {
        const int p = C.ms_ptr[s] + 32 * j + lane;
        const int e = crow_ptr[I] + j;
        if (e < crow_ptr[I + 1]) { C.mnb[p] = ccol[e]; slot_entry[p] = e; epos[e] = p; }
        else C.mnb[p] = I;   // padding: self, coefficient 0
      }
    }
    for (int p = 0; p < C.ms_ptr[S]; ++p) {
      if (slot_entry[p] >= 0) for (int f : gal_lists[slot_entry[p]]) gal_idx.push_back(f);
      gal_ptr[p + 1] = (int)gal_idx.size();
    }
    sell_to_csr(C, nc);
    // upload
    AmgLevelDev<P>& D = A->L[lev + 1];
    D.n = nc; D.n_slices = S; D.n_sell = C.ms_ptr[S];
    D.nnz = (int64_t)ccol.size();
    int *p0, *p1, *p2, *p3 = nullptr;
    // perm == 2 (relabel): the coarse rows are RENUMBERED by their SELL slot
    // on the device (row q lives in slot q, no indirection): columns, member
    // lists, diagonal lists and the fine level's aggregate map are uploaded
    // in slot order (the fine rows in the fine level's slot order).  The host
    // levels keep the original numbering, so the aggregation below — hence
    // the hierarchy and every per-row sum order — is that of natural order;
    // only storage padding (and own-row contiguity) changes.
    const bool relabel = A->prm.perm == 2 && !C.perm.empty();
    std::vector<int> mnb_u, mem_ptr_u, mem_u, dg_ptr_u, dg_idx_u, agg_u;
    const std::vector<int>* up_mnb = &C.mnb;
    const std::vector<int>*up_mp = &mem_ptr, *up_mem = &mem, *up_dp = &dg_ptr, *up_di = &dg_idx, *up_agg = &agg;
    if (relabel) {
      const std::vector<int>& pf = F.slot_of;   // the fine level's relabelling (level 0: none)
      auto PF = [&](int i) { return pf.empty() ? i : pf[i]; };
      mnb_u.resize(C.mnb.size());
      for (size_t k = 0; k < C.mnb.size(); ++k) mnb_u[k] = C.slot_of[C.mnb[k]];
      mem_ptr_u.assign(nc + 1, 0); dg_ptr_u.assign(nc + 1, 0);
      mem_u.reserve(mem.size()); dg_idx_u.reserve(dg_idx.size());
      for (int q = 0; q < nc; ++q) {
        const int I = C.perm[q];
        for (int k = mem_ptr[I]; k < mem_ptr[I + 1]; ++k) mem_u.push_back(PF(mem[k]));
        for (int k = dg_ptr[I]; k < dg_ptr[I + 1]; ++k) dg_idx_u.push_back(dg_idx[k]);
        mem_ptr_u[q + 1] = (int)mem_u.size();
        dg_ptr_u[q + 1] = (int)dg_idx_u.size();
      }
      agg_u.resize(agg.size());
      for (int i = 0; i < (int)agg.size(); ++i) agg_u[PF(i)] = C.slot_of[agg[i]];
      up_mnb = &mnb_u; up_mp = &mem_ptr_u; up_mem = &mem_u; up_dp = &dg_ptr_u; up_di = &dg_idx_u; up_agg = &agg_u;
    } else if (!C.perm.empty() && (st = A->up(&p3, C.perm))) {
      return st;
    }
    D.perm = p3;
    if ((st = A->up(&p0, C.ms_ptr)) || (st = A->up(&p1, C.ms_len)) || (st = A->up(&p2, *up_mnb)) ||
        (st = A->up(&D.gal_ptr, gal_ptr)) || (st = A->up(&D.gal_idx, gal_idx)) || (st = A->up(&D.dg_ptr, *up_dp)) ||
        (st = A->up(&D.dg_idx, *up_di)) || (st = A->up(&D.mem_ptr, *up_mp)) || (st = A->up(&D.mem, *up_mem)) ||
        (st = A->up(&A->L[lev].agg, *up_agg)) || (st = A->zalloc(&D.coef_own, (size_t)D.n_sell)) ||
        (st = A->zalloc(&D.diag_own, nc)) || (st = A->zalloc(&D.il1, nc)) || (st = A->zalloc(&D.x, nc)) ||
        (st = A->zalloc(&D.b, nc)) || (st = A->zalloc(&D.r, nc)) || (st = A->zalloc(&D.t, nc)) ||
        (st = A->zalloc(&D.e, nc)) || (st = A->zalloc(&D.r2, nc)))
      return st;
    D.ms_ptr = p0; D.ms_len = p1; D.mnb = p2;
    D.coef = D.coef_own; D.diag = D.diag_own;
    {
      // per-slot row lengths: DFVM_AMG_RLEN=1 stops each lane at its own
      // row (padding neither loaded nor gathered).  Default off: measured on
      // C5 round 2 at 335.1 / 337.7 ms/step against 334.6 / 333.6 with every
      // lane walking the slice length (profiles/r02_sweep_r2h.jsonl) — the
      // coarse kernels are bound by their gathers' latency, not by the
      // padding's bytes, and the divergent trip counts cost more
      std::vector<unsigned char> rl(nc);
      bool fits = true;
      for (int q = 0; q < nc; ++q) {
        const int I = row_at(q), l = crow_ptr[I + 1] - crow_ptr[I];
        fits = fits && l < 256;
        rl[q] = (unsigned char)std::min(l, 255);
      }
      const char* e = getenv("DFVM_AMG_RLEN");
      D.use_rlen = e && atoi(e) == 1;
      unsigned char* d_rl = nullptr;
      if (fits && (st = A->up(&d_rl, rl))) return st;
      D.rlen = fits ? d_rl : nullptr;
    }
    if (A->prm.csr && A->prm.perm == 0) {
      // CSR-stream copy: greedy warp chunks of whole rows (<= 32 rows,
      // <= kCsrChunk entries); a row longer than a chunk disables it
      std::vector<int> cptr(1, 0);
      bool ok = true;
      for (int I = 0; I < nc && ok;) {
        int rows = 0, ent = 0;
        while (I < nc && rows < 32 && ent + (crow_ptr[I + 1] - crow_ptr[I]) <= kCsrChunk) {
          ent += crow_ptr[I + 1] - crow_ptr[I];
          ++rows; ++I;
        }
        if (rows == 0) ok = false;
        else cptr.push_back(I);
      }
      if (ok) {
        D.n_chunk = (int)cptr.size() - 1;
        D.nnz_csr = (int64_t)ccol.size();
        if ((st = A->up(&D.c_ptr, cptr)) || (st = A->up(&D.c_rp, crow_ptr)) || (st = A->up(&D.c_col, ccol)) ||
            (st = A->up(&D.c_pos, epos)) || (st = A->zalloc(&D.c_coef, ccol.size())))
          return st;
      }
    }
    H.push_back(std::move(C));
    ++lev;
  }
  return DFVM_OK;
}

template <class P, class T>
static dfvm_status build(dfvm_mesh* m, const DevMesh<T>& M, AmgH<P>* A) {
  A->m = m;
  std::vector<HostLevel> H(1);
  H[0].n = M.n_own;
  H[0].ms_ptr = m->h_ms_ptr; H[0].ms_len = m->h_ms_len; H[0].mnb = m->h_mnb;
  sell_to_csr(H[0], M.n_own);
  // device view of level 0 (the mesh's matrix layout; coef / diag bound per update)
  AmgLevelDev<P>& L0 = A->L[0];
  L0.n = M.n_own; L0.n_slices = M.n_slices; L0.n_sell = M.n_minc; L0.nnz = M.nnz;
  L0.ms_ptr = M.ms_ptr; L0.ms_len = M.ms_len; L0.mnb = M.mnb;
  dfvm_status st;
  if ((st = A->zalloc(&L0.il1, M.n_own)) || (st = A->zalloc(&L0.x, M.n_cells)) || (st = A->zalloc(&L0.r, M.n_own)) ||
      (st = A->zalloc(&L0.t, M.n_cells)))
    return st;
  if (!std::is_same<P, T>::value) {
    if ((st = A->zalloc(&L0.coef_own, (size_t)M.n_minc)) || (st = A->zalloc(&L0.diag_own, M.n_own))) return st;
    L0.coef = L0.coef_own; L0.diag = L0.diag_own;
  }
  int lev = 0;
  if ((st = coarsen_serial(A, H, lev))) return st;
  A->nlev = lev + 1;
  if (getenv("DFVM_AMG_VERBOSE"))
    for (int k = 0; k <= lev; ++k)
      fprintf(stderr, "[amg] level %d: rows %d, SELL slots %lld, entries %d (%.2f per row, padding %.1f %%)\n", k,
              H[k].n, (long long)H[k].ms_ptr.back(), H[k].rp[H[k].n], (double)H[k].rp[H[k].n] / std::max(1, H[k].n),
              100.0 * (1.0 - (double)H[k].rp[H[k].n] / std::max<double>(1.0, (double)H[k].ms_ptr.back())));
  const int nc = A->L[lev].n;
  if (lev > 0 && nc <= A->prm.direct) {
    A->ainv_ld = (nc > kDirectMax && std::is_same<P, float>::value) ? (nc + 7) / 8 * 8 : nc;
    if ((st = A->zalloc(&A->ainv, (size_t)nc * A->ainv_ld))) return st;
  }
  return DFVM_OK;
}

// ---- several ranks: a distributed hierarchy.
// Aggregation stays rank-local (an aggregate never spans ranks), but every
// coarse operator is the Galerkin product of the GLOBAL matrix: the
// couplings through the interface become entries to ghost aggregates of the
// neighbouring ranks, each level carries a halo, and the coarsest level is
// solved globally.  So the preconditioner sees the whole domain at every
// level (round 1's rank-local coarse levels — block Jacobi across ranks —
// grew the PCG iterations from 13 to 71 per solve at P = 8 on a 12.5M-cell
// C5 pipe, profiles/r02_scale_iters_c5nz204_rank_local_amg.jsonl).
// Collective: all ranks build at the same time (host decisions are agreed
// through all-gathers, so every rank makes the same number of levels and the
// same halo / all-gather sequence in the cycle).
static dfvm_status agree_all(dfvm_mesh* m, double v, std::vector<double>& out, cudaStream_t s) {
  const int P = m->part.P;
  double *dl = nullptr, *da = nullptr;
  dfvm_status st;
  if ((st = dev_alloc_n(&dl, 1, s, false)) || (st = dev_alloc_n(&da, (size_t)P, s, false))) return st;
  DFVM_CUDA(cudaMemcpyAsync(dl, &v, 8, cudaMemcpyHostToDevice, s));
  if ((st = allgather_f64(m, dl, da, 1, s))) return st;
  out.assign(P, 0.0);
  DFVM_CUDA(cudaMemcpyAsync(out.data(), da, 8 * (size_t)P, cudaMemcpyDeviceToHost, s));
  DFVM_CUDA(cudaStreamSynchronize(s));
  dev_free(dl, s);
  dev_free(da, s);
  return DFVM_OK;
}

template <class P, class T>
static dfvm_status build_dist(dfvm_mesh* m, const DevMesh<T>& M, AmgH<P>* A, cudaStream_t s) {
  A->m = m;
  A->dist = true;
  const Part& Pt = m->part;
  const int NR = Pt.P;
  const int64_t Ng = m->H.N;
  std::vector<HostLevel> H(1);
  HostLevel& H0 = H[0];
  H0.n = M.n_own;
  H0.ms_ptr = m->h_ms_ptr; H0.ms_len = m->h_ms_len; H0.mnb = m->h_mnb;
  sell_to_csr(H0, M.n_own);
  sell_to_ghost_csr(H0);
  H0.ng = (int)Pt.n_ghost;
  H0.ghost_peer.assign(Pt.ghost_peer.begin(), Pt.ghost_peer.end());
  H0.ghost_key.resize(H0.ng);
  for (int k = 0; k < H0.ng; ++k) {
    const int q = Pt.ghost_peer[k];
    H0.ghost_key[k] = (int)(Pt.ghost_gid[k] - (int64_t)q * Ng / NR);
  }
  H0.halo.n_own = H0.n;
  H0.halo.peers = Pt.peers;
  H0.halo.send_off = Pt.peer_send_off;
  H0.halo.ghost_off = Pt.peer_ghost_off;
  H0.halo.send_idx.resize(Pt.send_gid.size());
  for (size_t i = 0; i < Pt.send_gid.size(); ++i) H0.halo.send_idx[i] = (int32_t)(Pt.send_gid[i] - Pt.lo);
  H0.halo.ready = true;
  A->halos[0] = H0.halo;
  AmgLevelDev<P>& L0 = A->L[0];
  L0.n = M.n_own; L0.n_slices = M.n_slices; L0.n_sell = M.n_minc; L0.nnz = M.nnz; L0.n_cells = M.n_cells;
  L0.ms_ptr = M.ms_ptr; L0.ms_len = M.ms_len; L0.mnb = M.mnb;
  dfvm_status st;
  if ((st = A->zalloc(&L0.il1, M.n_own)) || (st = A->zalloc(&L0.x, M.n_cells)) || (st = A->zalloc(&L0.r, M.n_own)) ||
      (st = A->zalloc(&L0.t, M.n_cells)))
    return st;
  if (!std::is_same<P, T>::value) {
    if ((st = A->zalloc(&L0.coef_own, (size_t)M.n_minc)) || (st = A->zalloc(&L0.diag_own, M.n_own))) return st;
    L0.coef = L0.coef_own; L0.diag = L0.diag_own;
  }
  // the global coarsest system holds NR * (rows per rank): stop each rank's
  // coarsening near 256 / NR rows (never below 32), so the redundant inverse
  // of each update stays at Np <= ~256 (<= kDirectMax = 512 enforced below)
  const int target = std::max(32, std::min(A->prm.coarse, 256 / NR));
  int lev = 0;
  std::vector<double> votes;
  int32_t* d_agg = nullptr;
  while (lev + 1 < kMaxLevels) {
    HostLevel& F = H[lev];
    // distribute while the level is large; once the union of the ranks'
    // rows is <= prm.agglom it is agglomerated (below) and the rest of the
    // hierarchy is replicated: the small levels are latency-bound anyway,
    // and every distributed visit costs halo exchanges
    std::vector<double> sizes;
    if ((st = agree_all(m, (double)F.n, sizes, s))) return st;
    double total = 0;
    for (double v : sizes) total += v;
    if (lev > 0 && total <= A->prm.agglom) break;
    int nc = 0;
    std::vector<int> agg = aggregate(F, nc);
    if (A->prm.renum) renumber_by_first_member(agg, nc);
    const bool want = F.n > target && nc < F.n * 0.85 && nc >= 32;
    if ((st = agree_all(m, want ? 1.0 : 0.0, votes, s))) return st;
    bool all = true;
    for (double v : votes) all = all && v > 0.5;
    if (!all) break;
    // owners' aggregate of every ghost row: one halo exchange of agg (int32 bits)
    std::vector<int> agg_ext(F.n + F.ng, -1);
    for (int i = 0; i < F.n; ++i) agg_ext[i] = agg[i];
    if ((st = dev_alloc_n(&d_agg, (size_t)(F.n + F.ng), s, false))) return st;
    DFVM_CUDA(cudaMemcpyAsync(d_agg, agg_ext.data(), 4 * (size_t)(F.n + F.ng), cudaMemcpyHostToDevice, s));
    if ((st = halo_exchange_lists(m, A->halos[lev], d_agg, 1, false, s))) return st;
    DFVM_CUDA(cudaMemcpyAsync(agg_ext.data(), d_agg, 4 * (size_t)(F.n + F.ng), cudaMemcpyDeviceToHost, s));
    DFVM_CUDA(cudaStreamSynchronize(s));
    dev_free(d_agg, s);
    d_agg = nullptr;
    // coarse ghosts: (owner, owner's aggregate) of every ghost column, sorted
    std::vector<std::pair<int, int>> cg;
    for (size_t k = 0; k < F.gcol.size(); ++k) {
      const int c = F.gcol[k];
      cg.push_back({F.ghost_peer[c - F.n], agg_ext[c]});
    }
    std::sort(cg.begin(), cg.end());
    cg.erase(std::unique(cg.begin(), cg.end()), cg.end());
    auto gidx = [&](int q, int key) {
      return nc + (int)(std::lower_bound(cg.begin(), cg.end(), std::make_pair(q, key)) - cg.begin());
    };
    HostLevel C;
    C.n = nc;
    C.ng = (int)cg.size();
    C.ghost_peer.resize(C.ng);
    C.ghost_key.resize(C.ng);
    for (int k = 0; k < C.ng; ++k) { C.ghost_peer[k] = cg[k].first; C.ghost_key[k] = cg[k].second; }
    // coarse halo: to peer q the aggregates of the fine rows sent to q, from
    // q the ghost aggregates owned by q (both ascending: the same list)
    C.halo.n_own = nc;
    C.halo.peers = F.halo.peers;
    C.halo.send_off.assign(1, 0);
    C.halo.ghost_off.assign(1, 0);
    for (size_t pi = 0; pi < F.halo.peers.size(); ++pi) {
      const int q = F.halo.peers[pi];
      std::vector<int> snd;
      for (int64_t k = F.halo.send_off[pi]; k < F.halo.send_off[pi + 1]; ++k) snd.push_back(agg[F.halo.send_idx[k]]);
      std::sort(snd.begin(), snd.end());
      snd.erase(std::unique(snd.begin(), snd.end()), snd.end());
      for (int v : snd) C.halo.send_idx.push_back(v);
      C.halo.send_off.push_back((int64_t)C.halo.send_idx.size());
      int64_t gcount = 0;
      for (int k = 0; k < C.ng; ++k) gcount += C.ghost_peer[k] == q;
      C.halo.ghost_off.push_back(C.halo.ghost_off.back() + gcount);
    }
    C.halo.ready = true;
    // members
    std::vector<int> mem_ptr(nc + 1, 0), mem(F.n);
    for (int i = 0; i < F.n; ++i) mem_ptr[agg[i] + 1]++;
    for (int I = 0; I < nc; ++I) mem_ptr[I + 1] += mem_ptr[I];
    {
      std::vector<int> pp(mem_ptr.begin(), mem_ptr.end() - 1);
      for (int i = 0; i < F.n; ++i) mem[pp[agg[i]]++] = i;
    }
    // coarse rows: owned columns agg[c], ghost columns their coarse ghost
    std::vector<int> crow_ptr(nc + 1, 0), ccol, dg_ptr(nc + 1, 0), dg_idx;
    std::vector<std::vector<int>> gal_lists;
    std::vector<std::pair<int, int>> buf;
    for (int I = 0; I < nc; ++I) {
      buf.clear();
      for (int q = mem_ptr[I]; q < mem_ptr[I + 1]; ++q) {
        const int i = mem[q];
        for (int k = F.rp[i]; k < F.rp[i + 1]; ++k) buf.push_back({agg[F.col[k]], F.pos[k]});
        for (int k = F.grp[i]; k < F.grp[i + 1]; ++k)
          buf.push_back({gidx(F.ghost_peer[F.gcol[k] - F.n], agg_ext[F.gcol[k]]), F.gpos[k]});
      }
      std::sort(buf.begin(), buf.end());
      for (size_t k = 0; k < buf.size();) {
        const int J = buf[k].first;
        size_t e = k;
        while (e < buf.size() && buf[e].first == J) ++e;
        if (J == I) {
          for (size_t u = k; u < e; ++u) dg_idx.push_back(buf[u].second);
        } else {
          ccol.push_back(J);
          gal_lists.emplace_back();
          for (size_t u = k; u < e; ++u) gal_lists.back().push_back(buf[u].second);
        }
        k = e;
      }
      crow_ptr[I + 1] = (int)ccol.size();
      dg_ptr[I + 1] = (int)dg_idx.size();
    }
    const int S = (nc + 31) / 32;
    C.ms_ptr.assign(S + 1, 0);
    C.ms_len.assign(S, 0);
    for (int sl = 0; sl < S; ++sl) {
      int w = 0;
      for (int I = sl * 32; I < std::min(nc, sl * 32 + 32); ++I) w = std::max(w, crow_ptr[I + 1] - crow_ptr[I]);
      C.ms_len[sl] = w;
      C.ms_ptr[sl + 1] = C.ms_ptr[sl] + 32 * w;
    }
    C.mnb.assign(C.ms_ptr[S], 0);
    std::vector<int> gal_ptr(C.ms_ptr[S] + 1, 0), gal_idx, slot_entry(C.ms_ptr[S], -1);
    for (int I = 0; I < nc; ++I) {
      const int sl = I / 32, lane = I % 32;
      for (int j = 0; j < C.ms_len[sl]; ++j) {
        const int pp = C.ms_ptr[sl] + 32 * j + lane;
        const int e = crow_ptr[I] + j;
        if (e < crow_ptr[I + 1]) { C.mnb[pp] = ccol[e]; slot_entry[pp] = e; }
        else C.mnb[pp] = I;
      }
    }
    for (int pp = 0; pp < C.ms_ptr[S]; ++pp) {
      if (slot_entry[pp] >= 0) for (int f : gal_lists[slot_entry[pp]]) gal_idx.push_back(f);
      gal_ptr[pp + 1] = (int)gal_idx.size();
    }
    sell_to_csr(C, nc);
    sell_to_ghost_csr(C);
    AmgLevelDev<P>& D = A->L[lev + 1];
    const int ncell = nc + C.ng;
    D.n = nc; D.n_slices = S; D.n_sell = C.ms_ptr[S]; D.n_cells = ncell;
    D.nnz = (int64_t)ccol.size();
    int *p0, *p1, *p2;
    if ((st = A->up(&p0, C.ms_ptr)) || (st = A->up(&p1, C.ms_len)) || (st = A->up(&p2, C.mnb)) ||
        (st = A->up(&D.gal_ptr, gal_ptr)) || (st = A->up(&D.gal_idx, gal_idx)) || (st = A->up(&D.dg_ptr, dg_ptr)) ||
        (st = A->up(&D.dg_idx, dg_idx)) || (st = A->up(&D.mem_ptr, mem_ptr)) || (st = A->up(&D.mem, mem)) ||
        (st = A->up(&A->L[lev].agg, agg)) || (st = A->zalloc(&D.coef_own, (size_t)D.n_sell)) ||
        (st = A->zalloc(&D.diag_own, nc)) || (st = A->zalloc(&D.il1, nc)) || (st = A->zalloc(&D.x, ncell)) ||
        (st = A->zalloc(&D.b, nc)) || (st = A->zalloc(&D.r, ncell)) || (st = A->zalloc(&D.t, ncell)) ||
        (st = A->zalloc(&D.e, ncell)) || (st = A->zalloc(&D.r2, nc)))
      return st;
    D.ms_ptr = p0; D.ms_len = p1; D.mnb = p2;
    D.coef = D.coef_own; D.diag = D.diag_own;
    A->halos[lev + 1] = C.halo;
    H.push_back(std::move(C));
    ++lev;
  }
  A->nlev = lev + 1;
  A->ld = lev;
  if (lev == 0) return DFVM_OK;   // nothing coarsened: the single-level path of cycle0
  // agglomeration of the level-lev rows of all ranks into G0 = level lev + 1
  HostLevel& Hd = H[lev];
  std::vector<double> cnts;
  if ((st = agree_all(m, (double)Hd.n, cnts, s))) return st;
  std::vector<int> cnt(NR), off(NR + 1, 0);
  for (int r = 0; r < NR; ++r) { cnt[r] = (int)cnts[r]; off[r + 1] = off[r] + cnt[r]; }
  const int NG = off[NR];
  const int me = Pt.rank;
  A->goff = off[me];
  // canonical values of this rank's rows: diag, owned-column entries, ghost-column entries
  std::vector<int> pk;
  std::vector<double> grow, gcolv;
  for (int i = 0; i < Hd.n; ++i) {
    pk.push_back(-1 - i); grow.push_back(off[me] + i); gcolv.push_back(off[me] + i);
    for (int k = Hd.rp[i]; k < Hd.rp[i + 1]; ++k) {
      pk.push_back(Hd.pos[k]); grow.push_back(off[me] + i); gcolv.push_back(off[me] + Hd.col[k]);
    }
    for (int k = Hd.grp[i]; k < Hd.grp[i + 1]; ++k) {
      const int c = Hd.gcol[k] - Hd.n;
      pk.push_back(Hd.gpos[k]); grow.push_back(off[me] + i);
      gcolv.push_back(off[Hd.ghost_peer[c]] + Hd.ghost_key[c]);
    }
  }
  std::vector<double> vm;
  if ((st = agree_all(m, (double)pk.size(), vm, s))) return st;
  int Vmax = 0, Nmax = 0;
  for (double v : vm) Vmax = std::max(Vmax, (int)v);
  for (int c : cnt) Nmax = std::max(Nmax, c);
  A->Vmax = Vmax; A->Nmax = Nmax; A->Vloc = (int)pk.size();
  // structure exchange: [rows | cols] per rank, padded with -1
  std::vector<double> sbuf(2 * (size_t)Vmax, -1.0), all((size_t)NR * 2 * Vmax);
  for (size_t k = 0; k < pk.size(); ++k) { sbuf[k] = grow[k]; sbuf[Vmax + k] = gcolv[k]; }
  {
    double *dl = nullptr, *da = nullptr;
    if ((st = dev_alloc_n(&dl, sbuf.size(), s, false)) || (st = dev_alloc_n(&da, all.size(), s, false))) return st;
    DFVM_CUDA(cudaMemcpyAsync(dl, sbuf.data(), 8 * sbuf.size(), cudaMemcpyHostToDevice, s));
    if ((st = allgather_f64(m, dl, da, 2 * Vmax, s))) return st;
    DFVM_CUDA(cudaMemcpyAsync(all.data(), da, 8 * all.size(), cudaMemcpyDeviceToHost, s));
    DFVM_CUDA(cudaStreamSynchronize(s));
    dev_free(dl, s);
    dev_free(da, s);
  }
  // G0: global rows, off-diagonal entries sorted by column, value sources
  std::vector<std::vector<std::pair<int, int>>> rows(NG);   // (col, source index)
  std::vector<int> gdmap(NG, -1);
  for (int r = 0; r < NR; ++r)
    for (int k = 0; k < Vmax; ++k) {
      const double rw = all[(size_t)r * 2 * Vmax + k];
      if (rw < 0) continue;
      const int gr = (int)rw, gc = (int)all[(size_t)r * 2 * Vmax + Vmax + k];
      const int src = r * Vmax + k;
      if (gr == gc) gdmap[gr] = src;
      else rows[gr].push_back({gc, src});
    }
  HostLevel G;
  G.n = NG;
  const int S = (NG + 31) / 32;
  G.ms_ptr.assign(S + 1, 0);
  G.ms_len.assign(S, 0);
  for (int I = 0; I < NG; ++I) std::sort(rows[I].begin(), rows[I].end());
  for (int sl = 0; sl < S; ++sl) {
    int w = 0;
    for (int I = sl * 32; I < std::min(NG, sl * 32 + 32); ++I) w = std::max(w, (int)rows[I].size());
    G.ms_len[sl] = w;
    G.ms_ptr[sl + 1] = G.ms_ptr[sl] + 32 * w;
  }
  G.mnb.assign(G.ms_ptr[S], 0);
  std::vector<int> gmap(std::max(1, G.ms_ptr[S]), -1);
  int64_t gnnz = 0;
  for (int I = 0; I < NG; ++I) {
    const int sl = I / 32, lane = I % 32;
    for (int j = 0; j < G.ms_len[sl]; ++j) {
      const int pp = G.ms_ptr[sl] + 32 * j + lane;
      if (j < (int)rows[I].size()) { G.mnb[pp] = rows[I][j].first; gmap[pp] = rows[I][j].second; ++gnnz; }
      else G.mnb[pp] = I;
    }
  }
  sell_to_csr(G, NG);
  const int lg = lev + 1;
  AmgLevelDev<P>& DG = A->L[lg];
  DG.n = NG; DG.n_slices = S; DG.n_sell = G.ms_ptr[S]; DG.nnz = gnnz; DG.n_cells = NG;
  int *q0, *q1, *q2;
  std::vector<int> pkv(std::max<size_t>(1, pk.size()), 0);
  for (size_t k = 0; k < pk.size(); ++k) pkv[k] = pk[k];
  if ((st = A->up(&q0, G.ms_ptr)) || (st = A->up(&q1, G.ms_len)) || (st = A->up(&q2, G.mnb)) ||
      (st = A->up(&A->d_gmap, gmap)) || (st = A->up(&A->d_gdmap, gdmap)) || (st = A->up(&A->d_pk, pkv)) ||
      (st = A->up(&A->d_cnt, cnt)) || (st = A->up(&A->d_off, off)) ||
      (st = A->zalloc(&DG.coef_own, (size_t)DG.n_sell)) || (st = A->zalloc(&DG.diag_own, NG)) ||
      (st = A->zalloc(&DG.il1, NG)) || (st = A->zalloc(&DG.x, NG)) || (st = A->zalloc(&DG.b, NG)) ||
      (st = A->zalloc(&DG.r, NG)) || (st = A->zalloc(&DG.t, NG)) || (st = A->zalloc(&DG.e, NG)) ||
      (st = A->zalloc(&DG.r2, NG)) || (st = A->zalloc(&A->d_vals, (size_t)Vmax)) ||
      (st = A->zalloc(&A->d_vals_all, (size_t)NR * Vmax)) || (st = A->zalloc(&A->d_rhs, (size_t)Nmax)) ||
      (st = A->zalloc(&A->d_rhs_all, (size_t)NR * Nmax)))
    return st;
  DG.ms_ptr = q0; DG.ms_len = q1; DG.mnb = q2;
  DG.coef = DG.coef_own; DG.diag = DG.diag_own;
  A->agglom = true;
  H.push_back(std::move(G));
  lev = lg;
  if ((st = coarsen_serial(A, H, lev))) return st;
  A->nlev = lev + 1;
  const int ncs = A->L[lev].n;
  if (lev > lg - 1 && ncs <= A->prm.direct) {
    A->ainv_ld = (ncs > kDirectMax && std::is_same<P, float>::value) ? (ncs + 7) / 8 * 8 : ncs;
    if ((st = A->zalloc(&A->ainv, (size_t)ncs * A->ainv_ld))) return st;
  }
  if (getenv("DFVM_AMG_VERBOSE"))
    for (int k = 0; k <= lev; ++k)
      fprintf(stderr, "[amg r%d] level %d: rows %d + %d ghosts, entries %d + %d to ghosts%s\n", Pt.rank, k, H[k].n,
              H[k].ng, H[k].rp[H[k].n], H[k].grp.empty() ? 0 : H[k].grp[H[k].n],
              k == lg ? " (agglomerated, replicated)" : (k > lg ? " (replicated)" : ""));
  return DFVM_OK;
}

// Lanes per row of each level's kernels: one thread per row
// while the level alone fills the GPU (kGroupFill threads), else the
// smallest power of two G <= 16 (32 for the restriction) that does, bounded
// by the entries (members) per row — the deep levels are latency bound, and
// G lanes cut a row's chain of dependent gathers by G.  Level 0 keeps one
// thread per row.  DFVM_AMG_GROUP=0: one thread per row everywhere.
constexpr int64_t kGroupFill = 148 * 2048;
static int group_for(int64_t n, double per_row, int gmax) {
  // DFVM_AMG_GFILL: the thread count a level must reach (default kGroupFill)
  const int64_t fill = [] { const char* e = getenv("DFVM_AMG_GFILL"); return e ? std::max<int64_t>(1, atoll(e)) : kGroupFill; }();
  int G = 1;
  while (G < gmax && n * G < fill && G < per_row) G *= 2;
  return G;
}
template <class P>
static void set_groups(AmgH<P>* A) {
  const char* e = getenv("DFVM_AMG_GROUP");
  const bool on = !(e && atoi(e) == 0);
  for (int l = 0; l < A->nlev; ++l) {
    AmgLevelDev<P>& L = A->L[l];
    L.G = (on && l > 0) ? group_for(L.n, (double)L.nnz / std::max(1, L.n), 16) : 1;
    L.Gr = (on && l > 0) ? group_for(L.n, (double)A->L[l - 1].n / std::max(1, L.n), 32) : 1;
  }
  if (getenv("DFVM_AMG_VERBOSE"))
    for (int l = 0; l < A->nlev; ++l) fprintf(stderr, "[amg] level %d: %d lanes per row, %d per restricted row\n", l, A->L[l].G, A->L[l].Gr);
}

template <class T>
dfvm_status amg_create(dfvm_mesh* m, const DevMesh<T>& M, bool fp32, Amg<T>** out, cudaStream_t s) {
  Amg<T>* A = new Amg<T>();
  dfvm_status st;
  const bool dist = m->part.P > 1;
  if (fp32 && !std::is_same<T, float>::value) {
    A->lo = new AmgH<float>();
    A->lo->prm.fp32_defaults();
    st = dist ? build_dist<float, T>(m, M, A->lo, s) : build<float, T>(m, M, A->lo);
  } else {
    A->same = new AmgH<T>();
    if (std::is_same<T, float>::value) A->same->prm.fp32_defaults();
    st = dist ? build_dist<T, T>(m, M, A->same, s) : build<T, T>(m, M, A->same);
  }
  if (st) { delete A; return st; }
  if (A->lo) set_groups(A->lo); else set_groups(A->same);
  DFVM_CUDA(cudaStreamSynchronize(nullptr));   // pageable uploads + zero-fills done before the caller's stream runs
  *out = A;
  return DFVM_OK;
}

template <class T>
void amg_destroy(Amg<T>* A) { delete A; }

template <class P>
static int levels(const AmgH<P>* A, int* sizes) {
  for (int l = 0; l < A->nlev; ++l) sizes[l] = A->L[l].n;
  return A->nlev;
}
template <class T>
int amg_levels(const Amg<T>* A, int* sizes) { return A->same ? levels(A->same, sizes) : levels(A->lo, sizes); }

// ------------------------------------------------------------ kernels
template <class P, class T>
__global__ void k_amg_cvt(int64_t n, const T* __restrict__ a, P* __restrict__ b) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (P)a[i];
}

template <class T>
__global__ void k_gal_off(int64_t n_sell, const int* __restrict__ gp, const int* __restrict__ gi,
                          const T* __restrict__ fcoef, T* __restrict__ ccoef) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_sell; e += (int64_t)gridDim.x * blockDim.x) {
    T s = T(0);
    for (int k = gp[e]; k < gp[e + 1]; ++k) s += fcoef[gi[k]];
    ccoef[e] = s;
  }
}

template <class T>
__global__ void k_gal_diag(int n, const int* __restrict__ mp, const int* __restrict__ mem,
                           const int* __restrict__ dp, const int* __restrict__ di, const T* __restrict__ fdiag,
                           const T* __restrict__ fcoef, T* __restrict__ cdiag) {
  PDL_ENTRY();
  for (int I = blockIdx.x * blockDim.x + threadIdx.x; I < n; I += gridDim.x * blockDim.x) {
    T s = T(0);
    for (int k = mp[I]; k < mp[I + 1]; ++k) s += fdiag[mem[k]];
    for (int k = dp[I]; k < dp[I + 1]; ++k) s += fcoef[di[k]];
    cdiag[I] = s;
  }
}

__device__ __forceinline__ int slot_row(const SellView& S, int q) { return S.perm ? __ldg(&S.perm[q]) : q; }

// inverse l1 diagonal: 1 / (a_ii + sum_j |a_ij|) over the row's SELL entries
// (stored inverted: the smoothers multiply, no fp64 division per gather)
template <class T>
__global__ void k_il1(int n, SellView S, const T* __restrict__ coef, const T* __restrict__ diag, T* __restrict__ il1) {
  PDL_ENTRY();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int r = slot_row(S, q), sl = q >> 5, lane = q & 31;
    T a = diag[r];
    for (int j = 0; j < S.ms_len[sl]; ++j) a += fabs(coef[S.ms_ptr[sl] + 32 * j + lane]);
    il1[r] = T(1) / a;
  }
}

// ---- SELL row sums with G lanes per row
// Slot q's entries j = sub, sub + G, sub + 2G, ... are summed by lane `sub`
// of the row's G-lane group, in batches of 4 entries: every column /
// coefficient load of the batch first, then every gathered value, then the
// FMAs in entry order; the last batch is predicated (no dependent load chain
// for a leftover entry: one memory round trip per batch).  G = 1 keeps the
// strict entry order of one thread per row.  G > 1 (small coarse levels,
// which are latency bound: one thread per row walks 15 entries in 4
// dependent rounds) splits the row over G lanes and combines the partials
// with a shuffle tree (lane 0 of the group ends with the sum).
template <int G, class T, class NB>
__device__ __forceinline__ T row_part(const SellView& S, int q, int sub, bool live, const T* __restrict__ coef, T acc,
                                      NB nb) {
  const int sl = q >> 5, lane = q & 31;
  // a lane stops at its own row's length (S.rlen): the padding slots of
  // shorter rows in the slice are neither loaded nor gathered — SELL-32
  // padding is 30-35 % on the aggregation levels, and a sector whose 8 lanes
  // are all padding is never fetched (same sums: padding coefficients are 0)
  const int len = live ? (S.rlen ? (int)__ldg(&S.rlen[q]) : __ldg(&S.ms_len[sl])) : 0;
  const int base = live ? __ldg(&S.ms_ptr[sl]) + lane : 0;
  if constexpr (G == 1) {
    // one thread per row: whole batches, then the leftover entries one by one
    // (measured on C5: a predicated last batch was 4 % slower on level 2)
    int j = 0;
    for (; j + 4 <= len; j += 4) {
      T a[4], v[4];
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = __ldg(&coef[base + 32 * (j + u)]); c[u] = __ldg(&S.mnb[base + 32 * (j + u)]); }
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = nb(c[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += a[u] * v[u];
    }
    for (; j < len; ++j) acc += __ldg(&coef[base + 32 * j]) * nb(__ldg(&S.mnb[base + 32 * j]));
    return acc;
  } else {
  for (int j = sub; j < len; j += 4 * G) {
    T a[4], v[4];
    int c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = j + u * G < len;
      a[u] = ok ? __ldg(&coef[base + 32 * (j + u * G)]) : T(0);
      c[u] = ok ? __ldg(&S.mnb[base + 32 * (j + u * G)]) : -1;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = c[u] >= 0 ? nb(c[u]) : T(0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c[u] >= 0) acc += a[u] * v[u];
  }
  return acc;
  }
}
template <int G, class T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, G);
  return v;
}
// Grid-stride loop over the n rows with G consecutive threads per row.  The
// trip count is rounded up to whole warps so every lane of a warp takes part
// in the group shuffles; `live` marks the threads that own a real row, q_ is
// the SELL slot, sub_ the lane within the row's group.
#define AMG_GROUP_LOOP(n, G)                                                                               \
  const int sub_ = (int)(threadIdx.x & ((G) - 1));                                                          \
  const int64_t nt_ = (int64_t)(n) * (G), nt32_ = (nt_ + 31) & ~(int64_t)31;                                \
  for (int64_t t_ = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t_ < nt32_; t_ += (int64_t)gridDim.x * blockDim.x) \
    if (const bool live = t_ < nt_; true)                                                                   \
      if (const int q_ = live ? (int)(t_ / (G)) : 0; true)

template <class T>
__device__ __forceinline__ T row_apply(const SellView& S, int q, int r, const T* __restrict__ coef,
                                       const T* __restrict__ diag, const T* __restrict__ x) {
  return row_part<1>(S, q, 0, true, coef, diag[r] * x[r], [&](int c) { return x[c]; });
}

// Streaming AMG vector kernels: each thread takes kUnr rows per grid-stride
// step (row i0 + u * stride, so every load stays coalesced across the warp)
// and issues all their loads before any store — kUnr independent row chains
// in flight per thread instead of one (the 4-byte vectors of the fp32
// hierarchy left these kernels at 0.25-0.6 of the roofline).
constexpr int kUnr = 4;
#define AMG_UNR_LOOP(n)                                                                                \
  const int64_t st_ = (int64_t)gridDim.x * blockDim.x;                                                 \
  for (int64_t i0_ = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0_ < (n); i0_ += kUnr * st_)

// x = b / d1 (pre-smoothing from a zero guess); b in the caller's type TB
template <class P, class TB, class TX>
__global__ void k_amg_pre(int n, const TB* __restrict__ b, const P* __restrict__ il1, TX* __restrict__ x,
                          const int* done) {
  PDL_ENTRY();
  if (*done) return;
  AMG_UNR_LOOP(n) {
    P bv[kUnr], dv[kUnr];
#pragma unroll
    for (int u = 0; u < kUnr; ++u) {
      const int64_t i = i0_ + u * st_;
      bv[u] = i < n ? (P)b[i] : P(0);
      dv[u] = i < n ? il1[i] : P(0);
    }
#pragma unroll
    for (int u = 0; u < kUnr; ++u) {
      const int64_t i = i0_ + u * st_;
      if (i < n) x[i] = (TX)(bv[u] * dv[u]);
    }
  }
}
// r = b - A x
template <int G, class P, class TB>
__global__ void k_amg_resid(int n, SellView S, const P* __restrict__ coef, const P* __restrict__ diag,
                            const P* __restrict__ x, const TB* __restrict__ b, P* __restrict__ r, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  AMG_GROUP_LOOP(n, G) {
    const int i = live ? slot_row(S, q_) : 0;
    P acc = (live && sub_ == 0) ? diag[i] * x[i] : P(0);
    acc = group_sum<G>(row_part<G>(S, q_, sub_, live, coef, acc, [&](int c) { return x[c]; }));
    if (live && sub_ == 0) r[i] = (P)b[i] - acc;
  }
}
// b_c[I] = sum over the aggregate's members of r_f (G lanes per coarse row:
// deep levels have 17-24 members per aggregate)
template <int G, class T>
__global__ void k_amg_restrict(int nc, const int* __restrict__ mp, const int* __restrict__ mem,
                               const T* __restrict__ rf, T* __restrict__ bc, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  // (G = 1 too: the members in predicated batches of 4 — measured on C5 at
  // 3.95 / 2.70 ms/step on levels 0 / 1 against 4.22 / 3.00 one member at a
  // time, and 5.67 / 4.12 with 4 coarse rows per thread instead)
  AMG_GROUP_LOOP(nc, G) {
    const int k0 = live ? __ldg(&mp[q_]) : 0, k1 = live ? __ldg(&mp[q_ + 1]) : 0;
    T s = T(0);
    for (int k = k0 + sub_; k < k1; k += 4 * G) {
      int f[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) f[u] = k + u * G < k1 ? __ldg(&mem[k + u * G]) : -1;
      T v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = f[u] >= 0 ? rf[f[u]] : T(0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (f[u] >= 0) s += v[u];
    }
    s = group_sum<G>(s);
    if (live && sub_ == 0) bc[q_] = s;
  }
}
// t = x + w x_c[agg[i]]  (coarse correction, out of place: t feeds the smoother)
template <class T>
__global__ void k_amg_prolong(int n, const int* __restrict__ agg, const T* __restrict__ xc, const T* __restrict__ x,
                              T* __restrict__ t, T w, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  AMG_UNR_LOOP(n) {
    int a[kUnr];
    T xv[kUnr];
#pragma unroll
    for (int u = 0; u < kUnr; ++u) {
      const int64_t i = i0_ + u * st_;
      a[u] = i < n ? __ldg(&agg[i]) : 0;
      xv[u] = i < n ? x[i] : T(0);
    }
    T cv[kUnr];
#pragma unroll
    for (int u = 0; u < kUnr; ++u) cv[u] = xc[a[u]];
#pragma unroll
    for (int u = 0; u < kUnr; ++u) {
      const int64_t i = i0_ + u * st_;
      if (i < n) t[i] = xv[u] + w * cv[u];
    }
  }
}
// fused pre-smooth + residual (rows without ghost columns): x0 = b / d1 for
// the row and, on the fly, for every neighbour; writes x0 and r = b - A x0
template <int G, class T>
__global__ void k_amg_pre_resid(int n, SellView S, const T* __restrict__ coef, const T* __restrict__ diag,
                                const T* __restrict__ il1, const T* __restrict__ b, T* __restrict__ x0,
                                T* __restrict__ r, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  AMG_GROUP_LOOP(n, G) {
    const int i = live ? slot_row(S, q_) : 0;
    T bi = T(0), xi = T(0), acc = T(0);
    if (live && sub_ == 0) { bi = b[i]; xi = bi * il1[i]; acc = diag[i] * xi; }
    acc = group_sum<G>(row_part<G>(S, q_, sub_, live, coef, acc, [&](int c) { return b[c] * il1[c]; }));
    if (live && sub_ == 0) { x0[i] = xi; r[i] = bi - acc; }
  }
}
// fused prolongation + post-smooth: t = x0 + w P x_c (on the fly for the row
// and its neighbours), out = t + (b - A t) / d1; accum: out += that instead
// (the W-cycle's second visit adds its correction in place)
template <int G, class T>
__global__ void k_amg_prolong_smooth(int n, SellView S, const T* __restrict__ coef, const T* __restrict__ diag,
                                     const T* __restrict__ il1, const int* __restrict__ agg, const T* __restrict__ xc,
                                     T w, const T* __restrict__ x0, const T* __restrict__ b, T* __restrict__ out,
                                     int accum, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  AMG_GROUP_LOOP(n, G) {
    const int i = live ? slot_row(S, q_) : 0;
    T ti = T(0), acc = T(0);
    if (live && sub_ == 0) { ti = x0[i] + w * xc[agg[i]]; acc = diag[i] * ti; }
    acc = group_sum<G>(
        row_part<G>(S, q_, sub_, live, coef, acc, [&](int c) { return x0[c] + w * xc[agg[c]]; }));
    if (live && sub_ == 0) {
      const T z = ti + (b[i] - acc) * il1[i];
      out[i] = accum ? out[i] + z : z;
    }
  }
}

// x += e
template <class T>
__global__ void k_amg_add(int n, const T* __restrict__ e, T* __restrict__ x, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] += e[i];
}
// out = x + (b - A x) / d1   (b in TB, out in TO: level 0 reads / writes the
// PCG's type); accum: out += that (W-cycle second visit, in place)
template <int G, class P, class TB, class TO>
__global__ void k_amg_smooth(int n, SellView S, const P* __restrict__ coef, const P* __restrict__ diag,
                             const P* __restrict__ il1, const P* __restrict__ x, const TB* __restrict__ b,
                             TO* __restrict__ out, int accum, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  AMG_GROUP_LOOP(n, G) {
    const int i = live ? slot_row(S, q_) : 0;
    P acc = (live && sub_ == 0) ? diag[i] * x[i] : P(0);
    acc = group_sum<G>(row_part<G>(S, q_, sub_, live, coef, acc, [&](int c) { return x[c]; }));
    if (live && sub_ == 0) {
      const TO z = (TO)(x[i] + ((P)b[i] - acc) * il1[i]);
      out[i] = accum ? (TO)(out[i] + z) : z;
    }
  }
}
// level-0 post-smoother with the PCG's r.z folded in: z = t + (r - A t) / d1
// and the deterministic grid sum of r_i z_i (fp64) driving control step `kind`
template <class P, class T>
__global__ void __launch_bounds__(kThreads) k_amg_smooth_dot(int n, SellView S, const P* __restrict__ coef,
    const P* __restrict__ diag, const P* __restrict__ il1, const P* __restrict__ x, const T* __restrict__ b,
    T* __restrict__ out, const int* done, double* partials, unsigned* ticket, KCtl* ctl, Red red, int kind) {
  PDL_ENTRY();
  if (*done) return;
  double v[1] = {0};
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = slot_row(S, q);
    const T bi = b[i];
    const T zi = (T)(x[i] + ((P)bi - row_apply(S, q, i, coef, diag, x)) * il1[i]);
    out[i] = zi;
    v[0] += (double)bi * (double)zi;
  }
  double t[1];
  if (grid_sum<1>(v, partials, ticket, t)) red_finish<1>(red, kind, ctl, t);
}

// coarsest level: `sweeps` l1-Jacobi sweeps from zero, one block, in shared memory
template <class P, class TB, class TO>
__global__ void __launch_bounds__(1024) k_amg_coarse(int n, SellView S, const P* __restrict__ coef,
                                                    const P* __restrict__ diag, const P* __restrict__ il1,
                                                    const TB* __restrict__ b, TO* __restrict__ xout, int sweeps,
                                                    const int* done) {
  PDL_ENTRY();
  if (*done) return;
  __shared__ P xs[2][kCoarseMax];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[0][i] = (P)b[i] * il1[i];
  __syncthreads();
  int cur = 0;
  for (int it = 1; it < sweeps; ++it) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const int i = slot_row(S, q);
      xs[cur ^ 1][i] = xs[cur][i] + ((P)b[i] - row_apply(S, q, i, coef, diag, xs[cur])) * il1[i];
    }
    __syncthreads();
    cur ^= 1;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) xout[i] = (TO)xs[cur][i];
}

// Dense inverse of the coarsest matrix, one block: densify the SELL rows,
// then in-place Gauss-Jordan without pivoting (the Galerkin coarse matrix of
// an SPD operator is SPD).  Step k: row k <- row k / a_kk (with a_kk <- 1 first),
// row i <- row i - a_ik row k (with a_ik <- 0 first).
template <class P>
__global__ void __launch_bounds__(1024) k_amg_dense_inv(int n, SellView S, const P* __restrict__ coef,
                                                        const P* __restrict__ diag, P* __restrict__ A) {
  PDL_ENTRY();
  __shared__ P colk[kDirectMax], rowk[kDirectMax];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) A[e] = P(0);
  __syncthreads();
  for (int q = threadIdx.x; q < n; q += blockDim.x) {      // thread q owns slot q (row i)
    const int i = slot_row(S, q);
    A[(size_t)i * n + i] = diag[i];
    const int sl = q >> 5, lane = q & 31;
    for (int j = 0; j < S.ms_len[sl]; ++j) {
      const int p = S.ms_ptr[sl] + 32 * j + lane;
      if (S.mnb[p] < n) A[(size_t)i * n + S.mnb[p]] += coef[p];   // (ghost columns: dropped, rank-local block)
    }
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const P piv = A[(size_t)k * n + k];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      colk[i] = A[(size_t)i * n + k];
      rowk[i] = (i == k ? P(1) : A[(size_t)k * n + i]) / piv;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      const P a = A[e];
      A[e] = (i == k) ? rowk[j] : ((j == k ? P(0) : a) - colk[i] * rowk[j]);
    }
    __syncthreads();
  }
}

// Multi-launch Gauss-Jordan for coarsest levels above kDirectMax rows
// (experimental, DFVM_AMG_COARSE / DFVM_AMG_DIRECT up to kDirectBig): densify,
// then per pivot k one staging launch (row k / a_kk, column k) and one
// update launch over all n^2 entries (same arithmetic as k_amg_dense_inv).
template <class P>
__global__ void k_dense_fill(int n, SellView S, const P* __restrict__ coef, const P* __restrict__ diag,
                             P* __restrict__ A) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n; e += (int64_t)gridDim.x * blockDim.x)
    A[e] = P(0);
}
template <class P>
__global__ void k_dense_rows(int n, SellView S, const P* __restrict__ coef, const P* __restrict__ diag,
                             P* __restrict__ A) {
  PDL_ENTRY();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = slot_row(S, q);
    A[(size_t)i * n + i] = diag[i];
    const int sl = q >> 5, lane = q & 31;
    for (int j = 0; j < S.ms_len[sl]; ++j) {
      const int p = S.ms_ptr[sl] + 32 * j + lane;
      if (S.mnb[p] < n) A[(size_t)i * n + S.mnb[p]] += coef[p];
    }
  }
}
template <class P>
__global__ void k_gj_stage(int n, int k, const P* __restrict__ A, P* __restrict__ rowk, P* __restrict__ colk) {
  PDL_ENTRY();
  const P piv = A[(size_t)k * n + k];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    colk[i] = A[(size_t)i * n + k];
    rowk[i] = (i == k ? P(1) : A[(size_t)k * n + i]) / piv;
  }
}
template <class P>
__global__ void k_gj_update(int n, int k, P* __restrict__ A, const P* __restrict__ rowk, const P* __restrict__ colk) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    const P a = A[e];
    A[e] = (i == k) ? rowk[j] : ((j == k ? P(0) : a) - colk[i] * rowk[j]);
  }
}

// Blocked symmetric sweep for coarsest levels above kDirectMax rows (fp32):
// the dense n x n matrix in global memory (L2 resident), pivot blocks of
// kBlk rows.  Block step K (rows / cols k0 .. k0 + kb):
//   S = A_KK^-1 (one CTA, shared-memory sweep);  P = A_:K S  (n x kb);
//   A_ij -= P_i A_Kj  for i, j outside K   (the rank-kb update: a tiled SIMT
//                                             GEMM, 2 n^2 kb flops);
//   A_iK = P_i,  A_Kj = P_j^T (symmetry),  A_KK = -S.
// After every block the matrix holds -A^-1 (the block form of the sweep
// operator of k_amg_dense_inv_sym; no pivoting: SPD).  Densified from the
// lower triangle and mirrored, so it stays symmetric.
constexpr int kBlk = 64;
constexpr int kTM = 128, kTN = 128;   // update tile
template <class P>
__global__ void k_dense_rows_sym(int n, int ld, SellView S, const P* __restrict__ coef, const P* __restrict__ diag,
                                 P* __restrict__ A) {
  PDL_ENTRY();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = slot_row(S, q);
    A[(size_t)i * ld + i] = diag[i];
    const int sl = q >> 5, lane = q & 31;
    for (int j = 0; j < S.ms_len[sl]; ++j) {
      const int p = S.ms_ptr[sl] + 32 * j + lane;
      const int c = S.mnb[p];
      if (c < i) { A[(size_t)i * ld + c] += coef[p]; A[(size_t)c * ld + i] += coef[p]; }
    }
  }
}
// S = A_KK^-1 by the sweep operator in shared memory (one CTA)
// (1024 threads: 4 entries per thread per pivot; 256 threads took 57 us per
// 64-pivot block on C5, a third of each block step)
template <class P>
__global__ void __launch_bounds__(1024) k_blk_inv(int n, int ld, int k0, int kb, const P* __restrict__ A, P* __restrict__ Sb) {
  PDL_ENTRY();
  __shared__ P a[kBlk][kBlk + 1];
  __shared__ P ck[kBlk];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e / kb, c = e - r * kb;
    a[r][c] = A[(size_t)(k0 + r) * ld + k0 + c];
  }
  __syncthreads();
  for (int k = 0; k < kb; ++k) {
    for (int j = threadIdx.x; j < kb; j += blockDim.x) ck[j] = a[j][k];
    __syncthreads();
    const P rd = P(1) / ck[k];
    // the full kBlk x kBlk square with constant shifts (no runtime division)
#pragma unroll
    for (int e = threadIdx.x; e < kBlk * kBlk; e += 1024) {
      const int r = e / kBlk, c = e % kBlk;
      if (r < kb && c < kb && r != k && c != k) a[r][c] -= ck[r] * rd * ck[c];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < kb; j += blockDim.x) {
      const P v = (j == k) ? -rd : ck[j] * rd;
      a[j][k] = v;
      a[k][j] = v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e / kb, c = e - r * kb;
    Sb[r * kBlk + c] = -a[r][c];
  }
}
// Pb[i][c] = sum_t A[i][k0 + t] S[t][c]  (4 rows per CTA)
template <class P>
__global__ void __launch_bounds__(256) k_blk_panel(int n, int ld, int k0, int kb, const P* __restrict__ A,
                                                   const P* __restrict__ Sb, P* __restrict__ Pb) {
  PDL_ENTRY();
  __shared__ P s[kBlk][kBlk + 1];
  __shared__ P ar[4][kBlk];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) s[e / kb][e % kb] = Sb[(e / kb) * kBlk + e % kb];
  for (int i0 = blockIdx.x * 4; i0 < n; i0 += gridDim.x * 4) {
    __syncthreads();
    for (int e = threadIdx.x; e < 4 * kb; e += blockDim.x) {
      const int r = e / kb, t = e - r * kb;
      ar[r][t] = (i0 + r < n) ? A[(size_t)(i0 + r) * ld + k0 + t] : P(0);
    }
    __syncthreads();
    const int r = threadIdx.x / kBlk, c = threadIdx.x % kBlk;
    if (i0 + r < n && c < kb) {
      P acc = P(0);
      for (int t = 0; t < kb; ++t) acc += ar[r][t] * s[t][c];
      Pb[(size_t)(i0 + r) * kBlk + c] = acc;
    }
  }
}
// A_ij -= sum_t Pb[i][t] A[k0 + t][j]  for i, j outside block K: 128 x 128
// tile per CTA, 8 x 8 outputs per thread, both operands staged in shared memory
constexpr int kSP = kTM + 4;   // padded shared-memory rows (16-byte aligned, 4-way store conflicts at most)
template <class P>
__global__ void __launch_bounds__(256) k_blk_update(int n, int ld, int k0, int kb, P* __restrict__ A, const P* __restrict__ Pb) {
  PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char blk_smem[];
  P* sP = reinterpret_cast<P*>(blk_smem);          // [kBlk][kSP]   Pb^T tile
  P* sR = sP + kBlk * kSP;                          // [kBlk][kSP]   block-row tile
  const int i0 = blockIdx.y * kTM, j0 = blockIdx.x * kTN;
  for (int e = threadIdx.x; e < kTM * kBlk; e += blockDim.x) {
    const int i = e / kBlk, t = e - i * kBlk;
    sP[t * kSP + i] = (i0 + i < n && t < kb) ? Pb[(size_t)(i0 + i) * kBlk + t] : P(0);
  }
  for (int e = threadIdx.x; e < kBlk * kTN; e += blockDim.x) {
    const int t = e / kTN, j = e - t * kTN;
    sR[t * kSP + j] = (j0 + j < n && t < kb) ? A[(size_t)(k0 + t) * ld + j0 + j] : P(0);
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  P acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = P(0);
  // thread (tx, ty) owns rows ty + 16 r and columns tx + 16 c: the 16 lanes
  // of a half-warp read 16 consecutive values (conflict free), two row
  // values per warp are broadcasts, and the output stores are coalesced
  for (int t = 0; t < kb; ++t) {
    P a[8], b[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = sP[t * kSP + ty + 16 * r];
#pragma unroll
    for (int c = 0; c < 8; ++c) b[c] = sR[t * kSP + tx + 16 * c];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] += a[r] * b[c];
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + ty + 16 * r;
    if (i >= n || (i >= k0 && i < k0 + kb)) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = j0 + tx + 16 * c;
      if (j < n && !(j >= k0 && j < k0 + kb)) A[(size_t)i * ld + j] -= acc[r][c];
    }
  }
}
// block column / row K <- P (and P^T), A_KK <- -S
template <class P>
__global__ void k_blk_finish(int n, int ld, int k0, int kb, P* __restrict__ A, const P* __restrict__ Pb, const P* __restrict__ Sb) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * kb; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / kb), c = (int)(e - (int64_t)i * kb);
    if (i >= k0 && i < k0 + kb) {
      A[(size_t)i * ld + k0 + c] = -Sb[(i - k0) * kBlk + c];
    } else {
      const P v = Pb[(size_t)i * kBlk + c];
      A[(size_t)i * ld + k0 + c] = v;
      A[(size_t)(k0 + c) * ld + i] = v;
    }
  }
}
template <class P>
__global__ void k_negate(int64_t n, P* __restrict__ A) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) A[e] = -A[e];
}

// ---- lower-triangle form of the blocked sweep (the default): only the
// lower triangle (i >= j) is kept valid; the panel kernel also saves the old
// block column Q = A_:K, so the rank update A_ij -= P_i Q_j^T reads two n x kb
// buffers (both coalesced) and touches only tiles on or below the diagonal —
// half the flops of the full form.  The result is mirrored (and negated) at
// the end.
__device__ __forceinline__ size_t lo_at(int i, int j, int ld) {
  return i >= j ? (size_t)i * ld + j : (size_t)j * ld + i;
}
template <class P>
__global__ void k_dense_rows_lower(int n, int ld, SellView S, const P* __restrict__ coef, const P* __restrict__ diag,
                                   P* __restrict__ A) {
  PDL_ENTRY();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = slot_row(S, q);
    A[(size_t)i * ld + i] = diag[i];
    const int sl = q >> 5, lane = q & 31;
    for (int j = 0; j < S.ms_len[sl]; ++j) {
      const int p = S.ms_ptr[sl] + 32 * j + lane;
      const int c = S.mnb[p];
      if (c < i) A[(size_t)i * ld + c] += coef[p];
    }
  }
}
template <class P>
__global__ void __launch_bounds__(1024) k_blk_inv_lo(int n, int ld, int k0, int kb, const P* __restrict__ A,
                                                     P* __restrict__ Sb) {
  PDL_ENTRY();
  __shared__ P a[kBlk][kBlk + 1];
  __shared__ P ck[kBlk];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e / kb, c = e - r * kb;
    a[r][c] = A[lo_at(k0 + r, k0 + c, ld)];
  }
  __syncthreads();
  for (int k = 0; k < kb; ++k) {
    for (int j = threadIdx.x; j < kb; j += blockDim.x) ck[j] = a[j][k];
    __syncthreads();
    const P rd = P(1) / ck[k];
#pragma unroll
    for (int e = threadIdx.x; e < kBlk * kBlk; e += 1024) {
      const int r = e / kBlk, c = e % kBlk;
      if (r < kb && c < kb && r != k && c != k) a[r][c] -= ck[r] * rd * ck[c];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < kb; j += blockDim.x) {
      const P v = (j == k) ? -rd : ck[j] * rd;
      a[j][k] = v;
      a[k][j] = v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e / kb, c = e - r * kb;
    Sb[r * kBlk + c] = -a[r][c];
  }
}
// Qb[i][t] = old A_{i, k0+t} (through the lower triangle), Pb[i][c] = Qb[i] S[:, c]
template <class P>
__global__ void __launch_bounds__(256) k_blk_panel_lo(int n, int ld, int k0, int kb, const P* __restrict__ A,
                                                      const P* __restrict__ Sb, P* __restrict__ Pb, P* __restrict__ Qb) {
  PDL_ENTRY();
  __shared__ P s[kBlk][kBlk + 1];
  __shared__ P ar[4][kBlk];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) s[e / kb][e % kb] = Sb[(e / kb) * kBlk + e % kb];
  for (int i0 = blockIdx.x * 4; i0 < n; i0 += gridDim.x * 4) {
    __syncthreads();
    for (int e = threadIdx.x; e < 4 * kb; e += blockDim.x) {
      const int r = e / kb, t = e - r * kb;
      const P v = (i0 + r < n) ? A[lo_at(i0 + r, k0 + t, ld)] : P(0);
      ar[r][t] = v;
      if (i0 + r < n) Qb[(size_t)(i0 + r) * kBlk + t] = v;
    }
    __syncthreads();
    const int r = threadIdx.x / kBlk, c = threadIdx.x % kBlk;
    if (i0 + r < n && c < kb) {
      P acc = P(0);
      for (int t = 0; t < kb; ++t) acc += ar[r][t] * s[t][c];
      Pb[(size_t)(i0 + r) * kBlk + c] = acc;
    }
  }
}
// A_ij -= sum_t Pb[i][t] Qb[j][t] for i >= j outside block K (tiles above the
// diagonal return at once)
template <class P>
__global__ void __launch_bounds__(256) k_blk_update_lo(int n, int ld, int k0, int kb, P* __restrict__ A,
                                                       const P* __restrict__ Pb, const P* __restrict__ Qb) {
  PDL_ENTRY();
  const int i0 = blockIdx.y * kTM, j0 = blockIdx.x * kTN;
  if (j0 > i0 + kTM - 1) return;
  extern __shared__ __align__(16) unsigned char blk_smem[];
  P* sP = reinterpret_cast<P*>(blk_smem);          // [kBlk][kSP]   Pb^T tile
  P* sR = sP + kBlk * kSP;                          // [kBlk][kSP]   Qb^T tile
  for (int e = threadIdx.x; e < kTM * kBlk; e += blockDim.x) {
    const int i = e / kBlk, t = e - i * kBlk;
    sP[t * kSP + i] = (i0 + i < n && t < kb) ? Pb[(size_t)(i0 + i) * kBlk + t] : P(0);
    sR[t * kSP + i] = (j0 + i < n && t < kb) ? Qb[(size_t)(j0 + i) * kBlk + t] : P(0);
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  P acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = P(0);
  for (int t = 0; t < kb; ++t) {
    P a[8], b[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = sP[t * kSP + ty + 16 * r];
#pragma unroll
    for (int c = 0; c < 8; ++c) b[c] = sR[t * kSP + tx + 16 * c];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] += a[r] * b[c];
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + ty + 16 * r;
    if (i >= n || (i >= k0 && i < k0 + kb)) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = j0 + tx + 16 * c;
      if (j <= i && !(j >= k0 && j < k0 + kb)) A[(size_t)i * ld + j] -= acc[r][c];
    }
  }
}
// new block column K (lower storage): A_{i,K} = P_i, A_KK = -S
template <class P>
__global__ void k_blk_finish_lo(int n, int ld, int k0, int kb, P* __restrict__ A, const P* __restrict__ Pb,
                                const P* __restrict__ Sb) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * kb; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / kb), c = (int)(e - (int64_t)i * kb);
    if (i >= k0 && i < k0 + kb) {
      if (i - k0 >= c) A[(size_t)i * ld + k0 + c] = -Sb[(i - k0) * kBlk + c];
    } else {
      A[lo_at(i, k0 + c, ld)] = Pb[(size_t)i * kBlk + c];
    }
  }
}
// the inverse from the swept lower triangle: A_ij = A_ji = -(swept)_ij
template <class P>
__global__ void k_mirror_negate(int n, int ld, P* __restrict__ A) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    if (j > i) continue;
    const P v = -A[(size_t)i * ld + j];
    A[(size_t)i * ld + j] = v;
    if (j < i) A[(size_t)j * ld + i] = v;
  }
}

// Dense inverse of the (SPD) coarsest matrix in SHARED memory by the
// symmetric sweep operator on the packed lower triangle (round 2: the
// global-memory Gauss-Jordan above re-read and re-wrote the whole n x n
// matrix through L2 from one SM at every pivot — 2.4 ms per update for the
// 240-row coarsest level of C2, a quarter of its step).  Pivot k, with
// d = a_kk (a_ij for i < j read as a_ji):
//   a_ij -= a_ik a_jk / d   (i, j != k);   a_ik /= d (i != k);   a_kk = -1/d
// After all n pivots the packed matrix holds -A^-1 (no pivoting: the
// Galerkin coarse matrix of an SPD operator is SPD).  The result is expanded
// row-major into Ai (both triangles).  One block; dynamic shared memory
// n (n + 1) / 2 + n values (fp32: n <= 340).
template <class P>
__global__ void __launch_bounds__(1024) k_amg_dense_inv_sym(int n, SellView S, const P* __restrict__ coef,
                                                            const P* __restrict__ diag, P* __restrict__ Ai) {
  PDL_ENTRY();
  extern __shared__ unsigned char dyn_smem[];
  P* a = reinterpret_cast<P*>(dyn_smem);            // packed lower triangle, a[i (i + 1) / 2 + j], j <= i
  P* ck = a + (size_t)n * (n + 1) / 2;              // column k of the current pivot
  auto at = [&](int i, int j) -> P& { return i >= j ? a[(size_t)i * (i + 1) / 2 + j] : a[(size_t)j * (j + 1) / 2 + i]; };
  const int np = n * (n + 1) / 2;
  for (int e = threadIdx.x; e < np; e += blockDim.x) a[e] = P(0);
  __syncthreads();
  // densify: slot q (row i) owns its row; only the lower triangle is stored
  // (the Galerkin operator is symmetric: a_ij = a_ji)
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const int i = slot_row(S, q);
    at(i, i) = diag[i];
    const int sl = q >> 5, lane = q & 31;
    for (int j = 0; j < S.ms_len[sl]; ++j) {
      const int p = S.ms_ptr[sl] + 32 * j + lane;
      const int c = S.mnb[p];
      if (c < i) at(i, c) += coef[p];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < n; ++k) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) ck[j] = at(j, k);
    __syncthreads();
    const P d = ck[k], rd = P(1) / d;
    // rank-1 update of every (i, j) with j <= i, i != k, j != k: warp per row
    for (int i = wid; i < n; i += nw) {
      if (i == k) continue;
      const P f = ck[i] * rd;
      P* row = a + (size_t)i * (i + 1) / 2;
      for (int j = lane; j <= i; j += 32)
        if (j != k) row[j] -= f * ck[j];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) at(j, k) = (j == k) ? -rd : ck[j] * rd;
    __syncthreads();
  }
  // Ai = -(swept matrix), row-major, both triangles
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    Ai[e] = -at(i, j);
  }
}
template <class P>
static size_t dense_inv_sym_smem(int n) { return ((size_t)n * (n + 1) / 2 + n) * sizeof(P); }
constexpr size_t kSmemOptIn = 227 * 1024;

// coarsest solve with the dense inverse: x_i = sum_j Ainv_ij b_j, one warp
// per row (row-major Ainv: coalesced across the lanes, 4 loads in flight per
// lane), shuffle tree; as many blocks as the rows need (was one block: a
// 144-row solve took ~8 us).  accum: x += that (W-cycle second visit).
// large coarsest levels (row stride ld, a multiple of 4): 16-byte loads of
// the inverse's rows, 4 in flight per lane
template <class P>
__global__ void __launch_bounds__(kThreads) k_amg_dense_v4(int n, int ld, const P* __restrict__ Ai,
                                                           const P* __restrict__ b, P* __restrict__ x, int accum,
                                                           const int* done) {
  PDL_ENTRY();
  if (*done) return;
  const int lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
  const int n4 = n / 4;
  for (int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < n; i += nw) {
    const float4* row = reinterpret_cast<const float4*>(Ai + (size_t)i * ld);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    P acc = P(0);
#pragma unroll 4
    for (int j = lane; j < n4; j += 32) {
      const float4 a = __ldg(&row[j]), v = __ldg(&b4[j]);
      acc += a.x * v.x + a.y * v.y + a.z * v.z + a.w * v.w;
    }
    for (int j = 4 * n4 + lane; j < n; j += 32) acc += Ai[(size_t)i * ld + j] * b[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) x[i] = accum ? x[i] + acc : acc;
  }
}
// bf16 copy of the inverse and its mat-vec (16-byte loads = 8 entries, fp32 sums)
__global__ void k_to_bf16(int64_t n, const float* __restrict__ a, __nv_bfloat16* __restrict__ o) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    o[e] = __float2bfloat16_rn(a[e]);
}
__global__ void __launch_bounds__(kThreads) k_amg_dense_bf16(int n, int ld, const __nv_bfloat16* __restrict__ Ai,
                                                             const float* __restrict__ b, float* __restrict__ x,
                                                             int accum, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  const int lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
  const int n8 = n / 8;
  for (int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < n; i += nw) {
    const uint4* row = reinterpret_cast<const uint4*>(Ai + (size_t)i * ld);
    float acc = 0.f;
#pragma unroll 4
    for (int j = lane; j < n8; j += 32) {
      const uint4 raw = __ldg(&row[j]);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(b) + 2 * j);
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(b) + 2 * j + 1);
      const float2 a0 = __bfloat1622float2(h[0]), a1 = __bfloat1622float2(h[1]);
      const float2 a2 = __bfloat1622float2(h[2]), a3 = __bfloat1622float2(h[3]);
      acc += a0.x * b0.x + a0.y * b0.y + a1.x * b0.z + a1.y * b0.w + a2.x * b1.x + a2.y * b1.y + a3.x * b1.z +
             a3.y * b1.w;
    }
    for (int j = 8 * n8 + lane; j < n; j += 32) acc += __bfloat162float(Ai[(size_t)i * ld + j]) * b[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) x[i] = accum ? x[i] + acc : acc;
  }
}
template <class P, class TB, class TO>
__global__ void __launch_bounds__(kThreads) k_amg_dense(int n, const P* __restrict__ Ai, const TB* __restrict__ b,
                                                        TO* __restrict__ x, int accum, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  const int lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < n; i += nw) {
    P acc = P(0);
    const P* row = Ai + (size_t)i * n;
#pragma unroll 4
    for (int j = lane; j < n; j += 32) acc += row[j] * (P)b[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) x[i] = accum ? (TO)(x[i] + (TO)acc) : (TO)acc;
  }
}

// ---- CSR-stream coarse kernels (levels with one thread per row: C5 levels 1-2)
// SELL-32 makes lane i gather row i's j-th neighbour: 32 rows' neighbours per
// request, and 30-35 % padding on aggregation levels; ncu put those levels at
// 4.1-4.6 TB/s of DRAM traffic with L1 and L2 well below their peaks (gather
// latency bound).  Here a warp takes a chunk of whole consecutive rows (<= 32
// rows, <= kCsrChunk entries): the lanes load the chunk's entries in CSR
// order (coalesced coefficients and columns, no padding, neighbouring entries
// of one row gathered by neighbouring lanes), stage coefficient and gathered
// value in shared memory, and lane i then sums row i in its SELL entry order
// (diag x_i first, one FMA per entry): bitwise the SELL kernels' sums.
// c_coef = coef[c_pos] is refreshed with every Galerkin update.
template <class T>
__global__ void k_csr_coef(int64_t n, const int* __restrict__ pos, const T* __restrict__ coef, T* __restrict__ cc) {
  PDL_ENTRY();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    cc[k] = coef[pos[k]];
}
// MODE 0: r = b - A x.  MODE 1: out = x + (b - A x) / d1 (accum: out += that)
template <int MODE, class P>
__global__ void __launch_bounds__(kThreads) k_amg_csr(int nchunk, const int* __restrict__ cptr,
    const int* __restrict__ rp, const int* __restrict__ col, const P* __restrict__ cc, const P* __restrict__ diag,
    const P* __restrict__ il1, const P* __restrict__ x, const P* __restrict__ b, P* __restrict__ out, int accum,
    const int* done) {
  PDL_ENTRY();
  if (*done) return;
  __shared__ P sa[kWarpsPerBlock][kCsrChunk], sx[kWarpsPerBlock][kCsrChunk];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunk; c += nw) {
    const int r0 = __ldg(&cptr[c]), r1 = __ldg(&cptr[c + 1]);
    const int e0 = __ldg(&rp[r0]), e1 = __ldg(&rp[r1]);
    P a[kCsrChunk / 32];
    int cl[kCsrChunk / 32];
#pragma unroll
    for (int u = 0; u < kCsrChunk / 32; ++u) {
      const int k = e0 + lane + 32 * u;
      const bool ok = k < e1;
      a[u] = ok ? __ldg(&cc[k]) : P(0);
      cl[u] = ok ? __ldg(&col[k]) : -1;
    }
    P v[kCsrChunk / 32];
#pragma unroll
    for (int u = 0; u < kCsrChunk / 32; ++u) v[u] = cl[u] >= 0 ? x[cl[u]] : P(0);
#pragma unroll
    for (int u = 0; u < kCsrChunk / 32; ++u)
      if (cl[u] >= 0) { sa[w][lane + 32 * u] = a[u]; sx[w][lane + 32 * u] = v[u]; }
    __syncwarp();
    const int r = r0 + lane;
    if (r < r1) {
      P acc = diag[r] * x[r];
      const int k0 = __ldg(&rp[r]) - e0, k1 = __ldg(&rp[r + 1]) - e0;
      for (int k = k0; k < k1; ++k) acc += sa[w][k] * sx[w][k];
      if (MODE == 0) {
        out[r] = b[r] - acc;
      } else {
        const P z = x[r] + (b[r] - acc) * il1[r];
        out[r] = accum ? out[r] + z : z;
      }
    }
    __syncwarp();
  }
}

// ---- software-pipelined one-thread-per-row residual / smoother (coarse
// levels in natural slot order).  While row q's gathers are in flight the
// thread already loads the next row's first entry batch (columns,
// coefficients) and the row after that's slice metadata, so in steady state
// a row costs one memory round trip (its gathers) plus its entries beyond
// the first 4, instead of three dependent ones.  Same per-row sums in the
// same order as row_part<1> (bitwise).
// MODE 0: r = b - A x.  MODE 1: out = x + (b - A x) / d1 (accum: out += that)
template <int MODE, class P>
__global__ void __launch_bounds__(kThreads) k_amg_rowpf(int n, SellView S, const P* __restrict__ coef,
    const P* __restrict__ diag, const P* __restrict__ il1, const P* __restrict__ x, const P* __restrict__ b,
    P* __restrict__ out, int accum, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  const int st = gridDim.x * blockDim.x;
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  auto meta = [&](int qq, int& ln, int& bs) {
    if (qq < n) { ln = __ldg(&S.ms_len[qq >> 5]); bs = __ldg(&S.ms_ptr[qq >> 5]) + (qq & 31); }
    else { ln = 0; bs = 0; }
  };
  auto batch = [&](int ln, int bs, P (&a)[4], int (&c)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = u < ln;
      a[u] = ok ? __ldg(&coef[bs + 32 * u]) : P(0);
      c[u] = ok ? __ldg(&S.mnb[bs + 32 * u]) : 0;
    }
  };
  int len, base, len_n, base_n;
  P a[4], a_n[4];
  int c[4], c_n[4];
  meta(q, len, base);
  batch(len, base, a, c);
  meta(q + st, len_n, base_n);
  for (; q < n; q += st) {
    P v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = x[c[u]];                 // this row's first gathers
    batch(len_n, base_n, a_n, c_n);                             // next row's first batch
    int len_nn, base_nn;
    meta(q + 2 * st, len_nn, base_nn);                          // the row after's metadata
    P acc = diag[q] * x[q];
    const int j4 = len < 4 ? len : 4;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < j4) acc += a[u] * v[u];
    int j = 4;
    for (; j + 4 <= len; j += 4) {
      P aa[4], vv[4];
      int cc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { aa[u] = __ldg(&coef[base + 32 * (j + u)]); cc[u] = __ldg(&S.mnb[base + 32 * (j + u)]); }
#pragma unroll
      for (int u = 0; u < 4; ++u) vv[u] = x[cc[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += aa[u] * vv[u];
    }
    for (; j < len; ++j) acc += __ldg(&coef[base + 32 * j]) * x[__ldg(&S.mnb[base + 32 * j])];
    if (MODE == 0) {
      out[q] = b[q] - acc;
    } else {
      const P z = x[q] + (b[q] - acc) * il1[q];
      out[q] = accum ? out[q] + z : z;
    }
    len = len_n; base = base_n;
#pragma unroll
    for (int u = 0; u < 4; ++u) { a[u] = a_n[u]; c[u] = c_n[u]; }
    len_n = len_nn; base_n = base_nn;
  }
}

// ---- host launchers for the group-templated kernels (G in {1,2,4,...,32})
#define AMG_G_SWITCH(G, CALL)                      \
  switch (G) {                                     \
    case 2: { constexpr int kG = 2; CALL; } break;   \
    case 4: { constexpr int kG = 4; CALL; } break;   \
    case 8: { constexpr int kG = 8; CALL; } break;   \
    case 16: { constexpr int kG = 16; CALL; } break; \
    case 32: { constexpr int kG = 32; CALL; } break; \
    default: { constexpr int kG = 1; CALL; } break;  \
  }
inline int grid_group(int64_t n, int G) { return grid_for(n * G); }

template <class P, class TB>
static void launch_resid(int G, int n, const SellView& S, const P* coef, const P* diag, const P* x, const TB* b, P* r,
                         const int* done, cudaStream_t s) {
  AMG_G_SWITCH(G, (k_amg_resid<kG, P, TB><<<grid_group(n, kG), kThreads, 0, s>>>(n, S, coef, diag, x, b, r, done)));
}
template <class P>
static void launch_restrict(int G, int nc, const int* mp, const int* mem, const P* rf, P* bc, const int* done,
                            cudaStream_t s) {
  AMG_G_SWITCH(G, (k_amg_restrict<kG, P><<<grid_group(nc, kG), kThreads, 0, s>>>(nc, mp, mem, rf, bc, done)));
}
template <class P>
static void launch_pre_resid(int G, int n, const SellView& S, const P* coef, const P* diag, const P* il1, const P* b,
                             P* x0, P* r, const int* done, cudaStream_t s) {
  AMG_G_SWITCH(G, (k_amg_pre_resid<kG, P><<<grid_group(n, kG), kThreads, 0, s>>>(n, S, coef, diag, il1, b, x0, r,
                                                                                 done)));
}
template <class P>
static void launch_prolong_smooth(int G, int n, const SellView& S, const P* coef, const P* diag, const P* il1,
                                  const int* agg, const P* xc, P w, const P* x0, const P* b, P* out, int accum,
                                  const int* done, cudaStream_t s) {
  AMG_G_SWITCH(G, (k_amg_prolong_smooth<kG, P><<<grid_group(n, kG), kThreads, 0, s>>>(n, S, coef, diag, il1, agg, xc,
                                                                                      w, x0, b, out, accum, done)));
}
template <class P, class TB, class TO>
static void launch_smooth(int G, int n, const SellView& S, const P* coef, const P* diag, const P* il1, const P* x,
                          const TB* b, TO* out, int accum, const int* done, cudaStream_t s) {
  AMG_G_SWITCH(G, (k_amg_smooth<kG, P, TB, TO><<<grid_group(n, kG), kThreads, 0, s>>>(n, S, coef, diag, il1, x, b,
                                                                                      out, accum, done)));
}
// DFVM_AMG_PF=1: the software-pipelined kernels on one-thread-per-row
// coarse levels.  Default off: measured on C5 round 2 at 306.3 / 307.4
// ms/step against 305.1 / 306.6 with the plain kernels
// (profiles/r02_sweep_r2ee_pf.jsonl; 40 registers against 32 — 48 resident
// warps per SM instead of 64 — cancel the deeper pipeline)
static bool amg_pf() {
  const char* e = getenv("DFVM_AMG_PF");
  return e && atoi(e) == 1;
}
// a coarse level's residual / smoother: CSR-stream where the level has it
template <class P>
static void level_resid(const AmgLevelDev<P>& L, const P* x, const P* b, P* r, const int* done, cudaStream_t s) {
  if (L.n_chunk > 0 && L.G == 1)
    k_amg_csr<0, P><<<grid_for((int64_t)L.n_chunk * 32), kThreads, 0, s>>>(L.n_chunk, L.c_ptr, L.c_rp, L.c_col,
                                                                            L.c_coef, L.diag, L.il1, x, b, r, 0, done);
  else if (L.G == 1 && !L.perm && amg_pf())
    k_amg_rowpf<0, P><<<grid_rows(k_amg_rowpf<0, P>, L.n), kThreads, 0, s>>>(L.n, L.sv(), L.coef, L.diag, L.il1, x,
                                                                             b, r, 0, done);
  else
    launch_resid<P, P>(L.G, L.n, L.sv(), L.coef, L.diag, x, b, r, done, s);
}
template <class P>
static void level_smooth(const AmgLevelDev<P>& L, const P* x, const P* b, P* out, int accum, const int* done,
                         cudaStream_t s) {
  if (L.n_chunk > 0 && L.G == 1)
    k_amg_csr<1, P><<<grid_for((int64_t)L.n_chunk * 32), kThreads, 0, s>>>(L.n_chunk, L.c_ptr, L.c_rp, L.c_col,
                                                                            L.c_coef, L.diag, L.il1, x, b, out, accum,
                                                                            done);
  else if (L.G == 1 && !L.perm && amg_pf())
    k_amg_rowpf<1, P><<<grid_rows(k_amg_rowpf<1, P>, L.n), kThreads, 0, s>>>(L.n, L.sv(), L.coef, L.diag, L.il1, x,
                                                                             b, out, accum, done);
  else
    launch_smooth<P, P, P>(L.G, L.n, L.sv(), L.coef, L.diag, L.il1, x, b, out, accum, done, s);
}

// ---- agglomeration of a distributed hierarchy (several ranks)
// this rank's level-ld values in the canonical order of the build (diag,
// owned-column entries, ghost-column entries per row), padded with zeros
template <class P>
__global__ void k_pack_vals(int V, int Vmax, const int* __restrict__ pk, const P* __restrict__ coef,
                            const P* __restrict__ diag, double* __restrict__ out) {
  PDL_ENTRY();
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < Vmax; k += gridDim.x * blockDim.x)
    out[k] = k < V ? (pk[k] >= 0 ? (double)coef[pk[k]] : (double)diag[-1 - pk[k]]) : 0.0;
}
// G0 coefficients / diagonal from the all-gathered values (fixed maps)
template <class P>
__global__ void k_gather_g0(int64_t n_sell, int n, const int* __restrict__ gmap, const int* __restrict__ gdmap,
                            const double* __restrict__ vals, P* __restrict__ coef, P* __restrict__ diag) {
  PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_sell; e += (int64_t)gridDim.x * blockDim.x)
    coef[e] = gmap[e] >= 0 ? (P)vals[gmap[e]] : P(0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) diag[i] = (P)vals[gdmap[i]];
}
template <class P>
__global__ void k_pack_rhs(int n, int nmax, const P* __restrict__ b, double* __restrict__ out, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nmax; i += gridDim.x * blockDim.x)
    out[i] = i < n ? (double)b[i] : 0.0;
}
// G0 right-hand side from the all-gathered padded pieces: rank r's row k -> off[r] + k
template <class P>
__global__ void k_scatter_g0(int nranks, int nmax, const int* __restrict__ cnt, const int* __restrict__ off,
                             const double* __restrict__ all, P* __restrict__ bg, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nranks * nmax; e += gridDim.x * blockDim.x) {
    const int r = e / nmax, k = e - r * nmax;
    if (k < cnt[r]) bg[off[r] + k] = (P)all[e];
  }
}
// this rank's rows of the replicated G0 solution
template <class P>
__global__ void k_extract_g0(int n, int goff, const P* __restrict__ xg, P* __restrict__ x, const int* done) {
  PDL_ENTRY();
  if (*done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = xg[goff + i];
}

// ------------------------------------------------------------ host drivers
// Algorithmic bytes per launch: n rows, Z real off-diagonal
// entries (column 4 B + coefficient pb), vb bytes of the PCG vectors (T),
// pb of the hierarchy (P); gathered values counted once; 4 B/row of SELL
// row metadata on the matrix kernels.
template <class P, class T>
static dfvm_status update(AmgH<P>* A, const T* pcoef, const T* pdiag, cudaStream_t s, int* nl) {
  AmgLevelDev<P>& L0 = A->L[0];
  Prof* pr = A->prof;
  const double pb = sizeof(P), vb = sizeof(T);
  if (std::is_same<P, T>::value) {
    L0.coef = (const P*)pcoef; L0.diag = (const P*)pdiag;
  } else {
    PLAUNCH(pr, "k_amg_cvt", 0, (vb + pb) * (double)L0.n_sell, s,
            (k_amg_cvt<P, T><<<grid_for(L0.n_sell), kThreads, 0, s>>>(L0.n_sell, pcoef, L0.coef_own)));
    PLAUNCH(pr, "k_amg_cvt", 0, (vb + pb) * (double)L0.n, s,
            (k_amg_cvt<P, T><<<grid_for(L0.n), kThreads, 0, s>>>(L0.n, pdiag, L0.diag_own)));
    *nl += 2;
  }
  PLAUNCH(pr, "k_il1", 0, (4 + pb) * (double)L0.nnz + (4 + 2 * pb) * L0.n, s,
          (k_il1<P><<<grid_for(L0.n), kThreads, 0, s>>>(L0.n, L0.sv(), L0.coef, L0.diag, L0.il1)));
  ++*nl;
  for (int l = 1; l < A->nlev; ++l) {
    AmgLevelDev<P>& F = A->L[l - 1];
    AmgLevelDev<P>& C = A->L[l];
    if (A->agglom && l == A->ld + 1) {
      // G0 = every rank's level-ld rows: pack, all-gather, gather into the replicated level
      const int V = A->Vmax, NR = A->m->part.P;
      PLAUNCH(pr, "k_pack_vals", A->ld, 8.0 * V + (4 + pb) * A->Vloc, s,
              (k_pack_vals<P><<<grid_for(V), kThreads, 0, s>>>(A->Vloc, V, A->d_pk, F.coef, F.diag, A->d_vals)));
      if (dfvm_status e = allgather_f64(A->m, A->d_vals, A->d_vals_all, V, s)) return e;
      PLAUNCH(pr, "k_gather_g0", l, (4 + 8 + pb) * (double)C.n_sell + (12 + pb) * C.n, s,
              (k_gather_g0<P><<<grid_for(C.n_sell), kThreads, 0, s>>>(C.n_sell, C.n, A->d_gmap, A->d_gdmap,
                                                                      A->d_vals_all, C.coef_own, C.diag_own)));
      PLAUNCH(pr, "k_il1", l, (4 + pb) * (double)C.nnz + (4 + 2 * pb) * C.n, s,
              (k_il1<P><<<grid_for(C.n), kThreads, 0, s>>>(C.n, C.sv(), C.coef, C.diag, C.il1)));
      (void)NR;
      *nl += 3;
      continue;
    }
    PLAUNCH(pr, "k_gal_off", l, (8 + pb) * (double)C.nnz + (4 + pb) * (double)F.nnz, s,
            (k_gal_off<P><<<grid_for(C.n_sell), kThreads, 0, s>>>(C.n_sell, C.gal_ptr, C.gal_idx, F.coef, C.coef_own)));
    PLAUNCH(pr, "k_gal_diag", l, (8 + pb) * (double)C.n + (4 + pb) * (double)F.n, s,
            (k_gal_diag<P><<<grid_for(C.n), kThreads, 0, s>>>(C.n, C.mem_ptr, C.mem, C.dg_ptr, C.dg_idx, F.diag, F.coef,
                                                               C.diag_own)));
    PLAUNCH(pr, "k_il1", l, (4 + pb) * (double)C.nnz + (4 + 2 * pb) * C.n, s,
            (k_il1<P><<<grid_for(C.n), kThreads, 0, s>>>(C.n, C.sv(), C.coef, C.diag, C.il1)));
    *nl += 3;
    if (C.n_chunk > 0) {
      PLAUNCH(pr, "k_csr_coef", l, (4 + 2 * pb) * (double)C.nnz_csr, s,
              (k_csr_coef<P><<<grid_for(C.nnz_csr), kThreads, 0, s>>>(C.nnz_csr, C.c_pos, C.coef, C.c_coef)));
      ++*nl;
    }
  }
  if (A->ainv) {
    const AmgLevelDev<P>& C = A->L[A->nlev - 1];
    const size_t sm = dense_inv_sym_smem<P>(C.n);
    // DFVM_AMG_INV_EVERY=k (k > 1): the large coarsest inverse is refreshed on
    // every k-th matrix update only (a lagged coarse solve; the Galerkin
    // levels above it are always current, and the stale inverse is still an
    // SPD coarse solve)
    const int inv_every = [] { const char* e = getenv("DFVM_AMG_INV_EVERY"); return e ? std::max(1, atoi(e)) : 1; }();
    if (C.n > kDirectMax && std::is_same<P, float>::value && (A->inv_refreshes++ % inv_every) != 0) {
      DFVM_CUDA(cudaGetLastError());
      return DFVM_OK;
    }
    if (C.n > kDirectMax && std::is_same<P, float>::value) {
      // blocked symmetric sweep (fp32): 4 launches per block of kBlk pivots
      const int n = C.n;
      const bool lower = [] { const char* e = getenv("DFVM_AMG_BLK"); return !(e && e[0] == 'f'); }();
      const bool inv16 = [] { const char* e = getenv("DFVM_AMG_INV16"); return e && atoi(e) == 1; }() &&
                         A->ainv_ld % 8 == 0;
      if (inv16 && !A->ainv16 &&
          dev_alloc_n(&A->ainv16, (size_t)n * A->ainv_ld, nullptr, true) != DFVM_OK)
        return DFVM_E_CUDA;
      if (!A->gj_buf && (dev_alloc_n(&A->gj_buf, 2 * (size_t)n * kBlk + kBlk * kBlk, nullptr, true) != DFVM_OK))
        return DFVM_E_CUDA;
      P* Pb = A->gj_buf;
      P* Sb = A->gj_buf + (size_t)n * kBlk;
      const size_t usm = 2 * (size_t)kBlk * kSP * sizeof(P);
      DFVM_CUDA(cudaFuncSetAttribute(k_blk_update<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
      DFVM_CUDA(cudaFuncSetAttribute(k_blk_update_lo<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
      PLAUNCH(pr, "k_amg_dense_inv", A->nlev - 1, 2 * pb * (double)n * n, s, {
        const int ld = A->ainv_ld;
        cudaMemsetAsync(A->ainv, 0, sizeof(P) * (size_t)n * ld, s);
        const dim3 tg((n + kTN - 1) / kTN, (n + kTM - 1) / kTM);
        if (lower) {
          P* Qb = Pb + (size_t)n * kBlk + kBlk * kBlk;
          k_dense_rows_lower<P><<<grid_for(n), kThreads, 0, s>>>(n, ld, C.sv(), C.coef, C.diag, A->ainv);
          for (int k0 = 0; k0 < n; k0 += kBlk) {
            const int kb = std::min(kBlk, n - k0);
            k_blk_inv_lo<P><<<1, 1024, 0, s>>>(n, ld, k0, kb, A->ainv, Sb);
            k_blk_panel_lo<P><<<std::min(kMaxBlocks, (n + 3) / 4), 256, 0, s>>>(n, ld, k0, kb, A->ainv, Sb, Pb, Qb);
            k_blk_update_lo<P><<<tg, 256, usm, s>>>(n, ld, k0, kb, A->ainv, Pb, Qb);
            k_blk_finish_lo<P><<<grid_for((int64_t)n * kb), kThreads, 0, s>>>(n, ld, k0, kb, A->ainv, Pb, Sb);
          }
          k_mirror_negate<P><<<grid_for((int64_t)n * n), kThreads, 0, s>>>(n, ld, A->ainv);
        } else {
          k_dense_rows_sym<P><<<grid_for(n), kThreads, 0, s>>>(n, ld, C.sv(), C.coef, C.diag, A->ainv);
          for (int k0 = 0; k0 < n; k0 += kBlk) {
            const int kb = std::min(kBlk, n - k0);
            k_blk_inv<P><<<1, 1024, 0, s>>>(n, ld, k0, kb, A->ainv, Sb);
            k_blk_panel<P><<<std::min(kMaxBlocks, (n + 3) / 4), 256, 0, s>>>(n, ld, k0, kb, A->ainv, Sb, Pb);
            k_blk_update<P><<<tg, 256, usm, s>>>(n, ld, k0, kb, A->ainv, Pb);
            k_blk_finish<P><<<grid_for((int64_t)n * kb), kThreads, 0, s>>>(n, ld, k0, kb, A->ainv, Pb, Sb);
          }
          k_negate<P><<<grid_for((int64_t)n * ld), kThreads, 0, s>>>((int64_t)n * ld, A->ainv);
        }
        if (inv16) {
          // ld is a multiple of 4; the bf16 rows need 16-byte alignment too: ld16 = ld rounded to 8
          k_to_bf16<<<grid_for((int64_t)n * ld), kThreads, 0, s>>>((int64_t)n * ld, (const float*)A->ainv, A->ainv16);
        }
      });
      *nl += 2 + 4 * ((n + kBlk - 1) / kBlk);
      DFVM_CUDA(cudaGetLastError());
      return DFVM_OK;
    }
    if (C.n > kDirectMax) {
      // multi-launch Gauss-Jordan (fp64 large coarsest level)
      if (!A->gj_buf && (dev_alloc_n(&A->gj_buf, 2 * (size_t)C.n, nullptr, true) != DFVM_OK)) return DFVM_E_CUDA;
      P* rowk = A->gj_buf;
      P* colk = A->gj_buf + C.n;
      const int gn = grid_for((int64_t)C.n * C.n);
      k_dense_fill<P><<<gn, kThreads, 0, s>>>(C.n, C.sv(), C.coef, C.diag, A->ainv);
      k_dense_rows<P><<<grid_for(C.n), kThreads, 0, s>>>(C.n, C.sv(), C.coef, C.diag, A->ainv);
      for (int k = 0; k < C.n; ++k) {
        k_gj_stage<P><<<grid_for(C.n), kThreads, 0, s>>>(C.n, k, A->ainv, rowk, colk);
        k_gj_update<P><<<gn, kThreads, 0, s>>>(C.n, k, A->ainv, rowk, colk);
      }
      *nl += 2 + 2 * C.n;
      DFVM_CUDA(cudaGetLastError());
      return DFVM_OK;
    }
    const bool sym_on = [] { const char* e = getenv("DFVM_AMG_INV"); return !(e && atoi(e) == 0); }();
    if (sym_on && sm <= kSmemOptIn &&
        cudaFuncSetAttribute(k_amg_dense_inv_sym<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) ==
            cudaSuccess) {
      PLAUNCH(pr, "k_amg_dense_inv", A->nlev - 1, 2 * pb * (double)C.n * C.n, s,
              (k_amg_dense_inv_sym<P><<<1, 1024, sm, s>>>(C.n, C.sv(), C.coef, C.diag, A->ainv)));
    } else {
      cudaGetLastError();
      PLAUNCH(pr, "k_amg_dense_inv", A->nlev - 1, 2 * pb * (double)C.n * C.n, s,
              (k_amg_dense_inv<P><<<1, 1024, 0, s>>>(C.n, C.sv(), C.coef, C.diag, A->ainv)));
    }
    ++*nl;
  }
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

template <class T>
dfvm_status amg_update(Amg<T>* A, const T* pcoef, const T* pdiag, cudaStream_t s, int* nl, Prof* prof) {
  if (A->same) { A->same->prof = prof; return update<T, T>(A->same, pcoef, pdiag, s, nl); }
  A->lo->prof = prof;
  return update<float, T>(A->lo, pcoef, pdiag, s, nl);
}

// Coarsest level l: exact dense solve, or l1-Jacobi sweeps from zero.
// accum (dense solve only, see accum_ok): x += the solution.
template <class P>
static void coarsest(AmgH<P>* A, int l, const P* b, P* x, const int* done, cudaStream_t s, int* nl, bool accum = false) {
  AmgLevelDev<P>& F = A->L[l];
  Prof* pr = A->prof;
  const double pb = sizeof(P), n = F.n;
  if (A->ainv16 && std::is_same<P, float>::value) {
    PLAUNCH(pr, "k_amg_dense", l, 2 * n * n + (accum ? 3 : 2) * pb * n, s,
            (k_amg_dense_bf16<<<grid_for((int64_t)F.n * 32), kThreads, 0, s>>>(F.n, A->ainv_ld, A->ainv16,
                                                                              (const float*)b, (float*)x,
                                                                              accum ? 1 : 0, done)));
    ++*nl;
  } else if (A->ainv && F.n > kDirectMax && std::is_same<P, float>::value) {
    PLAUNCH(pr, "k_amg_dense", l, pb * n * n + (accum ? 3 : 2) * pb * n, s,
            (k_amg_dense_v4<P><<<grid_for((int64_t)F.n * 32), kThreads, 0, s>>>(F.n, A->ainv_ld, A->ainv, b, x,
                                                                                 accum ? 1 : 0, done)));
    ++*nl;
  } else if (A->ainv) {
    PLAUNCH(pr, "k_amg_dense", l, pb * n * n + (accum ? 3 : 2) * pb * n, s,
            (k_amg_dense<P, P, P><<<grid_for((int64_t)F.n * 32), kThreads, 0, s>>>(F.n, A->ainv, b, x, accum ? 1 : 0,
                                                                                    done)));
    ++*nl;
  } else if (F.n <= kCoarseMax) {
    PLAUNCH(pr, "k_amg_coarse", l, (4 + pb) * (double)F.nnz + 4 * pb * n, s,
            (k_amg_coarse<P, P, P><<<1, 1024, 0, s>>>(F.n, F.sv(), F.coef, F.diag, F.il1, b, x,
                                                     A->prm.sweeps, done)));
    ++*nl;
  } else {
    // coarsening stopped above the one-block capacity (stall, or the level
    // cap): the same l1-Jacobi polynomial from zero, multi-block, ping-pong
    // between x and t (an odd sweep count ends in x)
    const int g = grid_for(F.n);
    PLAUNCH(pr, "k_amg_pre", l, 3 * pb * n, s, (k_amg_pre<P, P, P><<<g, kThreads, 0, s>>>(F.n, b, F.il1, x, done)));
    P* cur = x;
    P* nxt = F.t;
    const int sw = A->prm.sweeps + (A->prm.sweeps % 2 == 0 ? 1 : 0);
    for (int it = 1; it < sw; ++it) {
      PLAUNCH(pr, "k_amg_smooth", l, 4 * n + (4 + pb) * (double)F.nnz + 5 * pb * n, s,
              launch_smooth<P, P, P>(F.G, F.n, F.sv(), F.coef, F.diag, F.il1, cur, b, nxt, 0, done, s));
      std::swap(cur, nxt);
    }
    *nl += sw;
  }
}

// Coarse level l >= 1 (no ghost columns): x = M_l^-1 b from a zero guess with
// the fused kernels (launches dominate there): pre-smooth + residual,
// restriction, coarse correction (twice for the W-cycle: the second visit
// solves for the residual of the first), prolongation + post-smooth.  Each
// level's operator is symmetric (adjoint pre/post Jacobi, symmetric coarse
// solve, two successive symmetric corrections 2B - BAB), so the
// preconditioner stays SPD.
// Can level l's cycle add its result into x in place (the last kernel of
// the visit takes an accumulate flag)?  Every non-coarsest level (its
// prolongation + post-smoother) and a dense coarsest solve can.
template <class P>
static bool accum_ok(const AmgH<P>* A, int l) { return l < A->nlev - 1 || A->ainv != nullptr; }

template <class P>
static void cycle_coarse(AmgH<P>* A, int l, const P* b, P* x, const int* done, cudaStream_t s, int* nl,
                         bool accum = false) {
  if (l == A->nlev - 1) { coarsest(A, l, b, x, done, s, nl, accum); return; }
  AmgLevelDev<P>& F = A->L[l];
  AmgLevelDev<P>& C = A->L[l + 1];
  Prof* pr = A->prof;
  const P w = (P)A->prm.omega;
  const double pb = sizeof(P), n = F.n, nc = C.n;
  const int gF = grid_for(F.n);
  const bool fused = l >= A->prm.fused_from;
  if (fused) {
    PLAUNCH(pr, "k_amg_pre_resid", l, 4 * n + (4 + pb) * (double)F.nnz + 5 * pb * n, s,
            launch_pre_resid<P>(F.G, F.n, F.sv(), F.coef, F.diag, F.il1, b, F.t, F.r, done, s));
  } else {
    PLAUNCH(pr, "k_amg_pre", l, 3 * pb * n, s, (k_amg_pre<P, P, P><<<gF, kThreads, 0, s>>>(F.n, b, F.il1, F.t, done)));
    PLAUNCH(pr, "k_amg_resid", l, 4 * n + (4 + pb) * (double)F.nnz + 4 * pb * n, s,
            level_resid<P>(F, F.t, b, F.r, done, s));
    ++*nl;
  }
  PLAUNCH(pr, "k_amg_restrict", l, (4 + pb) * (n + nc), s,
          launch_restrict<P>(C.Gr, C.n, C.mem_ptr, C.mem, F.r, C.b, done, s));
  *nl += 2;
  cycle_coarse(A, l + 1, C.b, C.x, done, s, nl);
  if (A->prm.wcycle && l + 1 < A->nlev - 1 && A->depth(l + 1) <= A->prm.wmax) {
    PLAUNCH(pr, "k_amg_resid", l + 1, 4 * nc + (4 + pb) * (double)C.nnz + 4 * pb * nc, s,
            level_resid<P>(C, C.x, C.b, C.r2, done, s));
    ++*nl;
    if (accum_ok(A, l + 1)) {
      cycle_coarse(A, l + 1, C.r2, C.x, done, s, nl, true);   // x_c += M^-1 r2 in place
    } else {
      cycle_coarse(A, l + 1, C.r2, C.e, done, s, nl);
      PLAUNCH(pr, "k_amg_add", l + 1, 3 * pb * nc, s,
              (k_amg_add<P><<<grid_for(C.n), kThreads, 0, s>>>(C.n, C.e, C.x, done)));
      ++*nl;
    }
  }
  const double acc_b = accum ? pb * n : 0.0;
  if (fused) {
    PLAUNCH(pr, "k_amg_prolong_smooth", l, 4 * n + (4 + pb) * (double)F.nnz + (4 + 5 * pb) * n + pb * nc + acc_b, s,
            launch_prolong_smooth<P>(F.G, F.n, F.sv(), F.coef, F.diag, F.il1, F.agg, C.x, w, F.t, b, x,
                                     accum ? 1 : 0, done, s));
  } else {
    // F.r is free after the restriction: the prolonged t = x0 + w x_c[agg] goes there
    PLAUNCH(pr, "k_amg_prolong", l, (4 + 2 * pb) * n + pb * nc, s,
            (k_amg_prolong<P><<<gF, kThreads, 0, s>>>(F.n, F.agg, C.x, F.t, F.r, w, done)));
    PLAUNCH(pr, "k_amg_smooth", l, 4 * n + (4 + pb) * (double)F.nnz + 5 * pb * n + acc_b, s,
            level_smooth<P>(F, F.r, b, x, accum ? 1 : 0, done, s));
    ++*nl;
  }
  ++*nl;
}

template <class P>
static dfvm_status coarse_correction(AmgH<P>* A, int l, const int* done, cudaStream_t s, int* nl);

// Distributed hierarchy (several ranks): level l >= 1 with ghost aggregates.
// Unfused kernels, a halo exchange before every kernel that gathers
// neighbour values (t, the prolonged r, and the W-cycle's coarse x), the
// coarsest level solved globally (all-gather of the padded right-hand sides,
// every rank applies its rows of the redundant inverse).  Every rank issues
// the same sequence of exchanges (the level count is agreed at build).
template <class P>
static dfvm_status cycle_dist(AmgH<P>* A, int l, const P* b, P* x, const int* done, cudaStream_t s, int* nl) {
  AmgLevelDev<P>& F = A->L[l];
  Prof* pr = A->prof;
  const bool f64 = std::is_same<P, double>::value;
  const double pb = sizeof(P), n = F.n;
  dfvm_status e;
  if (l == A->ld) {
    if (!A->agglom) { coarsest(A, l, b, x, done, s, nl); return DFVM_OK; }
    // agglomerated: all-gather the ranks' right-hand sides into the
    // replicated G0, cycle the replicated hierarchy, take this rank's rows
    AmgLevelDev<P>& G = A->L[l + 1];
    const int NR = A->m->part.P;
    PLAUNCH(pr, "k_pack_rhs", l, (pb + 8) * n, s,
            (k_pack_rhs<P><<<grid_for(A->Nmax), kThreads, 0, s>>>(F.n, A->Nmax, b, A->d_rhs, done)));
    if ((e = allgather_f64(A->m, A->d_rhs, A->d_rhs_all, A->Nmax, s))) return e;
    PLAUNCH(pr, "k_scatter_g0", l + 1, (8 + pb) * (double)G.n, s,
            (k_scatter_g0<P><<<grid_for((int64_t)NR * A->Nmax), kThreads, 0, s>>>(NR, A->Nmax, A->d_cnt, A->d_off,
                                                                                  A->d_rhs_all, G.b, done)));
    cycle_coarse(A, l + 1, G.b, G.x, done, s, nl);
    PLAUNCH(pr, "k_extract_g0", l, 2 * pb * n, s,
            (k_extract_g0<P><<<grid_for(F.n), kThreads, 0, s>>>(F.n, A->goff, G.x, x, done)));
    *nl += 3;
    return DFVM_OK;
  }
  AmgLevelDev<P>& C = A->L[l + 1];
  const P w = (P)A->prm.omega;
  const double nc = C.n;
  const int gF = grid_for(F.n);
  PLAUNCH(pr, "k_amg_pre", l, 3 * pb * n, s, (k_amg_pre<P, P, P><<<gF, kThreads, 0, s>>>(F.n, b, F.il1, F.t, done)));
  if ((e = halo_exchange_lists(A->m, A->halos[l], F.t, 1, f64, s))) return e;
  PLAUNCH(pr, "k_amg_resid", l, 4 * n + (4 + pb) * (double)F.nnz + 4 * pb * n, s,
          launch_resid<P, P>(F.G, F.n, F.sv(), F.coef, F.diag, F.t, b, F.r, done, s));
  PLAUNCH(pr, "k_amg_restrict", l, (4 + pb) * (n + nc), s,
          launch_restrict<P>(C.Gr, C.n, C.mem_ptr, C.mem, F.r, C.b, done, s));
  *nl += 3;
  if ((e = coarse_correction(A, l + 1, done, s, nl))) return e;
  PLAUNCH(pr, "k_amg_prolong", l, (4 + 2 * pb) * n + pb * nc, s,
          (k_amg_prolong<P><<<gF, kThreads, 0, s>>>(F.n, F.agg, C.x, F.t, F.r, w, done)));
  if ((e = halo_exchange_lists(A->m, A->halos[l], F.r, 1, f64, s))) return e;
  PLAUNCH(pr, "k_amg_smooth", l, 4 * n + (4 + pb) * (double)F.nnz + 5 * pb * n, s,
          launch_smooth<P, P, P>(F.G, F.n, F.sv(), F.coef, F.diag, F.il1, F.r, b, x, 0, done, s));
  *nl += 2;
  return DFVM_OK;
}

// The coarse correction of level l (its rhs L[l].b already restricted):
// x_l = M_l^-1 b_l, and for the W-cycle the second visit on the residual
// r2 = b - A x, added.
template <class P>
static dfvm_status coarse_correction(AmgH<P>* A, int l, const int* done, cudaStream_t s, int* nl) {
  AmgLevelDev<P>& C = A->L[l];
  Prof* pr = A->prof;
  const bool f64 = std::is_same<P, double>::value;
  const double pb = sizeof(P), nc = C.n;
  const int gC = grid_for(C.n);
  dfvm_status e;
  if (A->dist) { if ((e = cycle_dist(A, l, C.b, C.x, done, s, nl))) return e; }
  else cycle_coarse(A, l, C.b, C.x, done, s, nl);
  if (A->prm.wcycle && l < A->nlev - 1 && A->depth(l) <= A->prm.wmax) {
    if (A->dist && (e = halo_exchange_lists(A->m, A->halos[l], C.x, 1, f64, s))) return e;
    PLAUNCH(pr, "k_amg_resid", l, 4 * nc + (4 + pb) * (double)C.nnz + 4 * pb * nc, s,
            level_resid<P>(C, C.x, C.b, C.r2, done, s));
    ++*nl;
    if (!A->dist && accum_ok(A, l)) {
      cycle_coarse(A, l, C.r2, C.x, done, s, nl, true);   // x_c += M^-1 r2 in place
    } else {
      if (A->dist) { if ((e = cycle_dist(A, l, C.r2, C.e, done, s, nl))) return e; }
      else cycle_coarse(A, l, C.r2, C.e, done, s, nl);
      PLAUNCH(pr, "k_amg_add", l, 3 * pb * nc, s, (k_amg_add<P><<<gC, kThreads, 0, s>>>(C.n, C.e, C.x, done)));
      ++*nl;
    }
  }
  return DFVM_OK;
}

// Level 0: reads the PCG residual r (type T), writes z (type T); its own
// vectors are in P and carry ghost slices (exchanged before each SpMV).
// Level 0 uses the unfused kernels (measured on B200: the fused versions
// re-gather b/d1 (x0/agg/xc) per neighbour and ran 20 % slower per iteration
// at 50 M rows), and must with several ranks (x0 and t need a halo exchange).
template <class P, class T>
static dfvm_status cycle0(AmgH<P>* A, const T* r, T* z, const int* done, cudaStream_t s, int* nl, cudaEvent_t* ev,
                          const KDot* dot, bool pre_done, bool* dot_done) {
  if (dot_done) *dot_done = false;
  AmgLevelDev<P>& F = A->L[0];
  Prof* pr = A->prof;
  const bool f64 = std::is_same<P, double>::value;
  const double pb = sizeof(P), vb = sizeof(T), n = F.n;
  dfvm_status e;
  if (A->nlev == 1) {
    if (A->m->part.P > 1 || F.n > kCoarseMax) {
      // single level with ghost columns (or too large for the one-block
      // solve): one l1-Jacobi step.  With several ranks the two level-0 halo
      // exchanges of the multi-level cycle are still made, so every rank
      // issues the same communication sequence whatever its level count
      // (a rank whose block did not coarsen must not desynchronise the
      // send / recv pairing of its peers).
      PLAUNCH(pr, "k_amg_pre", 0, (2 * vb + pb) * n, s,
              (k_amg_pre<P, T, T><<<grid_for(F.n), kThreads, 0, s>>>(F.n, r, F.il1, z, done)));
      if ((e = halo_exchange_p(A->m, F.x, 1, f64, s)) || (e = halo_exchange_p(A->m, F.t, 1, f64, s))) return e;
    } else {
      PLAUNCH(pr, "k_amg_coarse", 0, (4 + pb) * (double)F.nnz + 4 * pb * n, s,
              (k_amg_coarse<P, T, T><<<1, 1024, 0, s>>>(F.n, F.sv(), F.coef, F.diag, F.il1, r, z,
                                                       A->prm.sweeps, done)));
    }
    ++*nl;
    return DFVM_OK;
  }
  AmgLevelDev<P>& C = A->L[1];
  const double nc = C.n;
  const int g0 = grid_for(F.n);
  if (!pre_done) {
    PLAUNCH(pr, "k_amg_pre", 0, (vb + 2 * pb) * n, s,
            (k_amg_pre<P, T, P><<<g0, kThreads, 0, s>>>(F.n, r, F.il1, F.x, done)));
    ++*nl;
  }
  if ((e = halo_exchange_p(A->m, F.x, 1, f64, s))) return e;
  if (ev) record_event(ev[0], s);
  PLAUNCH(pr, "k_amg_resid", 0, 4 * n + (4 + pb) * (double)F.nnz + (3 * pb + vb) * n, s,
          launch_resid<P, T>(F.G, F.n, F.sv(), F.coef, F.diag, F.x, r, F.r, done, s));
  if (ev) record_event(ev[1], s);
  PLAUNCH(pr, "k_amg_restrict", 0, (4 + pb) * (n + nc), s,
          launch_restrict<P>(C.Gr, C.n, C.mem_ptr, C.mem, F.r, C.b, done, s));
  *nl += 2;
  if ((e = coarse_correction(A, 1, done, s, nl))) return e;
  PLAUNCH(pr, "k_amg_prolong", 0, (4 + 2 * pb) * n + pb * nc, s,
          (k_amg_prolong<P><<<g0, kThreads, 0, s>>>(F.n, F.agg, C.x, F.x, F.t, (P)A->prm.omega, done)));
  if ((e = halo_exchange_p(A->m, F.t, 1, f64, s))) return e;
  if (ev) record_event(ev[2], s);
  if (dot) {
    PLAUNCH(pr, "k_amg_smooth_dot", 0, 4 * n + (4 + pb) * (double)F.nnz + (3 * pb + 2 * vb) * n, s,
            (k_amg_smooth_dot<P, T><<<g0, kThreads, 0, s>>>(F.n, F.sv(), F.coef, F.diag, F.il1,
                                                            F.t, r, z, done, dot->partials, dot->ticket, dot->ctl,
                                                            dot->red, dot->kind)));
    if (dot_done) *dot_done = true;
  } else {
    PLAUNCH(pr, "k_amg_smooth", 0, 4 * n + (4 + pb) * (double)F.nnz + (3 * pb + 2 * vb) * n, s,
            launch_smooth<P, T, T>(F.G, F.n, F.sv(), F.coef, F.diag, F.il1, F.t, r, z, 0, done, s));
  }
  if (ev) record_event(ev[3], s);
  *nl += 2;
  return DFVM_OK;
}

// z = M^-1 r; skipped on the device when *done is set
template <class T>
dfvm_status amg_apply(Amg<T>* A, const T* r, T* z, const int* done, cudaStream_t s, int* nl, cudaEvent_t* ev,
                      Prof* prof, const KDot* dot, bool pre_done, bool* dot_done) {
  dfvm_status e;
  if (A->same) { A->same->prof = prof; e = cycle0<T, T>(A->same, r, z, done, s, nl, ev, dot, pre_done, dot_done); }
  else { A->lo->prof = prof; e = cycle0<float, T>(A->lo, r, z, done, s, nl, ev, dot, pre_done, dot_done); }
  if (e) return e;
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

template <class T>
void amg_level0_pre(Amg<T>* A, void** x0, const void** il1, int* p_bytes) {
  *x0 = nullptr; *il1 = nullptr; *p_bytes = 0;
  if (A->same && A->same->nlev > 1) { *x0 = A->same->L[0].x; *il1 = A->same->L[0].il1; *p_bytes = sizeof(T); }
  if (A->lo && A->lo->nlev > 1) { *x0 = A->lo->L[0].x; *il1 = A->lo->L[0].il1; *p_bytes = 4; }
}

template <class T>
int amg_level_nnz(const Amg<T>* A, int64_t* nnz) {
  if (A->same) { for (int l = 0; l < A->same->nlev; ++l) nnz[l] = A->same->L[l].nnz; return A->same->nlev; }
  for (int l = 0; l < A->lo->nlev; ++l) nnz[l] = A->lo->L[l].nnz;
  return A->lo->nlev;
}

#define INST(T)                                                                           \
  template dfvm_status amg_create<T>(dfvm_mesh*, const DevMesh<T>&, bool, Amg<T>**, cudaStream_t); \
  template void amg_destroy<T>(Amg<T>*);                                                  \
  template int amg_levels<T>(const Amg<T>*, int*);                                        \
  template dfvm_status amg_update<T>(Amg<T>*, const T*, const T*, cudaStream_t, int*, Prof*); \
  template dfvm_status amg_apply<T>(Amg<T>*, const T*, T*, const int*, cudaStream_t, int*, cudaEvent_t*, Prof*,     \
                                    const KDot*, bool, bool*);                                                   \
  template void amg_level0_pre<T>(Amg<T>*, void**, const void**, int*);                                          \
  template int amg_level_nnz<T>(const Amg<T>*, int64_t*);
INST(double)
INST(float)

}  // namespace dfvm
