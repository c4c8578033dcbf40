// internal.h — libdfvm internal data structures (host side + device views).
//
// Layout in HBM: after RCM renumbering and the
// (owner, neighbour) face re-sort, each rank holds
//   cells   [n_own owned | n_ghost ghosts]   vectors AoS [n][3]
//   faces   [F_l internal | B_l non-empty boundary | E_l empty]
//   fgeo[F_l]  {Sx, Sy, Sz, w}        32 B (fp64) / 16 B (fp32) records
//   fcor[F_l]  {kx, ky, kz, delta}
//   fcell[F_l] {owner, neighbour}     local cell ids
//   bgeo[B_l]  {Sx, Sy, Sz, delta_b}, bcell[B_l]
//   SELL-32 incidence lists per owned row (one warp = 32 consecutive rows,
//   entry k of lane l at slice_ptr[s] + 32 k + l):
//     inc  (int2 {a, b}): internal entries first (ascending face), then
//          boundary entries; a = f (cell is owner) or ~f (cell is
//          neighbour) with b = neighbour cell; boundary: a = boundary face,
//          b = -1; padding b = -2
//     mnb  (int):  internal entries only, the neighbour cell (matrix layout
//          for PCG / momentum coefficients; padding -> the row itself with
//          coefficient 0)
#pragma once
#include <cstdint>
#include <string>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>

#include "dfvm.h"

namespace dfvm {

// ------------------------------------------------------------ errors
void set_error(dfvm_status code, const std::string& msg, int64_t index = -1);
dfvm_status cuda_error(cudaError_t e, const char* where);
#define DFVM_CUDA(call)                                                     \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess) return ::dfvm::cuda_error(e_, #call);            \
  } while (0)

void count_launch(int n = 1);

// device workspace (alloc.cpp): through the caller's allocator if one is set
// (dfvm_set_allocator), else cudaMallocAsync; stream-ordered zero-fill
dfvm_status dev_alloc(void** p, size_t bytes, cudaStream_t s, bool zero);
void dev_free(void* p, cudaStream_t s);
int64_t dev_live_bytes();
template <class U>
inline dfvm_status dev_alloc_n(U** p, size_t n, cudaStream_t s, bool zero) {
  void* q = nullptr;
  dfvm_status st = dev_alloc(&q, (n ? n : 1) * sizeof(U), s, zero);
  *p = (U*)q;
  return st;
}

// ------------------------------------------------------------ host mesh
struct HostMesh {
  int64_t N = 0, F = 0, NF = 0;
  std::vector<int32_t> pkind;
  std::vector<int64_t> pstart, pn;
  std::vector<std::string> pname;
  int nonorth = DFVM_NONORTH_OVERRELAXED;
  // original-order fp64 geometry (O-1)
  std::vector<double> Sf0, xf0, xc0, V0;
  // maps
  std::vector<int32_t> new_of_old, old_of_new;      // cells
  std::vector<int32_t> fnew_of_old, fold_of_new;    // faces
  std::vector<int8_t> flip_old;                     // internal faces, by old index
  // new-order faces
  std::vector<int32_t> own, nb;                     // [F] internal (own < nb)
  std::vector<int32_t> bown;                        // [NF-F] boundary owner (new id)
  std::vector<int32_t> bpatch;                      // [NF-F]
  // global CSR of internal incidences (new numbering)
  std::vector<int32_t> row_ptr, inc_face, inc_nb;
  // new-order coefficients (O-3)
  std::vector<double> w, delta, k, delta_b;         // [F], [F], [3F], [NF-F]
  int64_t n_clamped = 0, bw_before = 0, bw_after = 0;
  bool is_empty_new(int64_t fnew) const { return fnew >= F && pkind[bpatch[fnew - F]] == DFVM_PATCH_EMPTY; }
};

struct Part {
  int P = 1, rank = 0;
  int64_t lo = 0, hi = 0, n_own = 0, n_ghost = 0;
  std::vector<int32_t> ghost_gid, ghost_peer, send_gid, send_peer;
  std::vector<int32_t> peers;                       // ascending
  std::vector<int64_t> peer_ghost_off, peer_send_off; // per peer, [n_peers + 1]
  std::vector<int32_t> lf_gid, lf_own, lf_nb;        // local internal faces
  std::vector<int32_t> lb_gid, lb_cell;              // local boundary faces (non-empty then empty)
  int64_t n_lb = 0, n_le = 0;
  std::vector<int32_t> cell_gid;                     // local cell -> global new id
};

// validation + geometry + renumbering (host_mesh.cpp)
dfvm_status build_host_mesh(HostMesh& H, const double* points, int64_t n_points, const int64_t* fo,
                            const int32_t* fp, int64_t nf, const int32_t* owner, const int32_t* neigh, int64_t F,
                            const dfvm_patch_desc* patches, int32_t np, int nonorth, int rcm);
void build_part(const HostMesh& H, int P, int rank, Part& part);

// ------------------------------------------------------------ device mesh
template <class T> struct alignas(4 * sizeof(T)) V4 { T x, y, z, w; };

template <class T>
struct DevMesh {
  int n_own = 0, n_cells = 0, F = 0, B = 0, E = 0;
  int n_slices = 0, max_row = 0;
  V4<T>* fgeo = nullptr;   // [F]
  V4<T>* fcor = nullptr;   // [F]
  T* fw = nullptr;         // [F] copy of the weights (kernels that need w alone read 8 B, not a 32 B record)
  T* fwd = nullptr;        // [2F] {w, delta} per face (k_pcoef: one 16 B load instead of 8 B + a 32 B record)
  V4<T>* fkw = nullptr;    // [F] {k_x, k_y, k_z, w} (k_prhs: one 32 B load instead of 8 B + a 32 B record)
  int2* fcell = nullptr;   // [F]
  V4<T>* bgeo = nullptr;   // [B]
  int* bcell = nullptr;    // [B]
  T* vol = nullptr;        // [n_own]
  int* sl_ptr = nullptr;   // [n_slices + 1] (full incidence SELL)
  int* sl_len = nullptr;   // [n_slices]
  int2* inc = nullptr;
  int* ms_ptr = nullptr;   // matrix SELL (internal only)
  int* ms_len = nullptr;
  int* mnb = nullptr;
  int64_t n_inc = 0, n_minc = 0;
  int64_t nnz = 0;         // real matrix entries of the owned rows (= 2F at P = 1; algorithmic bytes)
};

struct Comm;

// halo lists of one partitioned vector space (comm.cpp halo_exchange_lists)
struct HaloLists {
  bool ready = false;
  int64_t n_own = 0;
  std::vector<int32_t> peers;               // ascending
  std::vector<int64_t> send_off, ghost_off; // per peer, [n_peers + 1]
  std::vector<int32_t> send_idx;            // owned local rows, per peer ascending
  int32_t* d_send_idx = nullptr;
  void* d_send = nullptr;
  size_t buf_bytes = 0;
};

}  // namespace dfvm

// opaque ABI objects
struct dfvm_mesh {
  dfvm::HostMesh H;
  dfvm::Part part;
  int precision = DFVM_F64;
  int device = 0;
  dfvm::DevMesh<double> d64;
  dfvm::DevMesh<float> d32;
  std::vector<void*> allocations;
  int64_t device_bytes = 0;
  double host_seconds = 0;
  bool host_only = false;
  // host copy of the matrix SELL structure (AMG hierarchy setup)
  std::vector<int> h_ms_ptr, h_ms_len, h_mnb;
  dfvm_comm* comm = nullptr;
  // lazily built device maps for device-side import/export
  int32_t* d_cell_orig = nullptr;   // [n_cells] original id of local cell
  int32_t* d_face_orig = nullptr;   // [n_faces_local] original face id, sign-flip flag in bit 31
  // halo of the cells (P > 1)
  dfvm::HaloLists halo0;
  // persistent device staging buffer of host<->device field import/export
  // (grown on demand, guarded: one import/export at a time per mesh)
  void* d_stage = nullptr;
  size_t stage_bytes = 0;
  std::mutex stage_mu;
  int64_t n_faces_local() const { return (int64_t)part.lf_gid.size() + (int64_t)part.lb_gid.size(); }
};

struct dfvm_field {
  dfvm_mesh* m = nullptr;
  void* ptr = nullptr;
  int32_t loc = DFVM_CELLS;   // 0 cells, 1 faces (unoriented values), 2 face flux (oriented)
  int32_t n_comp = 1;
  bool owned = false;
  int64_t count() const {
    return loc == DFVM_CELLS ? m->part.n_own + m->part.n_ghost : m->n_faces_local();
  }
};

struct dfvm_bcs {
  dfvm_mesh* m = nullptr;
  // host specs [field][patch]
  std::vector<dfvm_bc_desc> spec[3];
  std::vector<uint8_t> set[3];
  // device per-boundary-face kind (0 fixed, 1 zeroGradient) and values
  uint8_t* d_kind[3] = {nullptr, nullptr, nullptr};
  void* d_val[3] = {nullptr, nullptr, nullptr};
  bool dirty[3] = {true, true, true};
  std::vector<uint8_t> h_kind[3];
  std::vector<double> h_val[3];
  std::vector<char> h_valT[3];  // staging in mesh precision
  // time-varying multipliers (A-41), per field slot and patch: nh < 0 = steady
  struct Wave { int nh = -1; double period = 1, a[17] = {0}, b[17] = {0}; };
  std::vector<Wave> wave[3];
  double t_eval = 0;
  void* d_base[3] = {nullptr, nullptr, nullptr};   // steady values (mesh precision) of wave slots
  int8_t* d_wid[3] = {nullptr, nullptr, nullptr};  // per boundary face: patch-wave index or -1
  std::vector<int> wave_patches[3];                // patches with a wave, in index order
};

namespace dfvm {
int field_slot(char fld);  // 'U' 0, 'p' 1, 's' 2, else -1
dfvm_status bcs_device(dfvm_bcs* b, int slot, cudaStream_t s);  // validate + upload
dfvm_status bcs_time(dfvm_bcs* b, int slot, double t, cudaStream_t s);  // apply waveforms at time t
constexpr int kMaxWaves = 16;
template <class T> struct WaveG { T g[kMaxWaves]; };
template <class T>
void launch_bc_wave(T* val, const T* base, const int8_t* wid, int64_t B, int nc, const WaveG<T>& g, cudaStream_t s);
}
