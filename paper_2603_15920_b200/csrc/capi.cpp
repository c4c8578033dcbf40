// capi.cpp — C ABI of libdfvm (include/dfvm.h): errors, mesh creation and
// upload (SELL-32 layout), fields, boundary conditions and the operator
// entry points.  The solver entry points live in solver.cu.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>
#include <atomic>

#include "internal.h"
#include "launch.h"

namespace dfvm {

static thread_local std::string g_msg;
static thread_local int64_t g_index = -1;
static std::atomic<int64_t> g_launches{0};

void set_error(dfvm_status code, const std::string& msg, int64_t index) {
  (void)code;
  g_msg = msg;
  g_index = index;
}
dfvm_status cuda_error(cudaError_t e, const char* where) {
  set_error(e == cudaErrorMemoryAllocation ? DFVM_E_OOM : DFVM_E_CUDA,
            std::string(where) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? DFVM_E_OOM : DFVM_E_CUDA;
}
void count_launch(int n) { g_launches += n; }

int field_slot(char fld) { return fld == 'U' ? 0 : fld == 'p' ? 1 : fld == 's' ? 2 : -1; }

// halo exchange hook (comm.cpp)
dfvm_status halo_exchange(dfvm_mesh* m, void* data, int nc, cudaStream_t s);

template <class T>
static dfvm_status dalloc(dfvm_mesh* m, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  void* q = nullptr;
  if (dfvm_status st = dev_alloc(&q, count * sizeof(T), nullptr, false)) return st;   // legacy stream, before the uploads
  m->allocations.push_back(q);
  m->device_bytes += (int64_t)(count * sizeof(T));
  *p = (T*)q;
  return DFVM_OK;
}
template <class T>
static dfvm_status upload(dfvm_mesh* m, T** p, const std::vector<T>& h) {
  if (dfvm_status st = dalloc(m, p, h.size())) return st;
  if (!h.empty()) DFVM_CUDA(cudaMemcpy(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return DFVM_OK;
}

// Build the SELL-32 incidence layouts and the face / cell records of this
// rank's part, convert to precision T and upload.
template <class T>
static dfvm_status upload_mesh(dfvm_mesh* m, DevMesh<T>& D) {
  const HostMesh& H = m->H;
  const Part& P = m->part;
  const int64_t n_own = P.n_own, F_l = (int64_t)P.lf_gid.size();
  D.n_own = (int)n_own;
  D.n_cells = (int)(P.n_own + P.n_ghost);
  D.F = (int)F_l;
  D.B = (int)P.n_lb;
  D.E = (int)P.n_le;
  // per-row incidence lists (CSR first)
  std::vector<int32_t> cnt(n_own + 1, 0), mcnt(n_own + 1, 0);
  for (int64_t i = 0; i < F_l; ++i) {
    if (P.lf_own[i] < n_own) { cnt[P.lf_own[i] + 1]++; mcnt[P.lf_own[i] + 1]++; }
    if (P.lf_nb[i] < n_own) { cnt[P.lf_nb[i] + 1]++; mcnt[P.lf_nb[i] + 1]++; }
  }
  for (int64_t b = 0; b < P.n_lb; ++b) cnt[P.lb_cell[b] + 1]++;
  for (int64_t r = 0; r < n_own; ++r) { cnt[r + 1] += cnt[r]; mcnt[r + 1] += mcnt[r]; }
  std::vector<int2> rows(cnt[n_own]);
  {
    std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < F_l; ++i) {
      const int32_t o = P.lf_own[i], n = P.lf_nb[i];
      if (o < n_own) rows[pos[o]++] = int2{(int)i, n};
      if (n < n_own) rows[pos[n]++] = int2{~(int)i, o};
    }
    for (int64_t b = 0; b < P.n_lb; ++b) rows[pos[P.lb_cell[b]]++] = int2{(int)b, -1};
  }
  const int64_t S = (n_own + 31) / 32;
  D.n_slices = (int)S;
  std::vector<int> sl_ptr(S + 1, 0), sl_len(S, 0), ms_ptr(S + 1, 0), ms_len(S, 0);
  int max_row = 0;
  for (int64_t s = 0; s < S; ++s) {
    int L = 0, ML = 0;
    for (int64_t r = s * 32; r < std::min<int64_t>(n_own, s * 32 + 32); ++r) {
      L = std::max(L, cnt[r + 1] - cnt[r]);
      ML = std::max(ML, mcnt[r + 1] - mcnt[r]);
    }
    max_row = std::max(max_row, L);
    sl_len[s] = L; ms_len[s] = ML;
    if ((int64_t)sl_ptr[s] + 32LL * L >= (1LL << 31)) { set_error(DFVM_E_INVALID_ARG, "SELL layout exceeds int32"); return DFVM_E_INVALID_ARG; }
    sl_ptr[s + 1] = sl_ptr[s] + 32 * L;
    ms_ptr[s + 1] = ms_ptr[s] + 32 * ML;
  }
  D.max_row = max_row;
  std::vector<int2> inc(sl_ptr[S], int2{0, -2});
  std::vector<int> mnb(ms_ptr[S], 0);
  for (int64_t s = 0; s < S; ++s)
    for (int lane = 0; lane < 32; ++lane) {
      const int64_t r = s * 32 + lane;
      if (r >= n_own) continue;
      int mj = 0;
      for (int j = 0; j < cnt[r + 1] - cnt[r]; ++j) {
        const int2 e = rows[cnt[r] + j];
        inc[sl_ptr[s] + 32 * j + lane] = e;
        if (e.y >= 0) mnb[ms_ptr[s] + 32 * (mj++) + lane] = e.y;
      }
      for (; mj < ms_len[s]; ++mj) mnb[ms_ptr[s] + 32 * mj + lane] = (int)r;   // padding: self, coef 0
    }
  D.n_inc = (int64_t)inc.size();
  D.n_minc = (int64_t)mnb.size();
  D.nnz = mcnt[n_own];
  if (m->h_ms_ptr.empty()) { m->h_ms_ptr = ms_ptr; m->h_ms_len = ms_len; m->h_mnb = mnb; }   // AMG setup
  // face records
  std::vector<V4<T>> fgeo(F_l), fcor(F_l), fkw(F_l), bgeo(P.n_lb);
  std::vector<T> fw(F_l), fwd(2 * F_l);
  std::vector<int2> fcell(F_l);
  std::vector<int> bcell(P.n_lb);
  for (int64_t i = 0; i < F_l; ++i) {
    const int64_t k = P.lf_gid[i];
    const int32_t fo = H.fold_of_new[k];
    const double sg = H.flip_old[fo] ? -1.0 : 1.0;
    fgeo[i] = V4<T>{(T)(sg * H.Sf0[3 * fo]), (T)(sg * H.Sf0[3 * fo + 1]), (T)(sg * H.Sf0[3 * fo + 2]), (T)H.w[k]};
    fcor[i] = V4<T>{(T)H.k[3 * k], (T)H.k[3 * k + 1], (T)H.k[3 * k + 2], (T)H.delta[k]};
    fkw[i] = V4<T>{(T)H.k[3 * k], (T)H.k[3 * k + 1], (T)H.k[3 * k + 2], (T)H.w[k]};
    fw[i] = (T)H.w[k];
    fwd[2 * i] = (T)H.w[k];
    fwd[2 * i + 1] = (T)H.delta[k];
    fcell[i] = int2{P.lf_own[i], P.lf_nb[i]};
  }
  for (int64_t b = 0; b < P.n_lb; ++b) {
    const int64_t k = P.lb_gid[b];
    const int32_t fo = H.fold_of_new[k];
    bgeo[b] = V4<T>{(T)H.Sf0[3 * fo], (T)H.Sf0[3 * fo + 1], (T)H.Sf0[3 * fo + 2], (T)H.delta_b[k - H.F]};
    bcell[b] = P.lb_cell[b];
  }
  std::vector<T> vol(n_own);
  for (int64_t i = 0; i < n_own; ++i) vol[i] = (T)H.V0[H.old_of_new[P.cell_gid[i]]];
  dfvm_status st;
  if ((st = upload(m, &D.fgeo, fgeo)) || (st = upload(m, &D.fcor, fcor)) || (st = upload(m, &D.fw, fw)) || (st = upload(m, &D.fwd, fwd)) || (st = upload(m, &D.fkw, fkw)) ||
      (st = upload(m, &D.fcell, fcell)) ||
      (st = upload(m, &D.bgeo, bgeo)) || (st = upload(m, &D.bcell, bcell)) || (st = upload(m, &D.vol, vol)) ||
      (st = upload(m, &D.sl_ptr, sl_ptr)) || (st = upload(m, &D.sl_len, sl_len)) || (st = upload(m, &D.inc, inc)) ||
      (st = upload(m, &D.ms_ptr, ms_ptr)) || (st = upload(m, &D.ms_len, ms_len)) || (st = upload(m, &D.mnb, mnb)))
    return st;
  // import / export maps
  std::vector<int32_t> corig(P.n_own + P.n_ghost), forig(m->n_faces_local());
  for (size_t i = 0; i < corig.size(); ++i) corig[i] = H.old_of_new[P.cell_gid[i]];
  for (int64_t i = 0; i < F_l; ++i) {
    const int32_t fo = H.fold_of_new[P.lf_gid[i]];
    forig[i] = H.flip_old[fo] ? ~fo : fo;
  }
  for (size_t b = 0; b < P.lb_gid.size(); ++b) forig[F_l + b] = H.fold_of_new[P.lb_gid[b]];
  if ((st = upload(m, &m->d_cell_orig, corig)) || (st = upload(m, &m->d_face_orig, forig))) return st;
  return DFVM_OK;
}

dfvm_status bcs_device(dfvm_bcs* b, int slot, cudaStream_t s) {
  dfvm_mesh* m = b->m;
  const HostMesh& H = m->H;
  const Part& P = m->part;
  for (size_t p = 0; p < H.pkind.size(); ++p)
    if (H.pkind[p] != DFVM_PATCH_EMPTY && !b->set[slot][p]) {
      set_error(DFVM_E_MISSING_BC, "non-empty patch '" + H.pname[p] + "' has no boundary condition for this field",
                (int64_t)p);
      return DFVM_E_MISSING_BC;
    }
  if (!b->dirty[slot]) return DFVM_OK;
  const int nc = slot == 0 ? 3 : 1;
  const int64_t B = P.n_lb;
  b->h_kind[slot].assign(std::max<int64_t>(B, 1), 1);
  b->h_val[slot].assign(std::max<int64_t>(B * nc, 1), 0.0);
  for (int64_t i = 0; i < B; ++i) {
    const int64_t k = P.lb_gid[i];
    const int p = H.bpatch[k - H.F];
    const dfvm_bc_desc& d = b->spec[slot][p];
    const int32_t fo = H.fold_of_new[k];
    switch (d.kind) {
      case DFVM_BC_FIXED_VALUE:
        b->h_kind[slot][i] = 0;
        for (int c = 0; c < nc; ++c) b->h_val[slot][i * nc + c] = d.value[c];
        break;
      case DFVM_BC_PARABOLIC: {
        const double* S = &H.Sf0[3 * fo];
        const double* x = &H.xf0[3 * fo];
        const double r0 = x[0] - d.center[0], r1 = x[1] - d.center[1], r2 = x[2] - d.center[2];
        const double A = std::sqrt(S[0] * S[0] + S[1] * S[1] + S[2] * S[2]);
        const double mag = d.u_max * (1.0 - (r0 * r0 + r1 * r1 + r2 * r2) / (d.radius * d.radius));
        b->h_kind[slot][i] = 0;
        for (int c = 0; c < 3; ++c) b->h_val[slot][i * 3 + c] = -mag * S[c] / A;
        break;
      }
      case DFVM_BC_WINDKESSEL:
        b->h_kind[slot][i] = 0;
        b->h_val[slot][i] = 0.0;   // set on device by the Windkessel kernel each corrector
        break;
      default:
        b->h_kind[slot][i] = 1;
    }
  }
  const size_t bytesT = m->precision == DFVM_F64 ? 8 : 4;
  const size_t nval = b->h_val[slot].size();
  b->h_valT[slot].resize(nval * bytesT);
  for (size_t i = 0; i < nval; ++i) {
    if (bytesT == 8) std::memcpy(&b->h_valT[slot][8 * i], &b->h_val[slot][i], 8);
    else { float v = (float)b->h_val[slot][i]; std::memcpy(&b->h_valT[slot][4 * i], &v, 4); }
  }
  // stream-ordered on the caller's stream: the kernels that read the values
  // follow on the same stream (the host vectors are members: they outlive
  // the copies)
  dfvm_status st;
  if (!b->d_kind[slot]) {
    if ((st = dev_alloc_n(&b->d_kind[slot], b->h_kind[slot].size(), s, false)) ||
        (st = dev_alloc(&b->d_val[slot], nval * bytesT, s, false)))
      return st;
  }
  DFVM_CUDA(cudaMemcpyAsync(b->d_kind[slot], b->h_kind[slot].data(), b->h_kind[slot].size(), cudaMemcpyHostToDevice, s));
  DFVM_CUDA(cudaMemcpyAsync(b->d_val[slot], b->h_valT[slot].data(), nval * bytesT, cudaMemcpyHostToDevice, s));
  // time-varying patches (A-41): steady base values + per-face wave index
  b->wave_patches[slot].clear();
  for (size_t p = 0; p < H.pkind.size(); ++p)
    if (H.pkind[p] != DFVM_PATCH_EMPTY && b->wave[slot][p].nh >= 0) {
      const int k = b->spec[slot][p].kind;
      if (k != DFVM_BC_FIXED_VALUE && k != DFVM_BC_PARABOLIC) {
        set_error(DFVM_E_INVALID_ARG, "time-varying waveform on patch '" + H.pname[p] +
                  "' which is not fixed-value / parabolic", (int64_t)p);
        return DFVM_E_INVALID_ARG;
      }
      b->wave_patches[slot].push_back((int)p);
    }
  if (!b->wave_patches[slot].empty()) {
    if ((int)b->wave_patches[slot].size() > kMaxWaves) {
      set_error(DFVM_E_INVALID_ARG, "more than 16 time-varying patches for one field");
      return DFVM_E_INVALID_ARG;
    }
    std::vector<int8_t> wid(std::max<int64_t>(B, 1), -1);
    for (int64_t i = 0; i < B; ++i) {
      const int p = H.bpatch[P.lb_gid[i] - H.F];
      for (size_t j = 0; j < b->wave_patches[slot].size(); ++j)
        if (b->wave_patches[slot][j] == p) wid[i] = (int8_t)j;
    }
    if (!b->d_base[slot]) {
      if ((st = dev_alloc(&b->d_base[slot], nval * bytesT, s, false)) ||
          (st = dev_alloc_n(&b->d_wid[slot], wid.size(), s, false)))
        return st;
    }
    DFVM_CUDA(cudaMemcpyAsync(b->d_base[slot], b->h_valT[slot].data(), nval * bytesT, cudaMemcpyHostToDevice, s));
    DFVM_CUDA(cudaMemcpyAsync(b->d_wid[slot], wid.data(), wid.size(), cudaMemcpyHostToDevice, s));
    DFVM_CUDA(cudaStreamSynchronize(s));   // `wid` is a local vector
  }
  b->dirty[slot] = false;
  if (!b->wave_patches[slot].empty()) count_launch();
  return bcs_time(b, slot, b->t_eval, s);
}

// g(t) of a patch wave: a0 + sum_k a_k cos(2 pi k t/T) + b_k sin(2 pi k t/T), ascending k (A-41)
static double wave_g(const dfvm_bcs::Wave& w, double t) {
  double g = w.a[0];
  for (int k = 1; k <= w.nh; ++k) {
    const double x = 2.0 * M_PI * k * t / w.period;
    g += w.a[k] * std::cos(x) + w.b[k] * std::sin(x);
  }
  return g;
}

dfvm_status bcs_time(dfvm_bcs* b, int slot, double t, cudaStream_t s) {
  b->t_eval = t;
  if (b->dirty[slot] || b->wave_patches[slot].empty()) return DFVM_OK;
  const int nc = slot == 0 ? 3 : 1;
  const int64_t B = b->m->part.n_lb;
  if (b->m->precision == DFVM_F64) {
    WaveG<double> g{};
    for (size_t j = 0; j < b->wave_patches[slot].size(); ++j) g.g[j] = wave_g(b->wave[slot][b->wave_patches[slot][j]], t);
    launch_bc_wave<double>((double*)b->d_val[slot], (const double*)b->d_base[slot], b->d_wid[slot], B, nc, g, s);
  } else {
    WaveG<float> g{};
    for (size_t j = 0; j < b->wave_patches[slot].size(); ++j) g.g[j] = (float)wave_g(b->wave[slot][b->wave_patches[slot][j]], t);
    launch_bc_wave<float>((float*)b->d_val[slot], (const float*)b->d_base[slot], b->d_wid[slot], B, nc, g, s);
  }
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

}  // namespace dfvm

using namespace dfvm;

#define CHECK_ARG(cond, msg)                                          \
  do {                                                                \
    if (!(cond)) { set_error(DFVM_E_INVALID_ARG, msg); return DFVM_E_INVALID_ARG; } \
  } while (0)

extern "C" {

const char* dfvm_last_error_message(void) { return g_msg.c_str(); }
int64_t dfvm_last_error_index(void) { return g_index; }
const char* dfvm_version(void) { return "libdfvm 0.1 (sm_100a, CUDA " __DATE__ ")"; }
int64_t dfvm_kernel_launches(void) { return g_launches.load(); }

dfvm_status dfvm_mesh_create(const double* points, int64_t n_points, const int64_t* face_offsets,
                             const int32_t* face_points, int64_t n_faces, const int32_t* owner,
                             const int32_t* neighbour, int64_t n_internal, const dfvm_patch_desc* patches,
                             int32_t n_patches, const dfvm_mesh_opts* opts, dfvm_comm* comm, dfvm_stream stream,
                             dfvm_mesh** out) {
  (void)stream;
  set_error(DFVM_OK, "", -1);
  CHECK_ARG(out && points && face_offsets && face_points, "NULL argument");
  dfvm_mesh_opts o{1, DFVM_NONORTH_OVERRELAXED, 1, 0, 0, DFVM_F64};
  if (opts) o = *opts;
  CHECK_ARG(o.n_parts >= 1 && o.rank >= 0 && o.rank < o.n_parts, "bad n_parts / rank");
  CHECK_ARG(o.precision == DFVM_F64 || o.precision == DFVM_F32, "bad precision");
  CHECK_ARG(o.n_parts == 1 || comm || o.device < 0, "n_parts > 1 needs a communicator");
  auto t0 = std::chrono::steady_clock::now();
  std::unique_ptr<dfvm_mesh> m(new (std::nothrow) dfvm_mesh());
  if (!m) return DFVM_E_OOM;
  const bool host_only = o.device < 0;   // maps / halo lists only (no device arrays, no compute)
  if (!host_only) {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      set_error(DFVM_E_CUDA, "no CUDA device available (libdfvm has no CPU fallback)");
      return DFVM_E_CUDA;
    }
    DFVM_CUDA(cudaSetDevice(o.device));
  }
  m->host_only = host_only;
  m->device = o.device;
  m->precision = o.precision;
  m->comm = comm;
  dfvm_status st = build_host_mesh(m->H, points, n_points, face_offsets, face_points, n_faces, owner, neighbour,
                                   n_internal, patches, n_patches, o.nonorth, o.renumber_rcm);
  if (st) return st;
  build_part(m->H, o.n_parts, o.rank, m->part);
  if (!host_only) {
    st = o.precision == DFVM_F64 ? upload_mesh<double>(m.get(), m->d64) : upload_mesh<float>(m.get(), m->d32);
    if (st) {
      for (void* p : m->allocations) dev_free(p, nullptr);
      return st;
    }
    DFVM_CUDA(cudaDeviceSynchronize());
  }
  m->host_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = m.release();
  return DFVM_OK;
}

dfvm_status dfvm_mesh_info_get(const dfvm_mesh* m, dfvm_mesh_info* info) {
  CHECK_ARG(m && info, "NULL argument");
  const HostMesh& H = m->H;
  int64_t nb = 0, ne = 0;
  for (int64_t k = H.F; k < H.NF; ++k) (H.pkind[H.bpatch[k - H.F]] == DFVM_PATCH_EMPTY ? ne : nb)++;
  info->n_cells = H.N; info->n_internal_faces = H.F; info->n_boundary_faces = nb; info->n_empty_faces = ne;
  info->n_owned = m->part.n_own; info->n_ghost = m->part.n_ghost;
  info->n_local_internal_faces = (int64_t)m->part.lf_gid.size();
  info->n_local_boundary_faces = m->part.n_lb;
  info->n_peers = (int32_t)m->part.peers.size();
  info->precision = m->precision;
  info->bandwidth_before = H.bw_before; info->bandwidth_after = H.bw_after;
  info->n_clamped = H.n_clamped;
  info->device_bytes = m->device_bytes;
  info->sell_max_row = m->precision == DFVM_F64 ? m->d64.max_row : m->d32.max_row;
  info->sell_slices = m->precision == DFVM_F64 ? m->d64.n_slices : m->d32.n_slices;
  info->host_seconds = m->host_seconds;
  return DFVM_OK;
}

dfvm_status dfvm_mesh_export_maps(const dfvm_mesh* m, int32_t* cell_new_of_old, int32_t* face_new_of_old,
                                  int8_t* face_flip, int32_t* cell_part, int32_t* row_ptr, int32_t* inc_face,
                                  int32_t* inc_nb) {
  CHECK_ARG(m, "NULL mesh");
  const HostMesh& H = m->H;
  if (cell_new_of_old) std::memcpy(cell_new_of_old, H.new_of_old.data(), 4 * H.N);
  if (face_new_of_old) std::memcpy(face_new_of_old, H.fnew_of_old.data(), 4 * H.NF);
  if (face_flip) std::memcpy(face_flip, H.flip_old.data(), H.F);
  if (cell_part) {
    const int P = m->part.P;
    for (int p = 0; p < P; ++p)
      for (int64_t c = (int64_t)p * H.N / P; c < (int64_t)(p + 1) * H.N / P; ++c) cell_part[c] = p;
  }
  if (row_ptr) std::memcpy(row_ptr, H.row_ptr.data(), 4 * (H.N + 1));
  if (inc_face) std::memcpy(inc_face, H.inc_face.data(), 4 * H.inc_face.size());
  if (inc_nb) std::memcpy(inc_nb, H.inc_nb.data(), 4 * H.inc_nb.size());
  return DFVM_OK;
}

dfvm_status dfvm_mesh_export_halo(const dfvm_mesh* m, int64_t* n_ghost, int32_t* ghost_gid, int32_t* ghost_peer,
                                  int64_t* n_send, int32_t* send_gid, int32_t* send_peer) {
  CHECK_ARG(m, "NULL mesh");
  const Part& P = m->part;
  if (n_ghost) *n_ghost = P.n_ghost;
  if (n_send) *n_send = (int64_t)P.send_gid.size();
  if (ghost_gid) std::memcpy(ghost_gid, P.ghost_gid.data(), 4 * P.ghost_gid.size());
  if (ghost_peer) std::memcpy(ghost_peer, P.ghost_peer.data(), 4 * P.ghost_peer.size());
  if (send_gid) std::memcpy(send_gid, P.send_gid.data(), 4 * P.send_gid.size());
  if (send_peer) std::memcpy(send_peer, P.send_peer.data(), 4 * P.send_peer.size());
  return DFVM_OK;
}

dfvm_status dfvm_mesh_export_geometry(const dfvm_mesh* m, double* Sf, double* xf, double* xc, double* V, double* w,
                                      double* delta, double* k, double* delta_b) {
  CHECK_ARG(m, "NULL mesh");
  const HostMesh& H = m->H;
  if (Sf) std::memcpy(Sf, H.Sf0.data(), 8 * H.Sf0.size());
  if (xf) std::memcpy(xf, H.xf0.data(), 8 * H.xf0.size());
  if (xc) std::memcpy(xc, H.xc0.data(), 8 * H.xc0.size());
  if (V) std::memcpy(V, H.V0.data(), 8 * H.V0.size());
  // coefficients are computed in the new orientation; report them in the
  // original orientation: w -> 1 - w and k -> -k on flipped faces
  for (int64_t f = 0; f < H.F; ++f) {
    const int64_t kk = H.fnew_of_old[f];
    const bool fl = H.flip_old[f];
    if (w) w[f] = fl ? 1.0 - H.w[kk] : H.w[kk];
    if (delta) delta[f] = H.delta[kk];
    if (k) for (int j = 0; j < 3; ++j) k[3 * f + j] = fl ? -H.k[3 * kk + j] : H.k[3 * kk + j];
  }
  if (delta_b)
    for (int64_t f = H.F; f < H.NF; ++f) delta_b[f - H.F] = H.delta_b[H.fnew_of_old[f] - H.F];
  return DFVM_OK;
}

dfvm_status dfvm_mesh_destroy(dfvm_mesh* m) {
  if (!m) return DFVM_OK;
  if (m->host_only) { delete m; return DFVM_OK; }
  cudaSetDevice(m->device);
  cudaDeviceSynchronize();
  for (void* p : m->allocations) dev_free(p, nullptr);
  dev_free(m->halo0.d_send, nullptr);
  dev_free(m->halo0.d_send_idx, nullptr);
  dev_free(m->d_stage, nullptr);
  delete m;
  return DFVM_OK;
}

// ------------------------------------------------------------------ fields
static size_t elem_bytes(const dfvm_mesh* m) { return m->precision == DFVM_F64 ? 8 : 4; }

dfvm_status dfvm_field_bytes(const dfvm_mesh* m, int32_t loc, int32_t n_comp, size_t* bytes) {
  CHECK_ARG(m && bytes && n_comp >= 1 && n_comp <= 9 && loc >= 0 && loc <= 2, "bad field arguments");
  if (m->host_only) { set_error(DFVM_E_CUDA, "host-only mesh (device < 0) has no device data"); return DFVM_E_CUDA; }
  const int64_t n = loc == DFVM_CELLS ? m->part.n_own + m->part.n_ghost : m->n_faces_local();
  *bytes = (size_t)std::max<int64_t>(n, 1) * n_comp * elem_bytes(m);
  return DFVM_OK;
}

dfvm_status dfvm_field_alloc(dfvm_mesh* m, int32_t loc, int32_t n_comp, dfvm_field** out) {
  size_t bytes = 0;
  if (dfvm_status st = dfvm_field_bytes(m, loc, n_comp, &bytes)) return st;
  CHECK_ARG(out, "NULL out");
  void* p = nullptr;
  if (dfvm_status st = dev_alloc(&p, bytes, nullptr, true)) return st;
  DFVM_CUDA(cudaStreamSynchronize(nullptr));   // zero-fill done before any use on a non-blocking stream
  dfvm_field* f = new dfvm_field();
  f->m = m; f->ptr = p; f->loc = loc; f->n_comp = n_comp; f->owned = true;
  *out = f;
  return DFVM_OK;
}

dfvm_status dfvm_field_wrap(dfvm_mesh* m, void* dev_ptr, int32_t loc, int32_t n_comp, dfvm_field** out) {
  size_t bytes = 0;
  if (dfvm_status st = dfvm_field_bytes(m, loc, n_comp, &bytes)) return st;
  CHECK_ARG(out && dev_ptr, "NULL argument");
  dfvm_field* f = new dfvm_field();
  f->m = m; f->ptr = dev_ptr; f->loc = loc; f->n_comp = n_comp; f->owned = false;
  *out = f;
  return DFVM_OK;
}

dfvm_status dfvm_field_data(const dfvm_field* f, void** dev_ptr) {
  CHECK_ARG(f && dev_ptr, "NULL argument");
  *dev_ptr = f->ptr;
  return DFVM_OK;
}

dfvm_status dfvm_field_destroy(dfvm_field* f) {
  if (!f) return DFVM_OK;
  if (f->owned && f->ptr) { cudaDeviceSynchronize(); dev_free(f->ptr, nullptr); }
  delete f;
  return DFVM_OK;
}

static int64_t global_count(const dfvm_field* f) {
  return f->loc == DFVM_CELLS ? f->m->H.N : f->m->H.NF;
}

// grow the mesh's persistent staging buffer (a per-call cudaMallocAsync of
// GBs per call returns and re-maps pool memory each time; the C5 e2e leg
// spent ~1.3 s/step in import/export with it)
static dfvm_status stage(dfvm_mesh* m, size_t bytes) {
  if (m->stage_bytes >= bytes) return DFVM_OK;
  if (m->d_stage) { DFVM_CUDA(cudaDeviceSynchronize()); dev_free(m->d_stage, nullptr); m->d_stage = nullptr; }
  if (dfvm_status st = dev_alloc(&m->d_stage, bytes, nullptr, false)) return st;
  DFVM_CUDA(cudaStreamSynchronize(nullptr));
  m->stage_bytes = bytes;
  return DFVM_OK;
}

dfvm_status dfvm_field_import(dfvm_field* f, const double* src, int32_t src_is_host, dfvm_stream stream) {
  CHECK_ARG(f && src, "NULL argument");
  dfvm_mesh* m = f->m;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = f->count();
  const int32_t* map = f->loc == DFVM_CELLS ? m->d_cell_orig : m->d_face_orig;
  const bool oriented = f->loc == 2;
  const double* dsrc = src;
  std::unique_lock<std::mutex> lk(m->stage_mu, std::defer_lock);
  if (src_is_host) {
    const size_t bytes = (size_t)global_count(f) * f->n_comp * 8;
    lk.lock();
    if (dfvm_status st = stage(m, bytes)) return st;
    DFVM_CUDA(cudaMemcpyAsync(m->d_stage, src, bytes, cudaMemcpyHostToDevice, s));
    dsrc = (const double*)m->d_stage;
  }
  if (m->precision == DFVM_F64) launch_import<double>((double*)f->ptr, dsrc, map, n, f->n_comp, oriented, s);
  else launch_import<float>((float*)f->ptr, dsrc, map, n, f->n_comp, oriented, s);
  DFVM_CUDA(cudaGetLastError());
  if (src_is_host) DFVM_CUDA(cudaStreamSynchronize(s));   // the caller may free src; staging reusable
  return DFVM_OK;
}

dfvm_status dfvm_field_export(const dfvm_field* f, double* dst, int32_t dst_is_host, dfvm_stream stream) {
  CHECK_ARG(f && dst, "NULL argument");
  dfvm_mesh* m = f->m;
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t* map = f->loc == DFVM_CELLS ? m->d_cell_orig : m->d_face_orig;
  const int64_t n = f->loc == DFVM_CELLS ? m->part.n_own : f->count();
  const bool oriented = f->loc == 2;
  const size_t bytes = (size_t)global_count(f) * f->n_comp * 8;
  double* ddst = dst;
  std::unique_lock<std::mutex> lk(m->stage_mu, std::defer_lock);
  if (dst_is_host) {
    lk.lock();
    if (dfvm_status st = stage(m, bytes)) return st;
    if (m->part.P > 1)   // keep the entries other ranks own
      DFVM_CUDA(cudaMemcpyAsync(m->d_stage, dst, bytes, cudaMemcpyHostToDevice, s));
    ddst = (double*)m->d_stage;
  }
  if (m->precision == DFVM_F64) launch_export<double>(ddst, (const double*)f->ptr, map, n, f->n_comp, oriented, s);
  else launch_export<float>(ddst, (const float*)f->ptr, map, n, f->n_comp, oriented, s);
  DFVM_CUDA(cudaGetLastError());
  if (dst_is_host) {
    DFVM_CUDA(cudaMemcpyAsync(dst, m->d_stage, bytes, cudaMemcpyDeviceToHost, s));
    DFVM_CUDA(cudaStreamSynchronize(s));
  }
  return DFVM_OK;
}

// --------------------------------------------------------------------- BCs
dfvm_status dfvm_bcs_create(dfvm_mesh* m, dfvm_bcs** out) {
  CHECK_ARG(m && out, "NULL argument");
  dfvm_bcs* b = new dfvm_bcs();
  b->m = m;
  for (int i = 0; i < 3; ++i) {
    b->spec[i].assign(m->H.pkind.size(), dfvm_bc_desc{});
    b->set[i].assign(m->H.pkind.size(), 0);
    b->wave[i].assign(m->H.pkind.size(), dfvm_bcs::Wave{});
  }
  *out = b;
  return DFVM_OK;
}

dfvm_status dfvm_bcs_set(dfvm_bcs* b, int32_t patch, char field, const dfvm_bc_desc* d) {
  CHECK_ARG(b && d, "NULL argument");
  const int slot = field_slot(field);
  if (slot < 0 || patch < 0 || patch >= (int32_t)b->m->H.pkind.size()) {
    set_error(DFVM_E_INVALID_ARG, "bad patch or field", patch);
    return DFVM_E_INVALID_ARG;
  }
  if (d->kind < 0 || d->kind > 3 || (d->kind == DFVM_BC_PARABOLIC && slot != 0) ||
      (d->kind == DFVM_BC_WINDKESSEL && slot != 1)) {
    set_error(DFVM_E_INVALID_ARG, "boundary condition kind not valid for this field", patch);
    return DFVM_E_INVALID_ARG;
  }
  if (d->kind == DFVM_BC_PARABOLIC && !(d->radius > 0)) {
    set_error(DFVM_E_INVALID_ARG, "parabolic inlet needs radius > 0", patch);
    return DFVM_E_INVALID_ARG;
  }
  b->spec[slot][patch] = *d;
  b->set[slot][patch] = 1;
  b->dirty[slot] = true;
  return DFVM_OK;
}

dfvm_status dfvm_bcs_set_waveform(dfvm_bcs* b, int32_t patch, char field, double period, int32_t nh,
                                  const double* a, const double* bc) {
  CHECK_ARG(b && a, "NULL argument");
  const int slot = field_slot(field);
  if (slot < 0 || slot > 1 || patch < 0 || patch >= (int32_t)b->m->H.pkind.size() || nh < 0 || nh > 16 ||
      !(period > 0)) {
    set_error(DFVM_E_INVALID_ARG, "bad waveform (field 'U' or 'p', 0 <= n_harmonics <= 16, period > 0)", patch);
    return DFVM_E_INVALID_ARG;
  }
  dfvm_bcs::Wave w;
  w.nh = nh; w.period = period;
  for (int k = 0; k <= nh; ++k) { w.a[k] = a[k]; w.b[k] = (k > 0 && bc) ? bc[k] : 0.0; }
  b->wave[slot][patch] = w;
  b->dirty[slot] = true;
  return DFVM_OK;
}

dfvm_status dfvm_bcs_set_time(dfvm_bcs* b, double t, dfvm_stream stream) {
  CHECK_ARG(b, "NULL argument");
  b->t_eval = t;
  for (int slot = 0; slot < 2; ++slot)
    if (!b->dirty[slot]) {
      dfvm_status st = bcs_time(b, slot, t, (cudaStream_t)stream);
      if (st) return st;
      if (!b->wave_patches[slot].empty()) count_launch();
    }
  return DFVM_OK;
}

dfvm_status dfvm_bcs_destroy(dfvm_bcs* b) {
  if (!b) return DFVM_OK;
  for (int i = 0; i < 3; ++i) {
    dev_free(b->d_kind[i], nullptr);
    dev_free(b->d_val[i], nullptr);
    dev_free(b->d_base[i], nullptr);
    dev_free(b->d_wid[i], nullptr);
  }
  delete b;
  return DFVM_OK;
}

// --------------------------------------------------------------- operators
static dfvm_status check_field(const dfvm_field* f, const dfvm_mesh* m, int loc, int nc, const char* what) {
  if (!f || f->m != m || (loc >= 0 && (loc == DFVM_FACES ? (f->loc == DFVM_CELLS) : f->loc != loc)) ||
      (nc > 0 && f->n_comp != nc)) {
    set_error(DFVM_E_INVALID_ARG, std::string("field argument '") + what + "' has the wrong mesh, location or size");
    return DFVM_E_INVALID_ARG;
  }
  return DFVM_OK;
}

#define DISPATCH(m, CALL64, CALL32) \
  do { if ((m)->precision == DFVM_F64) { CALL64; } else { CALL32; } } while (0)

dfvm_status dfvm_fvc_interpolate(dfvm_mesh* m, const dfvm_field* x, const dfvm_bcs* b, char fld, dfvm_field* xf,
                                 dfvm_stream stream) {
  CHECK_ARG(m && b && b->m == m, "NULL or mismatched argument");
  const int slot = field_slot(fld);
  CHECK_ARG(slot >= 0, "field must be 'U', 'p' or 's'");
  const int nc = slot == 0 ? 3 : 1;
  dfvm_status st;
  if ((st = check_field(x, m, DFVM_CELLS, nc, "x")) || (st = check_field(xf, m, DFVM_FACES, nc, "xf"))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = bcs_device(const_cast<dfvm_bcs*>(b), slot, s))) return st;
  if ((st = halo_exchange(m, x->ptr, nc, s))) return st;
  DISPATCH(m, launch_interpolate<double>(m->d64, (const double*)x->ptr, nc, b->d_kind[slot], (const double*)b->d_val[slot], (double*)xf->ptr, s),
              launch_interpolate<float>(m->d32, (const float*)x->ptr, nc, b->d_kind[slot], (const float*)b->d_val[slot], (float*)xf->ptr, s));
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

dfvm_status dfvm_fvc_grad(dfvm_mesh* m, const dfvm_field* x, const dfvm_bcs* b, char fld, dfvm_field* grad,
                          dfvm_stream stream) {
  CHECK_ARG(m && b && b->m == m, "NULL or mismatched argument");
  const int slot = field_slot(fld);
  CHECK_ARG(slot >= 0, "field must be 'U', 'p' or 's'");
  const int nc = slot == 0 ? 3 : 1;
  dfvm_status st;
  if ((st = check_field(x, m, DFVM_CELLS, nc, "x")) || (st = check_field(grad, m, DFVM_CELLS, 3 * nc, "grad"))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = bcs_device(const_cast<dfvm_bcs*>(b), slot, s))) return st;
  if ((st = halo_exchange(m, x->ptr, nc, s))) return st;
  DISPATCH(m, launch_grad<double>(m->d64, (const double*)x->ptr, nc, b->d_kind[slot], (const double*)b->d_val[slot], (double*)grad->ptr, s),
              launch_grad<float>(m->d32, (const float*)x->ptr, nc, b->d_kind[slot], (const float*)b->d_val[slot], (float*)grad->ptr, s));
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

dfvm_status dfvm_fvc_grad_faces(dfvm_mesh* m, const dfvm_field* fv, dfvm_field* grad, dfvm_stream stream) {
  CHECK_ARG(m && fv, "NULL argument");
  const int nc = fv->n_comp;
  CHECK_ARG(nc == 1 || nc == 3, "face values must have 1 or 3 components");
  dfvm_status st;
  if ((st = check_field(fv, m, DFVM_FACES, nc, "face_vals")) || (st = check_field(grad, m, DFVM_CELLS, 3 * nc, "grad"))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH(m, launch_grad_faces<double>(m->d64, (const double*)fv->ptr, nc, (double*)grad->ptr, s),
              launch_grad_faces<float>(m->d32, (const float*)fv->ptr, nc, (float*)grad->ptr, s));
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

dfvm_status dfvm_fvc_div(dfvm_mesh* m, const dfvm_field* flux, dfvm_field* out, dfvm_stream stream) {
  CHECK_ARG(m, "NULL mesh");
  dfvm_status st;
  if ((st = check_field(flux, m, DFVM_FACES, 1, "face_flux")) || (st = check_field(out, m, DFVM_CELLS, 1, "out"))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH(m, launch_div<double>(m->d64, (const double*)flux->ptr, (double*)out->ptr, s),
              launch_div<float>(m->d32, (const float*)flux->ptr, (float*)out->ptr, s));
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

dfvm_status dfvm_fvm_laplacian_apply(dfvm_mesh* m, const dfvm_field* gamma, const dfvm_bcs* b, char fld,
                                     const dfvm_field* x, const dfvm_field* grad, dfvm_field* y, dfvm_stream stream) {
  CHECK_ARG(m && b && b->m == m, "NULL or mismatched argument");
  const int slot = field_slot(fld);
  CHECK_ARG(slot == 1 || slot == 2, "laplacian field must be a scalar ('p' or 's')");
  dfvm_status st;
  if ((st = check_field(x, m, DFVM_CELLS, 1, "x")) || (st = check_field(y, m, DFVM_CELLS, 1, "y"))) return st;
  if (gamma && (st = check_field(gamma, m, DFVM_CELLS, 1, "gamma"))) return st;
  if (grad && (st = check_field(grad, m, DFVM_CELLS, 3, "grad"))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = bcs_device(const_cast<dfvm_bcs*>(b), slot, s))) return st;
  if ((st = halo_exchange(m, x->ptr, 1, s))) return st;
  if (gamma && (st = halo_exchange(m, gamma->ptr, 1, s))) return st;
  void* G = grad ? grad->ptr : nullptr;
  void* tmp = nullptr;
  if (!G) {
    if ((st = dev_alloc(&tmp, (size_t)(m->part.n_own + m->part.n_ghost) * 3 * elem_bytes(m), s, false))) return st;
    G = tmp;
    DISPATCH(m, launch_grad<double>(m->d64, (const double*)x->ptr, 1, b->d_kind[slot], (const double*)b->d_val[slot], (double*)G, s),
                launch_grad<float>(m->d32, (const float*)x->ptr, 1, b->d_kind[slot], (const float*)b->d_val[slot], (float*)G, s));
  }
  if ((st = halo_exchange(m, G, 3, s))) return st;
  DISPATCH(m, launch_laplacian<double>(m->d64, gamma ? (const double*)gamma->ptr : nullptr, (const double*)x->ptr, (const double*)G, b->d_kind[slot], (const double*)b->d_val[slot], (double*)y->ptr, s),
              launch_laplacian<float>(m->d32, gamma ? (const float*)gamma->ptr : nullptr, (const float*)x->ptr, (const float*)G, b->d_kind[slot], (const float*)b->d_val[slot], (float*)y->ptr, s));
  if (tmp) dev_free(tmp, s);
  DFVM_CUDA(cudaGetLastError());
  return DFVM_OK;
}

}  // extern "C"
