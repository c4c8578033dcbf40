/* dfvm.h — C ABI of libdfvm.so: DiFVM's data-parallel hot path on B200.
 *
 * The face-based finite-volume operator as a static gather/scatter over the
 * mesh graph (§2.3-§2.4) and the incompressible PISO step
 * built on it with the matrix-free Krylov pressure solve,
 * hand-written sm_100a kernels behind plain-pointer entry points.
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "§8(x)" = /root/repo/SURVEY.md section 8 row; readings "A-n" are listed in
 * DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every entry point returns dfvm_status; out-params are written only on
 *    DFVM_OK (solvers also on DFVM_E_NOT_CONVERGED: best iterate + report).
 *    dfvm_last_error_message()/dfvm_last_error_index() (thread-local) name
 *    the offending face / cell / patch in the CALLER'S ORIGINAL numbering.
 *    No C++ exception crosses the ABI.
 *  - Numbering: the caller always speaks its original cell / face / patch
 *    numbering.  The library renumbers internally (RCM + face re-sort,
 *    §8(c) O-9); dfvm_field_import/export permute, dfvm_mesh_export_maps
 *    exposes every integer map.
 *  - Ownership: mesh arrays passed to dfvm_mesh_create are host, caller-owned
 *    and copied (no pointer kept).  Device state created by the library is
 *    freed by the matching *_destroy.  dfvm_field_wrap wraps CALLER-OWNED
 *    device memory (e.g. a torch tensor's data_ptr()); the library never
 *    frees it and the caller keeps it alive until the stream has completed.
 *  - Streams: compute calls are asynchronous on the caller's cudaStream_t
 *    (pass torch.cuda.current_stream().cuda_stream; 0 = legacy default).
 *    Implicit synchronisations: dfvm_mesh_create, host export, report
 *    read-back at the end of dfvm_pressure_solve / dfvm_piso_step.
 *  - Precision: fixed per mesh (dfvm_mesh_opts.precision).  Field device
 *    data have the mesh precision; import/export buffers are always fp64.
 *    Dot products and Krylov scalars are fp64 in both precisions.
 *  - Indices are int32 inside the library: N and 2F must be < 2^31 (else
 *    DFVM_E_INVALID_ARG).
 *  - Threading: one solver per host thread; meshes are immutable after
 *    create and safe for concurrent reads.
 *  - No CPU fallback: every compute entry point runs CUDA kernels; without a
 *    usable CUDA device they return DFVM_E_CUDA.
 */
#ifndef DFVM_H
#define DFVM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dfvm_stream; /* == cudaStream_t */

typedef enum {
  DFVM_OK = 0,
  DFVM_E_INVALID_ARG = 1,
  DFVM_E_MESH_CONSISTENCY = 2,   /* S:46 (index: face or cell) */
  DFVM_E_DEGENERATE_FACE = 3,    /* S:64 (index: face) */
  DFVM_E_INVERTED_CELL = 4,      /* S:64 (index: cell) */
  DFVM_E_NONCONVEX_PAIR = 5,     /* S:134 S_f . d <= 0 (index: face) */
  DFVM_E_EXTREME_NONORTH = 6,
  DFVM_E_MISSING_BC = 7,         /* S:55 (index: patch) */
  DFVM_E_NOT_CONVERGED = 8,
  DFVM_E_BREAKDOWN = 9,
  DFVM_E_NONFINITE = 10,
  DFVM_E_CONTINUITY = 11,
  DFVM_E_INVALID_WK_PARAMS = 12,
  DFVM_E_CUDA = 13,
  DFVM_E_NCCL = 14,
  DFVM_E_OOM = 15
} dfvm_status;

const char* dfvm_last_error_message(void);
int64_t dfvm_last_error_index(void);
/* library build/version string (also names the CUDA arch it was built for) */
const char* dfvm_version(void);

/* ------------------------------------------------------------- allocator
 * §8(b) row b3 (north star: "PyTorch only for device memory"): every device
 * buffer the library owns (mesh arrays, boundary values, library-owned
 * fields, solver / AMG workspace, halo and staging buffers) comes from
 * alloc(bytes, stream, ctx) and goes back through free_(ptr, bytes, stream,
 * ctx); pass torch's caching allocator (torch.cuda.caching_allocator_alloc /
 * _delete) to let PyTorch own the memory.  Default (both NULL):
 * cudaMallocAsync / cudaFreeAsync on the stream.  `stream` is the caller's
 * stream of the compute call that allocates lazily, or the legacy stream (0)
 * for allocations made by *_create (which synchronise before returning);
 * the library zero-fills new buffers on that stream.  Process-wide; may only
 * be changed while no library allocation is live (else DFVM_E_INVALID_ARG,
 * index = number of live allocations).  alloc returning NULL -> DFVM_E_OOM.
 * The callbacks may be called from any thread that calls the library. */
typedef void* (*dfvm_alloc_fn)(size_t bytes, dfvm_stream stream, void* ctx);
typedef void (*dfvm_free_fn)(void* ptr, size_t bytes, dfvm_stream stream, void* ctx);
dfvm_status dfvm_set_allocator(dfvm_alloc_fn alloc, dfvm_free_fn free_, void* ctx);
/* bytes currently held by library allocations (all meshes / fields / solvers) */
int64_t dfvm_live_device_bytes(void);

/* ------------------------------------------------------------------ comm
 * Multi-GPU (§8(e)): one process per GPU.  Rank 0 calls dfvm_comm_unique_id,
 * the caller broadcasts the 128 bytes with torch.distributed, every rank
 * calls dfvm_comm_create.  NCCL over NVLink carries halo exchanges and the
 * Krylov / Windkessel reductions (deterministic all-gather + fixed-order
 * sum).  n_ranks == 1 needs no communicator (pass NULL). */
typedef struct dfvm_comm dfvm_comm;
dfvm_status dfvm_comm_unique_id(uint8_t id[128]);
dfvm_status dfvm_comm_create(int n_ranks, int rank, const uint8_t id[128], int device, dfvm_comm** out);
/* In-process group of n_ranks communicators (ranks as host threads of one
 * process, devices[r] per rank; NULL -> all on device 0).  Same partitioned
 * solver path as NCCL, with device-to-device copies and host barriers: lets
 * the multi-rank logic run (and be tested) on a single GPU.  out[n_ranks]. */
dfvm_status dfvm_comm_create_local(int n_ranks, const int* devices, dfvm_comm** out);
dfvm_status dfvm_comm_destroy(dfvm_comm* c);

/* ------------------------------------------------------------------ mesh
 * OpenFOAM polyMesh convention: internal faces first
 * with owner < neighbour, each face ring's right-hand normal points out of
 * its owner, patches tile [n_internal, n_faces) in order.
 * Validation (first failure wins, §8(c) O-0): vertex index range, owner /
 * neighbour range and >= 4 faces per cell, owner < neighbour, patch tiling,
 * empty patches only on extruded cells. */
typedef enum { DFVM_PATCH_GENERIC = 0, DFVM_PATCH_WALL = 1, DFVM_PATCH_EMPTY = 2 } dfvm_patch_kind;
typedef struct {
  const char* name;
  int32_t kind;        /* dfvm_patch_kind */
  int64_t start_face;
  int64_t n_faces;
} dfvm_patch_desc;

/* P:251-254 / Table 1 P:391 non-orthogonal correction (A-3, A-4) */
typedef enum {
  DFVM_NONORTH_NONE = 0,        /* eq:diff_ortho: delta = |S|/|d|, k = 0 */
  DFVM_NONORTH_MINIMUM = 1,     /* Delta = (S.d^) d^ */
  DFVM_NONORTH_ORTHOGONAL = 2,  /* Delta = |S| d^ */
  DFVM_NONORTH_OVERRELAXED = 3  /* Delta = (|S| / |S^.d^|) d^  (default) */
} dfvm_nonorth;

typedef enum { DFVM_F64 = 0, DFVM_F32 = 1 } dfvm_dtype;

typedef struct {
  int32_t renumber_rcm;  /* 1: RCM renumbering (default), 0: keep input order */
  int32_t nonorth;       /* dfvm_nonorth */
  int32_t n_parts;       /* number of ranks (1 = single GPU) */
  int32_t rank;
  int32_t device;        /* CUDA device ordinal; < 0: host-only mesh (integer maps and
                            halo lists only, no device arrays; compute calls fail) */
  int32_t precision;     /* dfvm_dtype */
} dfvm_mesh_opts;

typedef struct dfvm_mesh dfvm_mesh;

typedef struct {
  int64_t n_cells, n_internal_faces, n_boundary_faces, n_empty_faces; /* global */
  int64_t n_owned, n_ghost, n_local_internal_faces, n_local_boundary_faces;
  int32_t n_peers, precision;
  int64_t bandwidth_before, bandwidth_after;  /* max |new(o) - new(n)| over internal faces */
  int64_t n_clamped;                          /* over-relaxed clamp count (A-4) */
  int64_t device_bytes;                       /* mesh arrays resident on the GPU */
  int32_t sell_max_row, sell_slices;          /* SELL-32 incidence layout */
  double host_seconds;                        /* wall time of mesh_create */
} dfvm_mesh_info;

/* Builds the mesh on `opts->device`: validation, fp64 geometry (O-1),
 * RCM + face re-sort + cell->face CSR (O-9), partition part `opts->rank` of
 * `opts->n_parts` with its halo maps, face coefficients (O-3), and uploads
 * the SoA/SELL arrays.  Synchronous. comm may be NULL when n_parts == 1. */
dfvm_status dfvm_mesh_create(const double* points, int64_t n_points, const int64_t* face_offsets,
                             const int32_t* face_points, int64_t n_faces, const int32_t* owner,
                             const int32_t* neighbour, int64_t n_internal, const dfvm_patch_desc* patches,
                             int32_t n_patches, const dfvm_mesh_opts* opts, dfvm_comm* comm,
                             dfvm_stream stream, dfvm_mesh** out);
dfvm_status dfvm_mesh_info_get(const dfvm_mesh* m, dfvm_mesh_info* info);
/* Integer maps (global, bit-exact with §8(c) O-9); any pointer may be NULL.
 * cell_new_of_old[N], face_new_of_old[n_faces], face_flip[n_internal]
 * (indexed by old face), cell_part[N] (by new id), row_ptr[N+1],
 * inc_face[2F] (new face index, bit 31 set when the cell is the neighbour),
 * inc_nb[2F] (new neighbour id). */
dfvm_status dfvm_mesh_export_maps(const dfvm_mesh* m, int32_t* cell_new_of_old, int32_t* face_new_of_old,
                                  int8_t* face_flip, int32_t* cell_part, int32_t* row_ptr, int32_t* inc_face,
                                  int32_t* inc_nb);
/* This rank's halo lists in new (global) ids: ghost_gid[n_ghost] ordered by
 * (peer, id), ghost_peer[n_ghost]; send_gid[n_send], send_peer[n_send]
 * ordered by (peer, id).  Sizes: *n_ghost, *n_send (query with NULL arrays). */
dfvm_status dfvm_mesh_export_halo(const dfvm_mesh* m, int64_t* n_ghost, int32_t* ghost_gid, int32_t* ghost_peer,
                                  int64_t* n_send, int32_t* send_gid, int32_t* send_peer);
/* fp64 geometry and coefficients in ORIGINAL order (parity with O-1/O-3):
 * Sf[n_faces][3], xf[n_faces][3], xc[N][3], V[N], w[F], delta[F], k[F][3],
 * delta_b[n_faces - F] (0 on empty faces).  Any pointer may be NULL. */
dfvm_status dfvm_mesh_export_geometry(const dfvm_mesh* m, double* Sf, double* xf, double* xc, double* V,
                                      double* w, double* delta, double* k, double* delta_b);
dfvm_status dfvm_mesh_destroy(dfvm_mesh* m);

/* ---- OpenFOAM ASCII polyMesh reader (P:431-432
 * "reads OpenFOAM polyMesh files directly", Table 1).
 * dir: a case directory, its constant/polyMesh, or the polyMesh directory;
 * files points, faces, owner, neighbour, boundary in ASCII format (FoamFile
 * header `format ascii`; binary or gzip files -> DFVM_E_INVALID_ARG naming
 * the file, as are parse errors and cyclic / processor / wedge patches).
 * Patch type wall -> DFVM_PATCH_WALL, empty -> DFVM_PATCH_EMPTY, anything
 * else -> DFVM_PATCH_GENERIC.  The reader only parses: mesh invariants are
 * checked by dfvm_mesh_create.  dfvm_polymesh_arrays returns pointers owned
 * by the reader object (valid until dfvm_polymesh_destroy), laid out exactly
 * as dfvm_mesh_create takes them; n_cells = 1 + the largest owner /
 * neighbour label.  Host only. */
typedef struct dfvm_polymesh dfvm_polymesh;
dfvm_status dfvm_polymesh_read(const char* dir, dfvm_polymesh** out);
dfvm_status dfvm_polymesh_sizes(const dfvm_polymesh* m, int64_t* n_points, int64_t* n_faces,
                                int64_t* n_face_points, int64_t* n_internal_faces, int32_t* n_patches,
                                int64_t* n_cells);
dfvm_status dfvm_polymesh_arrays(const dfvm_polymesh* m, const double** points, const int64_t** face_offsets,
                                 const int32_t** face_points, const int32_t** owner, const int32_t** neighbour,
                                 const dfvm_patch_desc** patches);
dfvm_status dfvm_polymesh_destroy(dfvm_polymesh* m);

/* ---------------------------------------------------------------- fields
 * Cell fields: [n_owned + n_ghost][n_comp] in internal (RCM) order.
 * Face fields: [n_local_internal + n_local_boundary + n_local_empty][n_comp]
 * in internal face order.  Device element type = mesh precision. */
/* DFVM_FACES: unoriented face values (e.g. interpolated phi_f);
 * DFVM_FACE_FLUX: oriented face fluxes (phi, F of fvc_div) whose sign follows
 * the face orientation: import/export negate them on faces the renumbering
 * re-oriented (O-9 step 5), so the caller always sees its own orientation. */
typedef enum { DFVM_CELLS = 0, DFVM_FACES = 1, DFVM_FACE_FLUX = 2 } dfvm_loc;
typedef struct dfvm_field dfvm_field;
dfvm_status dfvm_field_bytes(const dfvm_mesh* m, int32_t loc, int32_t n_comp, size_t* bytes);
/* north-star `field_alloc`: library-owned device memory (zero-filled) */
dfvm_status dfvm_field_alloc(dfvm_mesh* m, int32_t loc, int32_t n_comp, dfvm_field** out);
/* wrap caller-owned device memory of dfvm_field_bytes() bytes */
dfvm_status dfvm_field_wrap(dfvm_mesh* m, void* dev_ptr, int32_t loc, int32_t n_comp, dfvm_field** out);
dfvm_status dfvm_field_data(const dfvm_field* f, void** dev_ptr);
/* src: fp64 [global count][n_comp] in ORIGINAL order (host if src_is_host,
 * else device).  Ghost cells are filled too (no halo exchange needed). */
dfvm_status dfvm_field_import(dfvm_field* f, const double* src, int32_t src_is_host, dfvm_stream stream);
/* dst: fp64 [global count][n_comp] in ORIGINAL order; only this rank's owned
 * entries are written (P=1: all).  Host export synchronises the stream. */
dfvm_status dfvm_field_export(const dfvm_field* f, double* dst, int32_t dst_is_host, dfvm_stream stream);
dfvm_status dfvm_field_destroy(dfvm_field* f); /* never frees wrapped memory */

/* ------------------------------------------------- boundary conditions
 * Per (patch, field) with field 'U' (vector), 'p' or 's' (scalars)
 * (Table 1; §2.6.2).  Every non-empty
 * patch needs a spec for each field an operator / solver reads
 * (DFVM_E_MISSING_BC otherwise). */
typedef enum {
  DFVM_BC_FIXED_VALUE = 0,     /* Dirichlet: value[] */
  DFVM_BC_ZERO_GRADIENT = 1,   /* Neumann: phi_b = phi_O */
  DFVM_BC_PARABOLIC = 2,       /* 'U' only: u_b = -u_max (1 - r^2/R^2) n_out (A-18),
                                  r = |x_b - center|, R = radius */
  DFVM_BC_WINDKESSEL = 3       /* 'p' only: set through dfvm_windkessel_set */
} dfvm_bc_kind;
typedef struct {
  int32_t kind;
  double value[3];
  double u_max;
  double center[3];
  double radius;
} dfvm_bc_desc;
typedef struct dfvm_bcs dfvm_bcs;
dfvm_status dfvm_bcs_create(dfvm_mesh* m, dfvm_bcs** out);
dfvm_status dfvm_bcs_set(dfvm_bcs* b, int32_t patch, char field, const dfvm_bc_desc* desc);
dfvm_status dfvm_bcs_destroy(dfvm_bcs* b);
/* Time-varying boundary value (Table 1 P:393 "time-varying inflow", P:401,
 * P:582 "a pulsatile parabolic velocity profile"; reading A-41):
 * the fixed-value or parabolic value of (patch, field) is multiplied by
 *   g(t) = a[0] + sum_{k=1..n_harmonics} a[k] cos(2 pi k t/period) + b[k] sin(2 pi k t/period),
 * evaluated on the host in fp64 at the time the values are used: t^{n+1} =
 * t^n + dt in dfvm_piso_step (the solver's time starts at 0 and advances by
 * dt per step), else the time of the last dfvm_bcs_set_time (initially 0).
 * field 'U' or 'p'; a[n_harmonics + 1], b[n_harmonics + 1] (b[0] unused;
 * b may be NULL = all zero) are copied.  n_harmonics in [0, 16], period > 0,
 * else DFVM_E_INVALID_ARG; a step whose waveform patch is not fixed-value /
 * parabolic fails with DFVM_E_INVALID_ARG. */
dfvm_status dfvm_bcs_set_waveform(dfvm_bcs* b, int32_t patch, char field, double period, int32_t n_harmonics,
                                  const double* a, const double* bcoef);
/* evaluate every waveform at time t (device values updated on `stream`) */
dfvm_status dfvm_bcs_set_time(dfvm_bcs* b, double t, dfvm_stream stream);

/* ------------------------------------------------------------ operators
 * Asynchronous on `stream`; each performs the halo exchange of its input
 * first when n_parts > 1.  Vector gradients: grad[c][k][l] = d(phi^k)/dx^l. */
/* phi_f = w phi_O + (1-w) phi_N; boundary faces phi_b; empty 0 */
dfvm_status dfvm_fvc_interpolate(dfvm_mesh* m, const dfvm_field* x, const dfvm_bcs* b, char field,
                                 dfvm_field* xf, dfvm_stream stream);
/* Gauss-Green gradient (eq:gauss_green P:207-214): G_c = V_c^-1 sum_f s_cf phi_f S_f */
dfvm_status dfvm_fvc_grad(dfvm_mesh* m, const dfvm_field* x, const dfvm_bcs* b, char field, dfvm_field* grad,
                          dfvm_stream stream);
/* same sum with caller-given face values (exact-face-value pin) */
dfvm_status dfvm_fvc_grad_faces(dfvm_mesh* m, const dfvm_field* face_vals, dfvm_field* grad, dfvm_stream stream);
/* D_c = sum_f s_cf F_f + sum_b F_b (eq:aggregate P:297-302; not divided by V) */
dfvm_status dfvm_fvc_div(dfvm_mesh* m, const dfvm_field* face_flux, dfvm_field* out, dfvm_stream stream);
/* y_c = sum_f s_cf gamma_f [delta_f (x_N - x_O) + k_f . (grad x)_f] + sum_{b fixed} gamma_O delta_b (x_b - x_c)
 * (eq:nonortho_flux P:240-250).  gamma NULL -> 1; grad NULL -> Gauss gradient of x. */
dfvm_status dfvm_fvm_laplacian_apply(dfvm_mesh* m, const dfvm_field* gamma, const dfvm_bcs* b, char field,
                                     const dfvm_field* x, const dfvm_field* grad, dfvm_field* y,
                                     dfvm_stream stream);

/* --------------------------------------------------------------- solver */
typedef struct {
  double nu, dt, rho;           /* kinematic viscosity, time step, density (Windkessel only, A-23) */
  int32_t n_corr;               /* PISO correctors ("typically twice") */
  int32_t n_nonorth;            /* non-orthogonal correctors per pressure solve (A-15) */
  int32_t convection;           /* 0 upwind (eq:upwind), 1 central (A-7), 2 SOU and 3 QUICK by
                                   deferred correction (eq:deferred_correction P:193-199,
                                   eq:sou P:200-206, QUICK reading of SPEC.md:233) */
  int64_t p_ref_cell;           /* original numbering; used when no fixed-value p patch exists (A-12) */
  double p_ref_value;
  double p_tol, p_rel_tol, p_rel_tol_final; int32_t p_maxit;  /* A-13 stopping rule */
  double U_tol, U_rel_tol; int32_t U_maxit;
  int32_t p_precond;            /* pressure CG preconditioner: 0 Jacobi (A-14), 1 aggregation-AMG
                                   cycle in the solver's precision (amg.cu),
                                   2 the same AMG with its hierarchy stored and cycled in fp32 under
                                   an fp64 PCG (residual, dots and iterates stay fp64; = 1 for fp32
                                   solvers).  Out of range -> DFVM_E_ARG. */
  int32_t time_scheme;          /* momentum / transport time scheme (Table 1; A-40, the
                                   theta method on the spatial operator A_s:
                                   (V/dt + theta A_s) x* = V/dt x^n + b_s - (1 - theta) A_s x^n):
                                   DFVM_TIME_BACKWARD_EULER (0, theta 1, default), DFVM_TIME_CRANK_NICOLSON
                                   (theta 1/2), DFVM_TIME_FORWARD_EULER (theta 0: diagonal predictor).
                                   Out of range -> DFVM_E_INVALID_ARG. */
  int32_t ddt_corr;             /* 1: add OpenFOAM's Euler ddtCorr Rhie-Chow term to phiHbyA on internal faces
                                   (A-42): rAU_f c_f (phi^n - U^n_f . S_f) / dt with
                                   c_f = 1 - min(|phi^n - U^n_f . S_f| / (|phi^n| + 1e-15), 1);
                                   0 (default): the paper's form without it (A-9) */
  double cont_tol;              /* continuity check ("divergence check failure -> ContinuityViolation";
                                   S:474 "max cell |sum mdot_f| <= 10 x pressure tolerance"): > 0 -> after the
                                   step, max_c |D_c(phi)| > cont_tol returns DFVM_E_CONTINUITY (the step is
                                   committed and the report filled, so the caller sees the offending value);
                                   0 (default): reported only */
} dfvm_piso_opts;
enum { DFVM_TIME_BACKWARD_EULER = 0, DFVM_TIME_CRANK_NICOLSON = 1, DFVM_TIME_FORWARD_EULER = 2 };

/* Krylov stopping rule (A-13): b = 0 -> x = 0, 0 iterations; else
 * stop when ||r||_2 <= max(tol ||b||_2, rel_tol ||r_0||_2), or at maxit; for
 * tol < 1e-12 also on stagnation at the round-off plateau (no new minimum for
 * max(50, best_it) iterations once the best residual is <= 1e-8 ||r_0||, A-13''). */
typedef struct { int32_t it; double res0, res; int32_t converged; } dfvm_solve_report;
typedef struct {
  dfvm_solve_report U[3];
  dfvm_solve_report p[16];
  int32_t n_p;                   /* number of pressure solves in the step */
  double cont_err_max, cont_err_sum;   /* max_c |D_c(phi)|, sum_c |D_c(phi)| */
  int32_t n_outlets;
  double Q[64], p_o[64];         /* Windkessel outlet flow and pressure of the last corrector */
  int32_t nonfinite;
  int32_t gpu_launches;          /* kernels launched by this call */
} dfvm_step_report;

typedef struct dfvm_solver dfvm_solver;
dfvm_status dfvm_solver_create(dfvm_mesh* m, dfvm_bcs* b, const dfvm_piso_opts* opts, dfvm_solver** out);
/* One pressure solve (eq:pressure_poisson P:337-340): A_p(rAU) p = rhs with
 * (A_p x)_c = sum_f c_f (x_c - x_nb) + sum_{b fixed p} c_b x_c,
 * c_f = (w rAU_O + (1-w) rAU_N) delta_f, c_b = rAU_O delta_b, the gauge of
 * A-12 when no fixed-value p patch exists; Jacobi CG warm-started from p. */
dfvm_status dfvm_pressure_solve(dfvm_solver* s, const dfvm_field* rAU, const dfvm_field* rhs, dfvm_field* p,
                                double tol, double rel_tol, int32_t maxit, dfvm_solve_report* rep,
                                dfvm_stream stream);
/* Momentum LDU of §8(c) O-5 from (U^n, phi^n, grad U^n): writes diag[cells]
 * and b[cells][3] (time, BC and explicit non-orthogonal terms; no pressure). */
dfvm_status dfvm_momentum_assemble(dfvm_solver* s, const dfvm_field* U, const dfvm_field* phi, dfvm_field* diag,
                                   dfvm_field* b, dfvm_stream stream);
/* y = M x with the last assembled momentum matrix, x, y: [cells][3] */
dfvm_status dfvm_momentum_apply(dfvm_solver* s, const dfvm_field* x, dfvm_field* y, dfvm_stream stream);
/* ---- NEXT-3: adjoint pieces of the implicit differentiation (
 * eq:vjp P:352-358, eq:implicit_diff P:366-370) ---- */
/* y = M^T x with the last assembled momentum (or transport) matrix, x, y:
 * [cells][3]; the transposed coefficients are written by the assembly (for
 * each incidence, the coefficient the other row holds for this face). */
dfvm_status dfvm_momentum_apply_transpose(dfvm_solver* s, const dfvm_field* x, dfvm_field* y, dfvm_stream stream);
/* Adjoint pressure solve A_p(rAU)^T lambda = g, "solved using the same
 * iterative solver as the forward pass": A_p is symmetric (c_f enters
 * both rows alike, the gauge of A-12 doubles a diagonal entry), so this is the
 * forward PCG on the same coefficients with the adjoint right-hand side g
 * (the gauge's right-hand-side term belongs to the forward system and is not
 * added).  lambda: warm start in, solution out.  Errors as dfvm_pressure_solve. */
dfvm_status dfvm_pressure_solve_adjoint(dfvm_solver* s, const dfvm_field* rAU, const dfvm_field* g, dfvm_field* lambda,
                                        double tol, double rel_tol, int32_t maxit, dfvm_solve_report* rep,
                                        dfvm_stream stream);
/* Gradient of a loss through a converged pressure solve A_p(rAU) p = rhs
 * (rhs held fixed, the gauge's term included): grad = dL/drAU [cells] from
 * p and lambda = A_p^-T dL/dp (implicit function theorem, eq:implicit_diff):
 * dL/dc_f = -(lambda_O - lambda_N)(p_O - p_N) per internal face (+ the gauge
 * row's lambda_r (p_ref - p_r)), -lambda_O p_O per fixed-value boundary face,
 * chained through c_f = (w rAU_O + (1-w) rAU_N) delta_f, c_b = rAU_O delta_b.
 * The boundary conditions are the solver's ('p'). */
dfvm_status dfvm_pressure_vjp(dfvm_solver* s, const dfvm_field* p, const dfvm_field* lambda, dfvm_field* grad,
                              dfvm_stream stream);
/* One implicit-Euler step of passive-scalar transport (NEXT-1; §3.1.2
 * P:477-491): dx/dt + div(phi x) - div(gamma grad x) = 0 with the face flux
 * phi [faces] fixed, field 's' boundary conditions, the solver's dt,
 * convection scheme and U_* tolerances; x [cells] updated in place.
 * Uses (and overwrites) the solver's transport matrix workspace. */
dfvm_status dfvm_transport_step(dfvm_solver* s, dfvm_field* x, const dfvm_field* phi, double gamma,
                                dfvm_solve_report* rep, dfvm_stream stream);
/* One PISO step (§8(c) O-6) advancing U [cells][3], p [cells],
 * phi [faces] in place. */
dfvm_status dfvm_piso_step(dfvm_solver* s, dfvm_field* U, dfvm_field* p, dfvm_field* phi, dfvm_step_report* rep,
                           dfvm_stream stream);
/* Windkessel RCR outlet (eq:windkessel_ode/discrete P:403-425): scheme 0
 * exact, 1 forward Euler, 2 backward Euler.  Sets the patch's p BC. */
dfvm_status dfvm_windkessel_set(dfvm_solver* s, int32_t patch, double Rp, double C, double Rd, double pc0,
                                int32_t scheme);
dfvm_status dfvm_windkessel_state(const dfvm_solver* s, int32_t patch, double* pc);
/* pure host scalar update (tests); the solver runs the device copy */
dfvm_status dfvm_windkessel_update(double pc, double Q, double dt, double Rp, double C, double Rd,
                                   int32_t scheme, double* pc_new, double* p_o);
dfvm_status dfvm_solver_destroy(dfvm_solver* s);

/* Live kernel timing for the roofline report: when on, the solver brackets
 * its pressure-CG kernels with CUDA events on the launching stream and
 * accumulates the durations of the iterations that actually ran.
 * ms[0]/count[0]: the PCG SpMV kernel (q = A p, p.q partials); ms[1]/count[1]:
 * one whole PCG iteration (p update, SpMV, r update, and with AMG the
 * preconditioner cycle and r.z).  With AMG: ms[2]/count[2] the level-0
 * residual SpMV of the V-cycle, ms[3]/count[3] the level-0 post-smoothing
 * SpMV.  set_timing resets the accumulators. */
dfvm_status dfvm_solver_set_timing(dfvm_solver* s, int32_t on);
dfvm_status dfvm_solver_get_timing(const dfvm_solver* s, double ms[4], int64_t count[4]);
/* AMG hierarchy (built at the first AMG pressure solve): number of levels,
 * rows per level and real off-diagonal matrix entries per level (sizes[] and
 * nnz[] may be NULL; at most 16 levels). */
dfvm_status dfvm_solver_amg_levels(const dfvm_solver* s, int32_t* n_levels, int64_t* sizes, int64_t* nnz);

/* Per-kernel live profile (north star "achieved HBM GB/s
 * ... for every kernel").  dfvm_solver_profile(s, 1) clears the table and
 * brackets every kernel launch of the following solver calls (piso_step,
 * pressure_solve, transport_step) with CUDA events on the launching stream;
 * AMG-PCG chunks are then captured and replayed as CUDA graphs one chunk at a
 * time, so the events time the GPU, not the host enqueue.  Rows aggregate
 * by (kernel, AMG level): launches, summed event time, summed algorithmic
 * bytes (the per-launch formulas of DESIGN.md §6).  Launches of Krylov
 * iterations the device skipped (solve already converged, the kernel exits
 * on the done flag) are booked to the row "(no-op launches after
 * convergence)" with zero bytes.  Profiling adds event nodes and disables the
 * cached chunk graphs: time the step itself with profiling off.
 * dfvm_solver_profile_get copies min(cap, n) rows and sets *n to the row
 * count. */
typedef struct {
  char name[48];        /* __global__ kernel name, "k_grad (U)" / "k_grad (p)" for the Gauss gradients */
  int32_t level;        /* AMG level the kernel runs on, -1 outside the AMG cycle */
  int64_t launches;
  double ms;            /* summed event-pair time */
  double alg_bytes;     /* summed algorithmic bytes */
} dfvm_kernel_stat;
dfvm_status dfvm_solver_profile(dfvm_solver* s, int32_t on);
dfvm_status dfvm_solver_profile_get(const dfvm_solver* s, dfvm_kernel_stat* out, int32_t cap, int32_t* n);

/* Kernel launch counter (all kernels this process launched through the
 * library), for bench.py's gpu_launches claim. */
int64_t dfvm_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* DFVM_H */
