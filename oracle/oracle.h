// oracle/oracle.h — internal header of the CPU oracle.
//
// TEST INFRASTRUCTURE ONLY.  The oracle is a plain, slow, single-threaded
// fp64 C++ transcription of DiFVM's finite-volume discretisation and PISO
// step (§2.3-§2.6) in the readings of SURVEY.md §8(c).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load liboracle.so.  It shares no code, header, table or helper with
// the CUDA library (paper_2603_15920_b200/); it works in the caller's
// original cell/face numbering.
//
// Summation order (SURVEY.md §8(c) "Oracle rules"): faces are visited in
// ascending face index (internal faces, then boundary patches in patch
// order); every cell accumulator receives its contributions in that order;
// dot products run in ascending cell order.
//
// Pins: every part is pinned by a closed form, a hand value or
// an already-pinned operator (tests/test_oracle_*.py), including the parts
// round 1 left unpinned: the explicit non-orthogonal momentum correction
// (O-5, by hand on a w = 3/4 two-cell fixture and against the pinned
// Laplacian), the non-orthogonal pressure right-hand side and Rhie-Chow flux
// term (A-9, by hand), the Windkessel coupling inside PISO (A-19: exact RCR
// fixed point, per-corrector recurrence) and the partition emulation (O-10,
// bitwise against the global apply) and the optional ddtCorr term (A-42, by
// hand on the same fixture, both branches of its min()) —
// tests/test_oracle_pins_r2.py.  No part is left "parity unpinned".
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace orc {

enum Status {
  OK = 0, E_INVALID_ARG, E_MESH_CONSISTENCY, E_DEGENERATE_FACE, E_INVERTED_CELL,
  E_NONCONVEX_PAIR, E_EXTREME_NONORTH, E_MISSING_BC, E_NOT_CONVERGED, E_BREAKDOWN,
  E_NONFINITE, E_CONTINUITY, E_INVALID_WK_PARAMS
};

void set_error(int code, const std::string& msg, int64_t index);

enum PatchKind { PK_GENERIC = 0, PK_WALL = 1, PK_EMPTY = 2 };
enum NonOrth { NO_NONE = 0, NO_MINIMUM = 1, NO_ORTHOGONAL = 2, NO_OVERRELAXED = 3 };
enum BcKind { BC_FIXED = 0, BC_ZEROGRAD = 1, BC_PARABOLIC = 2, BC_WINDKESSEL = 3, BC_UNSET = -1 };

struct Mesh {
  int64_t N = 0;      // cells
  int64_t F = 0;      // internal faces
  int64_t NF = 0;     // all faces
  std::vector<int32_t> owner, neigh;          // [NF], [F]
  std::vector<int> pkind;                     // per patch
  std::vector<int64_t> pstart, pn;            // per patch
  std::vector<int> face_patch;                // [NF - F]
  // O-1 geometry
  std::vector<double> Sf, xf;                 // [NF][3]
  std::vector<double> xc, V;                  // [N][3], [N]
  int64_t n_bad_pyramids = 0;
  // O-2 connectivity: per cell, faces in ascending face index
  std::vector<int64_t> cptr;                  // [N+1]
  std::vector<int64_t> cface;                 // face index
  // O-3 coefficients
  int nonorth = NO_OVERRELAXED;
  std::vector<double> w, delta, kf;           // [F], [F], [F][3]
  std::vector<double> delta_b;                // [NF - F] (0 on empty faces)
  int64_t n_clamped = 0;
  bool is_empty_face(int64_t f) const { return f >= F && pkind[face_patch[f - F]] == PK_EMPTY; }
};

struct BC {
  int kind = BC_UNSET;
  double value[3] = {0, 0, 0};
  double u_max = 0, center[3] = {0, 0, 0}, radius = 1;
  // time-varying multiplier of a fixed / parabolic value (
  // reading A-41): g(t) = a_0 + sum_{k=1..nh} a_k cos(2 pi k t/T) + b_k sin(2 pi k t/T)
  int nh = -1;                 // -1: steady
  double period = 1, wa[17] = {0}, wb[17] = {0};
};

struct BCs {
  const Mesh* m = nullptr;
  // per patch, per field 0 = 'U', 1 = 'p', 2 = 's' (generic scalar)
  std::vector<BC> bc[3];
  std::vector<double> wk_value;   // per patch: current Windkessel p BC value (p_o / rho)
  double t_eval = 0;              // time at which time-varying values are evaluated (t^{n+1} in a step)
};
double waveform(const BC& bc, double t);

int field_index(char fld);

// face value of field `fld` (n_comp components) on boundary face f (f >= F)
void boundary_value(const Mesh& m, const BCs& b, int fi, int ncomp, const double* x,
                    int64_t f, double* out);
bool is_fixed(const BCs& b, int fi, int64_t patch);   // fixed-value kind (incl. parabolic, Windkessel)

// operators (original numbering)
void interpolate(const Mesh& m, const BCs& b, int fi, int ncomp, const double* x, double* xf);
void grad_from_faces(const Mesh& m, int ncomp, const double* fv, double* g);
void grad(const Mesh& m, const BCs& b, int fi, int ncomp, const double* x, double* g);
void div(const Mesh& m, const double* flux, double* out);
void laplacian(const Mesh& m, const BCs& b, int fi, const double* gamma, const double* x,
               const double* g_in, double* y, double* yabs);

// LDU matrix over the internal faces (OpenFOAM addressing): row O col N = upper,
// row N col O = lower.
struct LDU {
  std::vector<double> diag, lower, upper;
};
void ldu_apply(const Mesh& m, const LDU& A, const double* x, double* y);

struct SolveReport { int it = 0; double res0 = 0, res = 0; int converged = 0; int status = 0; };
SolveReport cg(const Mesh& m, const LDU& A, const double* b, double* x, double tol, double rel_tol, int maxit);
SolveReport bicgstab(const Mesh& m, const LDU& A, const double* b, double* x, double tol, double rel_tol, int maxit);
SolveReport dense_solve(const Mesh& m, const LDU& A, const double* b, double* x);

}  // namespace orc
