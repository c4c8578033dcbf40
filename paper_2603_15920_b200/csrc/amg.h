// amg.h — aggregation-AMG preconditioner for the pressure PCG (amg.cu).
#pragma once
#include <cuda_runtime.h>

#include "internal.h"
#include "krylov.cuh"

namespace dfvm {

struct Prof;

template <class T> struct Amg;
// hierarchy from the mesh topology (host, once per mesh); fp32: store and
// cycle the hierarchy in fp32 under an fp64 solver ("amg32")
template <class T> dfvm_status amg_create(dfvm_mesh* m, const DevMesh<T>& M, bool fp32, Amg<T>** out, cudaStream_t s);
template <class T> void amg_destroy(Amg<T>* A);
template <class T> int amg_levels(const Amg<T>* A, int* sizes);
// Galerkin values + l1 diagonals for the current pressure matrix (pcoef, pdiag)
template <class T> dfvm_status amg_update(Amg<T>* A, const T* pcoef, const T* pdiag, cudaStream_t s, int* n_launch,
                                          Prof* prof);
// z = M^-1 r, one cycle; every kernel exits early when *done != 0.  ev (may be
// NULL): 4 events recorded around the level-0 residual SpMV (ev[0..1]) and
// the level-0 post-smoothing SpMV (ev[2..3]) for live timing.
// dot (may be NULL): fold r.z into the level-0 post-smoother (its kind and
// reduction target); *dot_done tells whether it was folded.  pre_done: the
// caller already wrote the level-0 pre-smoothed x0 = r / d1 (amg_level0_pre).
template <class T> dfvm_status amg_apply(Amg<T>* A, const T* r, T* z, const int* done, cudaStream_t s, int* n_launch,
                                         cudaEvent_t* ev, Prof* prof, const KDot* dot = nullptr,
                                         bool pre_done = false, bool* dot_done = nullptr);
// level-0 pre-smoothing target for a caller that fuses x0 = r * il1 into its
// own pass: x0 and il1 in the hierarchy's type (p_bytes 4 or 8), or NULL when
// the cycle has a single level
template <class T> void amg_level0_pre(Amg<T>* A, void** x0, const void** il1, int* p_bytes);
// real off-diagonal entries per level; returns the level count
template <class T> int amg_level_nnz(const Amg<T>* A, int64_t* nnz);

}  // namespace dfvm
