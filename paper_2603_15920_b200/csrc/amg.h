// amg.h — aggregation-AMG preconditioner for the pressure PCG (amg.cu).
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace dfvm {

struct Prof;

template <class T> struct Amg;
// hierarchy from the mesh topology (host, once per mesh); fp32: store and
// cycle the hierarchy in fp32 under an fp64 solver ("amg32")
template <class T> dfvm_status amg_create(dfvm_mesh* m, const DevMesh<T>& M, bool fp32, Amg<T>** out);
template <class T> void amg_destroy(Amg<T>* A);
template <class T> int amg_levels(const Amg<T>* A, int* sizes);
// Galerkin values + l1 diagonals for the current pressure matrix (pcoef, pdiag)
template <class T> dfvm_status amg_update(Amg<T>* A, const T* pcoef, const T* pdiag, cudaStream_t s, int* n_launch,
                                          Prof* prof);
// z = M^-1 r, one cycle; every kernel exits early when *done != 0.  ev (may be
// NULL): 4 events recorded around the level-0 residual SpMV (ev[0..1]) and
// the level-0 post-smoothing SpMV (ev[2..3]) for live timing.
template <class T> dfvm_status amg_apply(Amg<T>* A, const T* r, T* z, const int* done, cudaStream_t s, int* n_launch,
                                         cudaEvent_t* ev, Prof* prof);
// real off-diagonal entries per level; returns the level count
template <class T> int amg_level_nnz(const Amg<T>* A, int64_t* nnz);

}  // namespace dfvm
