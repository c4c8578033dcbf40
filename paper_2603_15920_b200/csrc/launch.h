// launch.h — host-callable kernel launchers (implemented in the .cu files).
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace dfvm {

// ---- import / export (ops.cu)
template <class T>
void launch_import(T* dst, const double* src, const int32_t* map, int64_t n, int nc, bool oriented,
                   cudaStream_t s);
template <class T>
void launch_export(double* dst, const T* src, const int32_t* map, int64_t n, int nc, bool oriented,
                   cudaStream_t s);

// ---- operators (ops.cu); bkind/bval: per non-empty boundary face BC
template <class T>
void launch_interpolate(const DevMesh<T>& M, const T* x, int nc, const uint8_t* bkind, const T* bval, T* xf,
                        cudaStream_t s);
template <class T>
void launch_grad(const DevMesh<T>& M, const T* x, int nc, const uint8_t* bkind, const T* bval, T* G,
                 cudaStream_t s);
template <class T>
void launch_grad_faces(const DevMesh<T>& M, const T* fv, int nc, T* G, cudaStream_t s);
template <class T>
void launch_div(const DevMesh<T>& M, const T* flux, T* out, cudaStream_t s);
template <class T>
void launch_laplacian(const DevMesh<T>& M, const T* gamma, const T* x, const T* G, const uint8_t* bkind,
                      const T* bval, T* y, cudaStream_t s);

}  // namespace dfvm
