// adjoint.h -- host entry of the backprojection kernels (adjoint.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "drt3d.h"

namespace d3 {
size_t adjoint_workspace_bytes(int transform, int N, uint32_t mask);
drt3d_status run_adjoint(int transform, const void *coef, int N, int n, const int8_t (*rows)[3], uint32_t mask,
                         int batch, int dtype, void *cube, void *ws, cudaStream_t st, int *launches);
}  // namespace d3
