// dispatch.h -- per-dtype kernel dispatch entry points (defined in k_*.cu).
#pragma once
#include "drt3d.h"
#include "common.cuh"
#include "djt_kernels.cuh"
#include "drt_kernels.cuh"

namespace d3 {
#define D3_DECL(NAME, PASS) \
    drt3d_status NAME(int K, int sin, int sout, bool first, bool fin, const PASS &prm, int ninst, cudaStream_t st);
D3_DECL(dispatch_drt_u8, DrtPass)
D3_DECL(dispatch_drt_i32, DrtPass)
D3_DECL(dispatch_drt_f32, DrtPass)
D3_DECL(dispatch_djt_u8, DjtPass)
D3_DECL(dispatch_djt_i32, DjtPass)
D3_DECL(dispatch_djt_f32, DjtPass)
#undef D3_DECL
// the separable on-chip N = 32 DRT (k_sep32.cu): two independent CTAs per instance
drt3d_status dispatch_drt_sep32(int in_dtype, const DrtPass &prm, int ninst, cudaStream_t st);
// the one-CTA N = 16 DRT (k_sep16.cu)
drt3d_status dispatch_drt_sep16(int in_dtype, const DrtPass &prm, int ninst, cudaStream_t st);
}  // namespace d3
