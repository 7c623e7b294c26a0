// k_djt_i32.cu -- kernel instantiations for one input dtype (see launch.cuh).
#include "launch.cuh"

namespace d3 {
drt3d_status dispatch_djt_i32(int K, int sin, int sout, bool first, bool fin, const DjtPass &prm, int ninst, cudaStream_t st) {
    D3_DJT_CASE(ST_U32, ST_U32, true, true, uint32_t, uint32_t, uint32_t)
    D3_DJT_CASE(ST_U32, ST_U32, true, false, uint32_t, uint32_t, uint32_t)
    D3_DJT_CASE(ST_U32, ST_U32, false, true, uint32_t, uint32_t, uint32_t)
    D3_DJT_CASE(ST_U32, ST_U32, false, false, uint32_t, uint32_t, uint32_t)
    return DRT3D_ERR_UNSUPPORTED;
}
}  // namespace d3
