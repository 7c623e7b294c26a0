// k_drt_f32.cu -- kernel instantiations for one input dtype (see launch.cuh).
#include "launch.cuh"

namespace d3 {
drt3d_status dispatch_drt_f32(int K, int sin, int sout, bool first, bool fin, const DrtPass &prm, int ninst, cudaStream_t st) {
    D3_DRT_CASE(ST_F32, ST_F32, true, true, float, float, float)
    D3_DRT_CASE(ST_F32, ST_F32, true, false, float, float, float)
    D3_DRT_CASE(ST_F32, ST_F32, false, true, float, float, float)
    D3_DRT_CASE(ST_F32, ST_F32, false, false, float, float, float)
    return DRT3D_ERR_UNSUPPORTED;
}
}  // namespace d3
