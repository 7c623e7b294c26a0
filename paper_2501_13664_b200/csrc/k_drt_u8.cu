// k_drt_u8.cu -- kernel instantiations for one input dtype (see launch.cuh).
#include "launch.cuh"

namespace d3 {
drt3d_status dispatch_drt_u8(int K, int sin, int sout, bool first, bool fin, const DrtPass &prm, int ninst, cudaStream_t st) {
    D3_DRT_CASE(ST_U8, ST_U32, true, true, uint8_t, uint32_t, uint32_t)
    D3_DRT_CASE(ST_U8, ST_U16, true, false, uint8_t, uint32_t, uint16_t)
    D3_DRT_CASE(ST_U8, ST_U32, true, false, uint8_t, uint32_t, uint32_t)
    D3_DRT_CASE(ST_U16, ST_U32, false, true, uint16_t, uint32_t, uint32_t)
    D3_DRT_CASE(ST_U16, ST_U32, false, false, uint16_t, uint32_t, uint32_t)
    D3_DRT_CASE(ST_U32, ST_U32, false, true, uint32_t, uint32_t, uint32_t)
    D3_DRT_CASE(ST_U32, ST_U32, false, false, uint32_t, uint32_t, uint32_t)
    return DRT3D_ERR_UNSUPPORTED;
}
}  // namespace d3

#ifdef D3_PROF_PASS
extern "C" int d3_pass_prof_read(unsigned long long *out16) {
    if (cudaMemcpyFromSymbol(out16, d3_pass_prof, 16 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    unsigned long long z[16] = {0};
    return cudaMemcpyToSymbol(d3_pass_prof, z, sizeof(z)) != cudaSuccess;
}
#endif

#ifdef D3_PROF_SWAR
extern "C" int d3_swar_prof_read(unsigned long long *out16) {
    if (cudaMemcpyFromSymbol(out16, d3::d3_swar_prof, 16 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    unsigned long long z[16] = {0};
    return cudaMemcpyToSymbol(d3::d3_swar_prof, z, sizeof(z)) != cudaSuccess;
}
#endif
