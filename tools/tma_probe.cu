// TMA start-coordinate probe (debug aid): one 2D box {64,1} of u16 at (x, y).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "tma.cuh"
using namespace d3;
__global__ void k(const __grid_constant__ CUtensorMap tm, uint16_t *out, int x, int y, int nops) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 8192);
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, 128 * nops);
        for (int i = 0; i < nops; ++i) tma_load_2d(sm + 256 * i, &tm, x, y + i, bar);
    }
    mbar_wait(bar, 0);
    if (threadIdx.x < 64) out[threadIdx.x] = reinterpret_cast<uint16_t *>(sm)[threadIdx.x];
}
int main(int argc, char **argv) {
    int x = atoi(argv[1]), y = atoi(argv[2]), nops = atoi(argv[3]);
    uint16_t h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = (uint16_t)(i + 1);
    uint16_t *d, *o;
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 256);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    void *f = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, 8}; cuuint64_t str[1] = {256};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 64, 8192 + 64>>>(tm, o, x, y, nops);
    cudaError_t e = cudaDeviceSynchronize();
    uint16_t ho[64] = {0};
    cudaMemcpy(ho, o, 128, cudaMemcpyDeviceToHost);
    printf("x=%d y=%d nops=%d encode=%d kernel=%s out: %d %d .. %d\n", x, y, nops, (int)r, cudaGetErrorString(e), ho[0], ho[1], ho[63]);
    return 0;
}
