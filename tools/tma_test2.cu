// mbarrier / bulk-copy / TMA micro tests (debug aid)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "tma.cuh"
using namespace d3;

__global__ void k(int mode, const __grid_constant__ CUtensorMap tm, const uint16_t *src, uint16_t *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 4096);
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
        } else if (mode == 1) {
            mbar_arrive_expect_tx(bar, 256);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm)),
                         "l"(src), "r"(256), "r"(smem_u32(bar)) : "memory");
        } else {
            mbar_arrive_expect_tx(bar, 128);
            tma_load_2d(sm, &tm, 0, 0, bar);
        }
    }
    mbar_wait(bar, 0);
    if (threadIdx.x < 64) out[threadIdx.x] = reinterpret_cast<uint16_t *>(sm)[threadIdx.x];
}

int main(int argc, char **argv) {
    int mode = atoi(argv[1]);
    uint16_t h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = (uint16_t)(i + 1);
    uint16_t *d, *o;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 256);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, 8};
    cuuint64_t str[1] = {256};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 64, 8192>>>(mode, tm, d, o);
    cudaError_t e = cudaDeviceSynchronize();
    uint16_t ho[64] = {0};
    cudaMemcpy(ho, o, 128, cudaMemcpyDeviceToHost);
    int dev; cudaGetDevice(&dev); cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
    printf("mode=%d encode=%d kernel=%s  out: %d %d %d  (cc %d.%d, drv)\n", mode, (int)r, cudaGetErrorString(e), ho[0], ho[1], ho[63], pr.major, pr.minor);
    return 0;
}
