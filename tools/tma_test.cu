// Minimal TMA sanity test (debug aid): 2D u16 tensor, box {BW,1}, OOB zero fill.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "tma.cuh"
using namespace d3;

template <bool FENCE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap *gtm, uint16_t *out, int x0, int bw, int useg) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 4096);
    if (threadIdx.x == 0) { mbar_init(bar, 1); if (FENCE) fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, 4 * bw * 2);
        for (int r = 0; r < 4; ++r) tma_load_2d(sm + r * 256, useg ? gtm : &tm, x0 + r, r, bar);
    }
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < 4 * bw; i += blockDim.x) out[i] = reinterpret_cast<uint16_t *>(sm + (i / bw) * 256)[i % bw];
}

int main(int argc, char **argv) {
    int x0 = atoi(argv[1]), bw = atoi(argv[2]), W = atoi(argv[3]), fence = atoi(argv[4]), useg = atoi(argv[5]), prom = atoi(argv[6]);
    const int P = 128, ROWS = 8;
    uint16_t h[ROWS * P];
    for (int i = 0; i < ROWS * P; ++i) h[i] = (uint16_t)(i + 1);
    uint16_t *d, *o;
    CUtensorMap *gtm;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 4 * 256 * 2);
    cudaMalloc(&gtm, sizeof(CUtensorMap));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)W, ROWS};
    cuuint64_t str[1] = {P * 2};
    cuuint32_t box[2] = {(cuuint32_t)bw, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    if (fence) k<true><<<1, 128, 8192>>>(tm, gtm, o, x0, bw, useg);
    else k<false><<<1, 128, 8192>>>(tm, gtm, o, x0, bw, useg);
    cudaError_t e = cudaDeviceSynchronize();
    uint16_t ho[4 * 256] = {0};
    cudaMemcpy(ho, o, 4 * bw * 2, cudaMemcpyDeviceToHost);
    printf("prom=%d x0=%d bw=%d W=%d fence=%d useg=%d encode=%d kernel=%s | r0: %d %d %d %d .. %d | r3: %d %d\n", prom, x0, bw, W, fence,
           useg, (int)r, cudaGetErrorString(e), ho[0], ho[1], ho[2], ho[3], ho[bw - 1], ho[3 * bw], ho[3 * bw + bw - 1]);
    return 0;
}
