// Microbenchmark + correctness probe (debug aid, not product code):
// per-row 2D TMA boxes at arbitrary element starts (u16 rows, zero-filled OOB)
// into shared memory at a chosen slot pitch, vs. cp.async 16-byte chunks.
// usage: tma_rows_bench <mode 0=tma-1thread 1=tma-32lanes 2=cpasync> <slot_pitch_bytes>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

static __device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int BW = 96, ROWS = 256, W = 288;

__device__ __forceinline__ int row_start(long long row) { return (((int)((row * 37) % 300) - 30) / 8) * 8; }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const uint16_t *src, int nrows_total, int sp,
                  unsigned long long *sink, int iters) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + ROWS * sp);
    const int tid = threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        const long long g = (long long)blockIdx.x + (long long)it * gridDim.x;
        const long long row0 = (g * ROWS) % nrows_total;
        if (MODE == 0 || MODE == 1) {
            if (MODE == 0 ? tid == 0 : tid < 32) {
                if (tid == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(ROWS * BW * 2));
                if (MODE == 1) __syncwarp();
                for (int r = (MODE == 0 ? 0 : tid); r < ROWS; r += (MODE == 0 ? 1 : 32)) {
                    const int x = row_start(row0 + r), y = (int)(row0 + r);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                            su32(sm + r * sp)),
                        "l"(&tm), "r"(x), "r"(y), "r"(su32(bar))
                        : "memory");
                }
            }
            // wait phase `it & 1`
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(su32(bar)), "r"(it & 1)
                    : "memory");
            }
        } else if (MODE == 3) {
            // plain LDG.128 -> STS.128 (4 loads in flight per thread)
            const int NCH = BW / 8 + 1;
            for (int base = tid; base < ROWS * NCH; base += 4 * blockDim.x) {
                uint4 v[4];
                int dsto[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = base + u * blockDim.x;
                    dsto[u] = -1;
                    v[u] = make_uint4(0, 0, 0, 0);
                    if (i < ROWS * NCH) {
                        const int r = i / NCH, c = i % NCH;
                        const int st = row_start(row0 + r);
                        const int cc = (st >> 3) + c;
                        if (cc >= 0 && cc < W / 8) v[u] = __ldg(reinterpret_cast<const uint4 *>(src + (row0 + r) * W + cc * 8));
                        dsto[u] = r * sp + 16 * c;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (dsto[u] >= 0) *reinterpret_cast<uint4 *>(sm + dsto[u]) = v[u];
            }
        } else {
            // cp.async 16-byte chunks covering [st, st + BW) (aligned source chunks; no realign)
            const int NCH = BW / 8 + 1;
            for (int i = tid; i < ROWS * NCH; i += blockDim.x) {
                const int r = i / NCH, c = i % NCH;
                const int st = row_start(row0 + r);
                const int cc = (st >> 3) + c;
                const bool ok = cc >= 0 && cc < W / 8;
                const uint16_t *s = ok ? src + (row0 + r) * W + cc * 8 : src;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(sm + r * sp + 16 * c)), "l"(s),
                             "r"(ok ? 16 : 0)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        // consume a little so the load is not dead
        for (int i = tid; i < ROWS; i += blockDim.x) acc += *reinterpret_cast<const uint16_t *>(sm + i * sp + 2 * (i % BW));
        if (it == 0 && blockIdx.x == 0) {
            // verify the whole tile against global memory
            for (int i = tid; i < ROWS * BW; i += blockDim.x) {
                const int r = i / BW, e = i % BW;
                const int j = row_start(row0 + r) + e;
                uint16_t expect = (j >= 0 && j < W) ? src[(row0 + r) * W + j] : 0;
                uint16_t got;
                if (MODE >= 2) {
                    const int st = row_start(row0 + r);
                    const int jj = j - ((st >> 3) << 3);
                    got = *reinterpret_cast<const uint16_t *>(sm + r * sp + 2 * jj);
                } else {
                    got = *reinterpret_cast<const uint16_t *>(sm + r * sp + 2 * e);
                }
                if (got != expect) atomicAdd(sink + 1, 1ull);
            }
        }
        __syncthreads();
    }
    atomicAdd(sink, acc);
}

int main(int argc, char **argv) {
    const int mode = atoi(argv[1]), sp = atoi(argv[2]);
    const int nrows = 65536;
    std::vector<uint16_t> h((size_t)nrows * W);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
    uint16_t *d;
    unsigned long long *sink;
    cudaMalloc(&d, h.size() * 2);
    cudaMalloc(&sink, 16);
    cudaMemset(sink, 0, 16);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)nrows};
    cuuint64_t str[1] = {W * 2};
    cuuint32_t box[2] = {BW, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = ROWS * sp + 64;
    auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = (argc > 4) ? atoi(argv[4]) : 296, iters = 40;
    if (argc > 3 && argv[3][0] == 'c') {   // explicit 1-CTA cluster launch
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(160); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t le = cudaLaunchKernelEx(&cfg, kern, tm, (const uint16_t *)d, nrows, sp, sink, 1);
        cudaError_t se = cudaDeviceSynchronize();
        unsigned long long hs[2];
        cudaMemcpy(hs, sink, 16, cudaMemcpyDeviceToHost);
        printf("cluster launch: launch=%s sync=%s mismatches=%llu\n", cudaGetErrorString(le), cudaGetErrorString(se), hs[1]);
        return 0;
    }
    kern<<<grid, 160, smem>>>(tm, d, nrows, sp, sink, 1);   // warm-up + verify
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, 160, smem>>>(tm, d, nrows, sp, sink, iters);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long hs[2];
    cudaMemcpy(hs, sink, 16, cudaMemcpyDeviceToHost);
    const double bytes = (double)grid * iters * ROWS * BW * 2;
    printf("mode=%d sp=%d encode=%d err=%s mismatches=%llu  %.3f ms  %.1f GB/s  (%.2f us per tile-wave, %.0f cyc/tile/CTA @1.9GHz)\n",
           mode, sp, (int)r, cudaGetErrorString(e), hs[1], ms, bytes / ms / 1e6, 1e3 * ms / iters,
           1.9e6 * ms / iters);
    return 0;
}
