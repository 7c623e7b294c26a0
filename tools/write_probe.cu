// Write-only HBM probe: grid-stride 16-byte stores of index-hashed (non-compressible) data.
// Built by hand: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cstdint>
#include <cuda_runtime.h>

__global__ void write_hash(uint4 *out, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u;
        out[i] = make_uint4(h, h ^ 0x9e3779b9u, h * 3u, h + 0x7f4a7c15u);
    }
}

extern "C" int write_probe(void *out, size_t bytes, int blocks, int threads, void *stream) {
    write_hash<<<blocks, threads, 0, (cudaStream_t)stream>>>((uint4 *)out, bytes / 16);
    return (int)cudaGetLastError();
}
