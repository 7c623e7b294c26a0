// common.cuh -- device/host helpers shared by the DRT and DJT kernels of the
// B200 library (product code; independent of oracle/).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace d3 {

// eq:digitalLine, recursive form, restated for the GPU path:
//   l^k_s(u) = l^{k-1}_{floor(s/2)}(u mod 2^{k-1}) + u_{k-1} * floor((s+1)/2).
// Used with compile-time arguments (fully unrolled loops) so every shift of
// the direct radix-2^K sums below is a register index, not a memory access.
__host__ __device__ constexpr int lk(int k, int s, int u) {
    return k == 0 ? 0 : lk(k - 1, s >> 1, u & ((1 << (k - 1)) - 1)) + ((u >> (k - 1)) & 1) * ((s + 1) >> 1);
}

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).  Used
// so that every line offset l^K_r(w) is a constant expression (register
// indexing), which plain `#pragma unroll` does not guarantee.
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// 32-bit lane arithmetic.  Integer paths accumulate in uint32 (exact sum mod
// 2^32, two's-complement wrap for the int32 output); float paths in fp32.
template <class Acc> struct Lane;
template <> struct Lane<uint32_t> {
    static __device__ __forceinline__ uint32_t get(uint32_t b) { return b; }
    static __device__ __forceinline__ uint32_t bits(uint32_t v) { return v; }
};
template <> struct Lane<float> {
    static __device__ __forceinline__ float get(uint32_t b) { return __uint_as_float(b); }
    static __device__ __forceinline__ uint32_t bits(float v) { return __float_as_uint(v); }
};

// element loads/stores converting between storage types and lane types
template <class T> struct Elem;
template <> struct Elem<uint8_t> {
    static __device__ __forceinline__ uint32_t load_bits(const uint8_t *p) { return (uint32_t)__ldg(p); }
};
template <> struct Elem<uint16_t> {
    static __device__ __forceinline__ uint32_t load_bits(const uint16_t *p) { return (uint32_t)__ldg(p); }
};
template <> struct Elem<uint32_t> {
    static __device__ __forceinline__ uint32_t load_bits(const uint32_t *p) { return __ldg(p); }
};
template <> struct Elem<float> {
    static __device__ __forceinline__ uint32_t load_bits(const float *p) { return __float_as_uint(__ldg(p)); }
};

template <class Out, class Acc> __device__ __forceinline__ Out to_out(Acc v);
template <> __device__ __forceinline__ uint16_t to_out<uint16_t, uint32_t>(uint32_t v) { return (uint16_t)v; }
template <> __device__ __forceinline__ uint32_t to_out<uint32_t, uint32_t>(uint32_t v) { return v; }
template <> __device__ __forceinline__ float to_out<float, float>(float v) { return v; }

// streaming (evict-first) 16-byte global store for final outputs that are
// never re-read by this call.
__device__ __forceinline__ void st_cs_v4(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Oriented-cube addressing (Alg. 2 permute + flip as an index remap,
// PAPER.md:342-348, reading A): element (x', y', z') of dodecant k lives at
// off0 + x'*sx + y'*sy + z'*sz in the original [x][y][z] cube.  fast = the
// oriented axis with unit stride (0 = x', 1 = y', 2 = z').
struct Orient {
    long long off0, sx, sy, sz;
    int fast;
    int dod;   // dodecant id k
};

constexpr int kMaxDod = 12;

enum Stor { ST_U8 = 0, ST_U16 = 1, ST_U32 = 2, ST_F32 = 3 };

}  // namespace d3
