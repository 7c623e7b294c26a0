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

// ---------------------------------------------------------------------------
// Staging of row segments into shared memory with batched 16-byte loads.
// Row r supplies elements j = st + dir*e, e in [0, W), of a contiguous source
// row `ptr` whose valid indices are [0, width) (others read as 0).  Each thread
// first issues up to ITEMS independent LDG.128 (chunk-aligned), then scatters
// the elements through dst(r, e, bits): load latency is overlapped instead of
// serialised element by element.
template <class In>
struct RowSrc {
    const In *ptr;
    int st, dir, width;
};

template <class In>
__device__ __forceinline__ uint32_t chunk_elem(const uint4 &v, int q) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if constexpr (sizeof(In) == 1) return (w[q >> 2] >> (8 * (q & 3))) & 0xFFu;
    else if constexpr (sizeof(In) == 2) return (w[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
    else return w[q];
}

__device__ __forceinline__ int floor_div(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

template <class In, int ITEMS, class RowFn, class DstFn>
__device__ __forceinline__ void stage_rows(int nrows, int W, RowFn &&rowfn, DstFn &&dst) {
    constexpr int EPC = 16 / (int)sizeof(In);
    const int nch = (W + EPC - 1) / EPC + 1;
    const int items = nrows * nch;
    const int nthr = blockDim.x;
    for (int base = threadIdx.x; base < items; base += nthr * ITEMS) {
        uint4 v[ITEMS];
        int cbs[ITEMS], rs[ITEMS];
        RowSrc<In> src[ITEMS];
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            const int it = base + u * nthr;
            v[u] = make_uint4(0u, 0u, 0u, 0u);
            rs[u] = -1;
            if (it < items) {
                const int r = it / nch, ch = it - r * nch;
                const RowSrc<In> ri = rowfn(r);
                const int jlo = ri.dir > 0 ? ri.st : ri.st - W + 1;
                const int cb = floor_div(jlo, EPC) * EPC + ch * EPC;
                rs[u] = r;
                cbs[u] = cb;
                src[u] = ri;
                if (cb >= 0 && cb < ri.width) v[u] = __ldg(reinterpret_cast<const uint4 *>(ri.ptr + cb));
            }
        }
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            if (rs[u] < 0) continue;
            const RowSrc<In> ri = src[u];
#pragma unroll
            for (int q = 0; q < EPC; ++q) {
                const int j = cbs[u] + q;
                const int e = ri.dir > 0 ? j - ri.st : ri.st - j;
                if (e >= 0 && e < W) dst(rs[u], e, (j >= 0 && j < ri.width) ? chunk_elem<In>(v[u], q) : 0u);
            }
        }
    }
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
