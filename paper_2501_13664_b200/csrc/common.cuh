// common.cuh -- device/host helpers shared by the DRT and DJT kernels of the
// B200 library (product code; independent of oracle/).
#pragma once
#include <atomic>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace d3 {

// ---- host: kernel attributes
template <class KernelT>
bool set_smem(KernelT k, int bytes) {
    // prefer the maximum shared-memory carveout so two CTAs of ~100 KB fit on one SM
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (bytes <= 48 * 1024) return true;
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess;
}

// set_smem once per kernel and device: `done` is one bit per device, a static of the caller's
// launcher instantiation (one per kernel; a static here would be shared by every kernel of the
// same signature).  Function attributes are per device, so a process driving several GPUs sets
// them on each; racing threads may both set them, which is harmless.
template <class KernelT>
bool set_smem_once(KernelT k, int bytes, std::atomic<uint32_t> &done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint32_t bit = 1u << (dev & 31);
    if (done.load(std::memory_order_acquire) & bit) return true;
    const bool ok = set_smem(k, bytes);
    if (ok) done.fetch_or(bit, std::memory_order_release);
    return ok;
}


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

// Two terms into an accumulator (the radix-2^K direct sums take rows two at a time).
// Integer lanes: ~3/8 of the output rows take their two adds as IMAD x*one + acc
// (FMA pipe, `one` a runtime 1) and the rest as one IADD3 (ALU pipe), so the
// two integer-capable pipes share the work.
template <class Acc>
__device__ __forceinline__ Acc add2(Acc acc, uint32_t x, uint32_t y, uint32_t one, bool fma) {
    if constexpr (std::is_same<Acc, uint32_t>::value) {
        if (fma) return x * one + (y * one + acc);
        return acc + x + y;
    } else {
        return acc + Lane<Acc>::get(x) + Lane<Acc>::get(y);
    }
}

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

// ---------------------------------------------------------------------------
// Residual pre-shift of intermediate rows.
// A pass reads stage-c row (s, v) starting at D + s1 w1 + s2 w2 (w = v mod 2^K);
// the writer stores that row shifted left by rho = (s1 w1 + s2 w2) mod EPC
// (EPC = elements per 16-byte chunk), so every reader window starts on a chunk
// boundary and staging is a plain aligned copy.  The writer realigns its
// register runs with one warp shuffle per word and a select network.

// o[i] = w[i + s] for a runtime word shift s in [0, 3] (two SEL stages).
template <int NO, int NW>
__device__ __forceinline__ void shift_words(const uint32_t (&w)[NW], int s, uint32_t (&o)[NO]) {
    static_assert(NW >= NO + 3, "window");
    uint32_t t[NO + 1];
#pragma unroll
    for (int i = 0; i < NO + 1; ++i) t[i] = (s & 2) ? w[i + 2] : w[i];
#pragma unroll
    for (int i = 0; i < NO; ++i) o[i] = (s & 1) ? t[i + 1] : t[i];
}

// 16-byte chunk = window elements [rho, rho + EPC) of a window of 32-bit words
// holding E = 4 / sizeof(elem) elements each (E = 2: u16 pairs, E = 1: 32-bit).
template <int E, int NW>
__device__ __forceinline__ void window_chunk(const uint32_t (&w)[NW], int rho, int q, uint32_t (&o)[4]) {
    // q = chunk index inside the window (the window starts at a chunk boundary)
    if constexpr (E == 2) {
        uint32_t t[5];
        uint32_t ww[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) ww[i] = (4 * q + i < NW) ? w[4 * q + i] : 0u;
        shift_words<5, 8>(ww, rho >> 1, t);
        const uint32_t sel = (rho & 1) ? 0x5432u : 0x3210u;
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = __byte_perm(t[i], t[i + 1], sel);
    } else {
        uint32_t ww[7];
#pragma unroll
        for (int i = 0; i < 7; ++i) ww[i] = (4 * q + i < NW) ? w[4 * q + i] : 0u;
        shift_words<4, 7>(ww, rho, o);
    }
}

__device__ __forceinline__ uint32_t sel4(const uint32_t (&v)[4], int i) {
    const uint32_t lo = (i & 1) ? v[1] : v[0], hi = (i & 1) ? v[3] : v[2];
    return (i & 2) ? hi : lo;
}

// Store elements [0, m) (head) or [EPC - t, EPC) (tail) of a 16-byte chunk
// with naturally aligned 8/4/2-byte stores.  E = elements per 32-bit word.
// (Runtime word choices go through selects, not register-array indexing.)
template <int E>
__device__ __forceinline__ void store_chunk_head(void *chunk, const uint32_t (&v)[4], int m) {
    unsigned char *p = reinterpret_cast<unsigned char *>(chunk);
    if (m >= 4 * E) { *reinterpret_cast<uint4 *>(p) = make_uint4(v[0], v[1], v[2], v[3]); return; }
    const int mb = m * (4 / E);                         // bytes to write, < 16
    if (mb & 8) *reinterpret_cast<uint2 *>(p) = make_uint2(v[0], v[1]);
    const int w4 = (mb & 8) ? 2 : 0;
    if (mb & 4) *reinterpret_cast<uint32_t *>(p + 4 * w4) = sel4(v, w4);
    if (E == 2 && (mb & 2)) {
        const int w2 = w4 + ((mb & 4) ? 1 : 0);
        *reinterpret_cast<uint16_t *>(p + 4 * w2) = (uint16_t)(sel4(v, w2) & 0xFFFFu);
    }
}
template <int E>
__device__ __forceinline__ void store_chunk_tail(void *chunk, const uint32_t (&v)[4], int t) {
    unsigned char *p = reinterpret_cast<unsigned char *>(chunk);
    if (t >= 4 * E) { *reinterpret_cast<uint4 *>(p) = make_uint4(v[0], v[1], v[2], v[3]); return; }
    const int tb = t * (4 / E);                         // bytes to write at the end, < 16
    int b = 16 - tb;                                    // first byte written
    if (E == 2 && (tb & 2)) {                           // odd u16 count: one u16 at an odd index
        *reinterpret_cast<uint16_t *>(p + b) = (uint16_t)(sel4(v, b >> 2) >> 16);
        b += 2;
    }
    if (tb & 4) { *reinterpret_cast<uint32_t *>(p + b) = sel4(v, b >> 2); b += 4; }
    if (tb & 8) *reinterpret_cast<uint2 *>(p + 8) = make_uint2(v[2], v[3]);
}

// ---------------------------------------------------------------------------
// L2 residency.  The 2.4 GB output streams through the
// 126 MB L2; the cube and the stage buffers (re-read by the next pass / the
// next dodecant) are marked evict_last so the stream does not push them out.
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_hint_v4(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_hint_v4(const void *p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

// Task -> (row, run) with quarter-warps on 8 consecutive runs of one row (conflict-free
// 16-byte shared loads): tasks below 8 * nrows cover runs 0..7, the rest runs 8..nr-1.  With
// row_fast the extra runs go row-fastest, so a quarter-warp of them reads 8 different rows at one
// run (their slots start in different bank groups) instead of 4 rows x 2 runs (which collide in
// the SWAR kernel's slot layout; measured neutral-to-worse for the 32-bit passes, so off there).
__device__ __forceinline__ void task_row_run(int t, int nr, int nrows, int &row, int &run, bool row_fast = false) {
    if (nr <= 8 || t < 8 * nrows) { row = t >> 3; run = t & 7; if (nr < 8) { row = t / nr; run = t - row * nr; } return; }
    const int u = t - 8 * nrows, extra = nr - 8;
    if (row_fast) {
        row = u % nrows;
        run = 8 + u / nrows;
    } else {
        row = u / extra;
        run = 8 + (u - row * extra);
    }
}


// streaming (evict-first) 16-byte global store for final outputs that are
// never re-read by this call.
__device__ __forceinline__ void st_cs_v4(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// 32-byte global stores (STG.256, sm_100): a lane fills one whole 32-byte sector, so a warp's
// scattered row stores need half the instructions (and L1 data-pipe wavefronts) of 16-byte ones.
// p must be 32-byte aligned.
__device__ __forceinline__ void st_cs_v8(void *p, const uint32_t (&v)[8]) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void st_v8(void *p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
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

// D tile width of the u16-input K = 4 final pass (the cfg3 kernel, launch.cuh); also the tile grid
// of the zero tiles the first pass writes for it (api.cu)
#ifndef D3_FINAL16_T
#define D3_FINAL16_T 48                 // 3 CTAs/SM (70 KB, 128 threads at 168 registers); 64: 2 CTAs/SM, 3.5% slower
#endif

enum Stor { ST_U8 = 0, ST_U16 = 1, ST_U32 = 2, ST_F32 = 3 };

}  // namespace d3
