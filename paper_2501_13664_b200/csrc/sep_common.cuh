// sep_common.cuh -- register-blocked direct sums shared by the separable on-chip small-cube DRT
// kernels (k_sep32.cu, k_sep16.cu).  Rows are read as 16-byte chunks through a chunk-address
// functor (the caller's layout, zero chunks outside a row); the offsets l^K_r(w) of eq:digitalLine
// are compile-time register indices.
#pragma once
#include "common.cuh"

namespace d3 {
namespace sep {

template <int I, class F>
__device__ __forceinline__ void with_const8(int v, F &&f) {
    if constexpr (I < 8) {
        if (v == I) f(std::integral_constant<int, I>{});
        else with_const8<I + 1>(v, f);
    }
}

// buf[0 .. NE) = elements 4 c0 .. 4 c0 + NE of a row whose chunk c lives at chunk(c) (the zero
// chunk outside the row)
template <int NE, class CF>
__device__ __forceinline__ void load_row(CF &&chunk, int c0, uint32_t (&buf)[NE]) {
#pragma unroll
    for (int i = 0; i < (NE + 3) / 4; ++i) {
        const uint4 v = *reinterpret_cast<const uint4 *>(chunk(c0 + i));
        buf[4 * i] = v.x;
        if (4 * i + 1 < NE) buf[4 * i + 1] = v.y;
        if (4 * i + 2 < NE) buf[4 * i + 2] = v.z;
        if (4 * i + 3 < NE) buf[4 * i + 3] = v.w;
    }
}

// Radix-8 direct sum over the 8 rows a of a run of RR outputs starting at chunk cb (elements 4 cb + j + l^3_r(a)),
// for the NR output slopes r = R0 .. R0 + NR - 1: acc[r - R0][j] (assigned, not accumulated).
template <int NR, int R0, int RR, class Acc, class RowChunk>
__device__ __forceinline__ void radix8(RowChunk &&rc, int cb, uint32_t one, Acc (&acc)[NR][RR]) {
    static_for<0, 4>([&](auto p_) {
        constexpr int a0 = 2 * decltype(p_)::value, a1 = a0 + 1;
        uint32_t b0[RR + a0], b1[RR + a1];
        load_row<RR + a0>([&](int c) { return rc(a0, c); }, cb, b0);
        load_row<RR + a1>([&](int c) { return rc(a1, c); }, cb, b1);
        static_for<0, NR>([&](auto r_) {
            constexpr int r = decltype(r_)::value;
            constexpr int o0 = lk(3, R0 + r, a0), o1 = lk(3, R0 + r, a1);
#pragma unroll
            for (int j = 0; j < RR; ++j) {
                if constexpr (a0 == 0) acc[r][j] = Lane<Acc>::get(b0[j + o0]) + Lane<Acc>::get(b1[j + o1]);
                else acc[r][j] = add2<Acc>(acc[r][j], b0[j + o0], b1[j + o1], one, false);
            }
        });
    });
}

// Radix-4 sum with a per-row shift SIG * V (compile time) over runs of RR outputs:
// acc[rho][j] = sum_V row_V[u0 + SIG V + j + l^2_rho(V)] for the 4 rows V, u0 = 4 cb (chunk aligned).
template <int SIG, int RR, class Acc, class RowChunk>
__device__ __forceinline__ void radix4(RowChunk &&rc, int cb, uint32_t one, Acc (&acc)[4][RR]) {
    static_for<0, 2>([&](auto p_) {
        constexpr int v0 = 2 * decltype(p_)::value, v1 = v0 + 1;
        constexpr int c0 = (SIG * v0) >> 2, o0 = (SIG * v0) & 3, c1 = (SIG * v1) >> 2, o1 = (SIG * v1) & 3;
        uint32_t b0[o0 + RR + v0], b1[o1 + RR + v1];
        load_row<o0 + RR + v0>([&](int c) { return rc(v0, c); }, cb + c0, b0);
        load_row<o1 + RR + v1>([&](int c) { return rc(v1, c); }, cb + c1, b1);
        static_for<0, 4>([&](auto r_) {
            constexpr int r = decltype(r_)::value;
            constexpr int e0 = o0 + lk(2, r, v0), e1 = o1 + lk(2, r, v1);
#pragma unroll
            for (int j = 0; j < RR; ++j) {
                if constexpr (v0 == 0) acc[r][j] = Lane<Acc>::get(b0[j + e0]) + Lane<Acc>::get(b1[j + e1]);
                else acc[r][j] = add2<Acc>(acc[r][j], b0[j + e0], b1[j + e1], one, false);
            }
        });
    });
}

template <class In>
__device__ __forceinline__ void load4(const In *p, uint32_t (&v)[4]) {
    if constexpr (sizeof(In) == 1) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(p));
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = (w >> (8 * k)) & 0xFFu;
    } else {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(p));
        v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
    }
}

}  // namespace sep
}  // namespace d3
