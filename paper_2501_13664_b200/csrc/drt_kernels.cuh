// drt_kernels.cuh -- 3D DRT of planes: one "radix-2^K pass" kernel.
//
// The Alg. 1 recursion (eq:map3D PAPER.md:213-227) is
// regrouped into passes of K consecutive stages.  Pass p starts from the
// stage-c partial transform (eq:3Dfm; c = bits done) and
// produces stage c+K.  By eq:digitalLine the stage-(c+K) value is a direct sum
// over a 2^K x 2^K group of stage-c rows:
//
//   f^{c+K}(s1', s2' | V1, V2 | D) = sum_{w1,w2 < 2^K} f^c(s1, s2 | V1 2^K + w1, V2 2^K + w2 |
//                 D + s1 w1 + s2 w2 + l^K_{r1}(w1) + l^K_{r2}(w2)),
//   s' = s 2^K + r  (s: c slope bits already built, r: the K new low bits).
//
// The runtime part (s1 w1 + s2 w2) is applied when a row is staged into
// shared memory; the compile-time part l^K_r(w) becomes register indexing in
// two separable direct sums (x then y).  Each CTA owns one group and one D
// tile of width T; all 4^K rows stay in shared memory.
//
// Storage of a stage-c buffer (per instance = one (cube, dodecant) pair):
//   rows  ((s1 2^c + s2) 2^(n-c) + v1) 2^(n-c) + v2,     (N^2 rows)
//   D' = D - base_c, base_c = 2N - 2(2^c - 1), valid width W_c = N + 2(2^c - 1)
// (the support of eq:3Dfm at stage c).  Stage 0 is the oriented cube
// itself (base 2N, width N); the final stage is the stacked output
// out[s1][s2][D], D in [0, 3N), zero outside the support.
#pragma once
#include "common.cuh"

namespace d3 {

struct DrtPass {
    const void *in;
    void *out;
    int N, n, c, m;                 // c = bits before the pass, m = n - c - K
    long long in_inst_stride;       // elements between instances (stage buffers)
    int in_pitch, in_base, in_width;
    long long out_inst_stride;
    int out_pitch, out_base, out_width;
    int inst0;                      // global instance of blockIdx.z == 0
    int ndod;                       // dodecants per cube (instances per batch entry)
    int layout;                     // final pass: 0 stacked, 1 mosaic
    Orient ori[kMaxDod];            // first pass: per-dodecant-slot orientation
    int8_t out_order[kMaxDod][2];   // mosaic: OutOrder[k][0..1]
    int8_t coords[kMaxDod][2];      // mosaic: DodecantCoords[k]
};

template <int K, int R, int T>
struct DrtGeom {
    static constexpr int S = 1 << K;
    static constexpr int H = S - 1;                      // max l^K_r(w) = w <= S-1
    static constexpr int WIN = T + 2 * H;                // staged row width
    static constexpr int NRX = (T + H + R - 1) / R;      // x-step runs per row
    static constexpr int NRY = T / R;                    // y-step runs per row
    static constexpr int NEED = NRX * R + S + 3;         // furthest word touched
    static constexpr int PI = ((NEED > WIN ? NEED : WIN) + 31) / 32 * 32;  // row pitch (words)
    static constexpr int XT = S * NRX;                   // x-step tasks
    static constexpr int YT = S * NRY;                   // y-step tasks
    static constexpr int THREADS = ((XT > YT ? XT : YT) + 31) / 32 * 32;
    static constexpr int SMEM = S * S * PI * 4;
    static_assert(T % R == 0 && R % 4 == 0, "tile shape");
};

// XOR swizzle of 16-byte chunks inside each 128-byte group of a staged row:
// makes the 8 lanes of an LDS.128 phase hit 8 distinct bank groups whether the
// lanes vary the first or the second row coordinate.
template <int K>
__device__ __forceinline__ int swz(int slot) { return ((slot >> K) ^ slot) & 7; }

// acc[r][j] += sum over the S rows a of row_a[j + l^K_r(a)], rows staged at
// slot(a) = slot_base + a * slot_step, the thread's run starting at chunk c0.
template <int K, int R, int PI, class Acc>
__device__ __forceinline__ void drt_direct_sum(const uint32_t *__restrict__ sm, int slot_base, int slot_step,
                                               int c0, Acc (&acc)[1 << K][R]) {
    constexpr int S = 1 << K;
    constexpr int NB = (R + S + 2) / 4;
    static_for<0, S>([&](auto a_) {
        constexpr int a = decltype(a_)::value;
        constexpr int NC = (R + a + 3) / 4;              // chunks holding [run, run + R + a)
        const int slot = slot_base + a * slot_step;
        const int sw = swz<K>(slot);
        const uint32_t *row = sm + slot * PI;
        uint32_t buf[NB * 4];
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            const uint4 v = *reinterpret_cast<const uint4 *>(row + (((c0 + i) ^ sw) << 2));
            buf[4 * i + 0] = v.x;
            buf[4 * i + 1] = v.y;
            buf[4 * i + 2] = v.z;
            buf[4 * i + 3] = v.w;
        }
        static_for<0, S>([&](auto r_) {
            constexpr int r = decltype(r_)::value;
            constexpr int off = lk(K, r, a);
#pragma unroll
            for (int j = 0; j < R; ++j) acc[r][j] = acc[r][j] + Lane<Acc>::get(buf[j + off]);
        });
    });
}

template <int K, int R, int T, class In, class Acc, class Out, bool FIRST, bool FINAL>
__global__ void __launch_bounds__(DrtGeom<K, R, T>::THREADS)
drt_pass_kernel(const DrtPass p) {
    using G = DrtGeom<K, R, T>;
    constexpr int S = G::S, PI = G::PI, WIN = G::WIN;
    extern __shared__ uint4 smem_u4[];
    uint32_t *sm = reinterpret_cast<uint32_t *>(smem_u4);

    const int tid = threadIdx.x;
    const int tile = blockIdx.x, g = blockIdx.y, li = blockIdx.z;
    const int inst = p.inst0 + li;
    const int m = p.m, c = p.c;
    const int V2 = g & ((1 << m) - 1);
    const int V1 = (g >> m) & ((1 << m) - 1);
    const int sig = g >> (2 * m);
    const int sg2 = sig & ((1 << c) - 1);
    const int sg1 = sig >> c;
    const int d0 = tile * T;                 // stored output coordinate of the tile
    const int Dabs = p.out_base + d0;        // absolute displacement D of the tile start
    const int N = p.N;
    const int cK = c + K;

    // ---- output addressing
    auto out_row_index = [&](int r1, int r2) -> long long {
        const int s1 = (sg1 << K) + r1, s2 = (sg2 << K) + r2;
        return ((((long long)s1 << cK) + s2) << (2 * m)) + ((long long)V1 << m) + V2;
    };
    Out *outp = reinterpret_cast<Out *>(p.out);
    const long long out_inst = FINAL ? (long long)inst * p.out_inst_stride : (long long)li * p.out_inst_stride;

    // mosaic placement of a final row (Alg. 2 OutOrder / DodecantCoords)
    auto mosaic_row = [&](int r1, int r2) -> long long {
        const int b = inst / p.ndod, j = inst - b * p.ndod;
        const int s[2] = {(sg1 << K) + r1, (sg2 << K) + r2};
        const int o0 = p.out_order[j][0], o1 = p.out_order[j][1];
        int w0 = s[(o0 < 0 ? -o0 : o0) - 1], w1 = s[(o1 < 0 ? -o1 : o1) - 1];
        if (o0 < 0) w0 = N - 1 - w0;
        if (o1 < 0) w1 = N - 1 - w1;
        const long long rr = (long long)(p.coords[j][0] * N + w0) * (4 * N) + (p.coords[j][1] * N + w1);
        return (long long)b * 16 * N * N * (3 * N - 2) + rr * (3 * N - 2);
    };
    auto store_scalar = [&](int r1, int r2, int e, Acc v) {
        const int D = d0 + e;
        if (D >= p.out_width) return;
        if (FINAL && p.layout == 1) {
            if (D >= 2) outp[mosaic_row(r1, r2) + D - 2] = to_out<Out, Acc>(v);
        } else {
            outp[out_inst + out_row_index(r1, r2) * p.out_pitch + D] = to_out<Out, Acc>(v);
        }
    };

    // ---- tiles entirely outside the support of all 4^K output rows: zeros
    // (support D >= 2N - s1 - s2)
    {
        const int s1max = (sg1 << K) + S - 1, s2max = (sg2 << K) + S - 1;
        if (Dabs + T <= 2 * N - s1max - s2max) {
            for (int i = tid; i < S * S * T; i += blockDim.x) {
                const int rr = i / T, e = i - rr * T;
                store_scalar(rr / S, rr % S, e, Acc(0));
            }
            return;
        }
    }

    // ---- stage the 4^K input rows of the group into shared memory
    if constexpr (FIRST) {
        const Orient o = p.ori[inst % p.ndod];
        const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
        const int z0 = Dabs - 2 * N;       // z' of element 0 (stage-0 rows: D = z' + 2N)
        const int xb = V1 << K, yb = V2 << K;
        for (int i = tid; i < S * S * WIN; i += blockDim.x) {
            int w1, w2, e;
            if (o.fast == 2) { e = i % WIN; const int rw = i / WIN; w2 = rw % S; w1 = rw / S; }
            else if (o.fast == 0) { w1 = i % S; const int rw = i / S; e = rw % WIN; w2 = rw / WIN; }
            else { w2 = i % S; const int rw = i / S; e = rw % WIN; w1 = rw / WIN; }
            const int z = z0 + e;
            uint32_t bits = 0;
            if ((unsigned)z < (unsigned)N)
                bits = Elem<In>::load_bits(cube + o.off0 + (xb + w1) * o.sx + (yb + w2) * o.sy + z * o.sz);
            const int slot = w1 * S + w2;
            sm[slot * PI + (((e >> 2) ^ swz<K>(slot)) << 2) + (e & 3)] = bits;
        }
    } else {
        const In *inb = reinterpret_cast<const In *>(p.in) + (long long)li * p.in_inst_stride;
        const int nc = p.n - c;
        const long long rbase = (((long long)sg1 << c) + sg2) << (2 * nc);
        for (int i = tid; i < S * S * WIN; i += blockDim.x) {
            const int e = i % WIN, slot = i / WIN;
            const int w1 = slot / S, w2 = slot % S;
            const long long row = rbase + ((long long)((V1 << K) + w1) << nc) + (V2 << K) + w2;
            const int idx = Dabs + sg1 * w1 + sg2 * w2 - p.in_base + e;
            uint32_t bits = 0;
            if ((unsigned)idx < (unsigned)p.in_width) bits = Elem<In>::load_bits(inb + row * p.in_pitch + idx);
            sm[slot * PI + (((e >> 2) ^ swz<K>(slot)) << 2) + (e & 3)] = bits;
        }
    }
    __syncthreads();

    // ---- x-step: X(r1, w2, j) = sum_w1 staged(w1, w2, j + l^K_{r1}(w1)), kept in registers,
    // then written in place over the staged rows (slot (r1, w2)).
    Acc acc[S][R];
    const bool xact = tid < G::XT;
    const int xb2 = tid & (S - 1), xr = tid >> K;
    if (xact) {
#pragma unroll
        for (int r = 0; r < S; ++r)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[r][j] = Acc(0);
        drt_direct_sum<K, R, PI, Acc>(sm, xb2, S, xr * (R / 4), acc);
    }
    __syncthreads();
    if (xact) {
#pragma unroll
        for (int r = 0; r < S; ++r) {
            const int slot = r * S + xb2;
            const int sw = swz<K>(slot);
#pragma unroll
            for (int q = 0; q < R / 4; ++q) {
                uint4 v;
                v.x = Lane<Acc>::bits(acc[r][4 * q + 0]);
                v.y = Lane<Acc>::bits(acc[r][4 * q + 1]);
                v.z = Lane<Acc>::bits(acc[r][4 * q + 2]);
                v.w = Lane<Acc>::bits(acc[r][4 * q + 3]);
                *reinterpret_cast<uint4 *>(sm + slot * PI + (((xr * (R / 4) + q) ^ sw) << 2)) = v;
            }
        }
    }
    __syncthreads();

    // ---- y-step: out(r1, r2, j) = sum_w2 X(r1, w2, j + l^K_{r2}(w2)); store
    if (tid < G::YT) {
        const int r1 = tid & (S - 1), yr = tid >> K;
#pragma unroll
        for (int r = 0; r < S; ++r)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[r][j] = Acc(0);
        drt_direct_sum<K, R, PI, Acc>(sm, r1 * S, 1, yr * (R / 4), acc);

        const int e0 = yr * R;
        const bool vec_ok = (!FINAL || p.layout == 0) && (d0 + e0 + R <= p.out_width) &&
                            ((p.out_pitch * (int)sizeof(Out)) % 16 == 0) && (((d0 + e0) * (int)sizeof(Out)) % 16 == 0);
#pragma unroll
        for (int r2 = 0; r2 < S; ++r2) {
            if (vec_ok) {
                Out *dst = outp + out_inst + out_row_index(r1, r2) * p.out_pitch + d0 + e0;
                if constexpr (sizeof(Out) == 2) {
#pragma unroll
                    for (int q = 0; q < R / 8; ++q) {
                        uint32_t w[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h)
                            w[h] = (uint32_t)to_out<Out, Acc>(acc[r2][8 * q + 2 * h]) |
                                   ((uint32_t)to_out<Out, Acc>(acc[r2][8 * q + 2 * h + 1]) << 16);
                        *reinterpret_cast<uint4 *>(dst + 8 * q) = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < R / 4; ++q) {
                        const uint32_t a0 = Lane<Acc>::bits(acc[r2][4 * q + 0]), a1 = Lane<Acc>::bits(acc[r2][4 * q + 1]);
                        const uint32_t a2 = Lane<Acc>::bits(acc[r2][4 * q + 2]), a3 = Lane<Acc>::bits(acc[r2][4 * q + 3]);
                        if (FINAL) st_cs_v4(dst + 4 * q, a0, a1, a2, a3);
                        else *reinterpret_cast<uint4 *>(dst + 4 * q) = make_uint4(a0, a1, a2, a3);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < R; ++j) store_scalar(r1, r2, e0 + j, acc[r2][j]);
            }
        }
    }
}

}  // namespace d3
