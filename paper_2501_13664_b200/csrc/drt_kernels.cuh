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
#include "tma.cuh"

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
    int vec_ok;                     // first pass: 16-byte chunked cube loads are aligned (N >= 16)
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
    static constexpr int NEED = (NRX - 1) * R + (R + H + 3) / 4 * 4;   // words touched by the last run
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
    const int mos_b = inst / p.ndod, mos_j = inst - mos_b * p.ndod;
    auto mosaic_row = [&](int r1, int r2) -> long long {
        const int b = mos_b, j = mos_j;
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
            constexpr int EPV = 16 / (int)sizeof(Out);
            const bool vz = (!FINAL || p.layout == 0) && ((p.out_pitch * (int)sizeof(Out)) % 16 == 0) &&
                            ((d0 * (int)sizeof(Out)) % 16 == 0) && (d0 + T <= p.out_width);
            if (vz) {
                for (int i = tid; i < S * S * (T / EPV); i += blockDim.x) {
                    const int rr = i / (T / EPV), q = i - rr * (T / EPV);
                    Out *dst = outp + out_inst + out_row_index(rr / S, rr % S) * p.out_pitch + d0 + q * EPV;
                    *reinterpret_cast<uint4 *>(dst) = make_uint4(0u, 0u, 0u, 0u);
                }
            } else {
                for (int i = tid; i < S * S * T; i += blockDim.x) {
                    const int rr = i / T, e = i - rr * T;
                    store_scalar(rr / S, rr % S, e, Acc(0));
                }
            }
            return;
        }
    }

    // ---- stage the 4^K input rows of the group into shared memory
    auto put = [&](int slot, int e, uint32_t bits) {
        sm[slot * PI + (((e >> 2) ^ swz<K>(slot)) << 2) + (e & 3)] = bits;
    };
    if constexpr (FIRST) {
        const Orient o = p.ori[inst % p.ndod];
        const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
        const int z0 = Dabs - 2 * N;       // z' of element 0 (stage-0 rows: D = z' + 2N)
        const int xb = V1 << K, yb = V2 << K;
        if (!p.vec_ok) {
            for (int i = tid; i < S * S * WIN; i += blockDim.x) {
                const int e = i % WIN, slot = i / WIN;
                const int w1 = slot / S, w2 = slot % S, z = z0 + e;
                uint32_t bits = 0;
                if ((unsigned)z < (unsigned)N)
                    bits = Elem<In>::load_bits(cube + o.off0 + (xb + w1) * o.sx + (yb + w2) * o.sy + z * o.sz);
                put(slot, e, bits);
            }
        } else if (sizeof(In) == 1 && o.fast == 2 && o.sz > 0 && (z0 & 15) == 0 && 16 * ((WIN + 15) / 16) <= PI) {
            // u8 rows along z' (forward, 16-aligned): one LDG.128 = 16 voxels = 4 SMEM chunks
            constexpr int NQ16 = (WIN + 15) / 16;
            constexpr int ITEMS = 4;
            for (int base = tid; base < S * S * NQ16; base += blockDim.x * ITEMS) {
                uint4 v[ITEMS];
                int sl[ITEMS], qq[ITEMS];
#pragma unroll
                for (int u = 0; u < ITEMS; ++u) {
                    const int it = base + u * blockDim.x;
                    v[u] = make_uint4(0u, 0u, 0u, 0u);
                    sl[u] = -1;
                    if (it < S * S * NQ16) {
                        const int slot = it / NQ16, q = it - slot * NQ16;
                        const int w1 = slot / S, w2 = slot - w1 * S, z = z0 + 16 * q;
                        sl[u] = slot;
                        qq[u] = q;
                        if ((unsigned)z < (unsigned)N)
                            v[u] = __ldg(reinterpret_cast<const uint4 *>(
                                cube + o.off0 + (long long)(xb + w1) * o.sx + (long long)(yb + w2) * o.sy + z));
                    }
                }
#pragma unroll
                for (int u = 0; u < ITEMS; ++u) {
                    if (sl[u] < 0) continue;
                    const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                    const int sw = swz<K>(sl[u]);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const uint4 o4 = make_uint4(__byte_perm(w[h], 0, 0x4440), __byte_perm(w[h], 0, 0x4441),
                                                    __byte_perm(w[h], 0, 0x4442), __byte_perm(w[h], 0, 0x4443));
                        *reinterpret_cast<uint4 *>(sm + sl[u] * PI + (((4 * qq[u] + h) ^ sw) << 2)) = o4;
                    }
                }
            }
        } else if (sizeof(In) == 1 && K == 4 && o.fast != 2) {
            // u8, unit stride along x' (fast 0) or y' (fast 1): one LDG.128 = the 16 voxels of a
            // run along that axis; 4 consecutive z' per item are transposed in registers so every
            // SMEM write is a 16-byte chunk (4 consecutive e of one slot)
            const bool fx = o.fast == 0;
            const long long sf = fx ? o.sx : o.sy, so = fx ? o.sy : o.sx;
            const int fb = fx ? xb : yb, ob = fx ? yb : xb;
            constexpr int NG = (WIN + 3) / 4;
            for (int it = tid; it < S * NG; it += blockDim.x) {
                const int other = it % S, g = it / S;
                uint4 v[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int z = z0 + 4 * g + t;
                    v[t] = make_uint4(0u, 0u, 0u, 0u);
                    if ((unsigned)z < (unsigned)N) {
                        const long long b = o.off0 + (long long)(ob + other) * so + (long long)z * o.sz +
                                            (sf > 0 ? (long long)fb : -(long long)(fb + 15));
                        v[t] = __ldg(reinterpret_cast<const uint4 *>(cube + b));
                    }
                }
#pragma unroll
                for (int wf = 0; wf < 16; ++wf) {
                    const int byte = sf > 0 ? wf : 15 - wf;     // runtime-uniform direction
                    uint32_t q4[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint32_t w[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
                        q4[t] = __byte_perm(w[byte >> 2], 0, 0x4440 | (byte & 3));
                    }
                    const int slot = fx ? wf * S + other : other * S + wf;
                    *reinterpret_cast<uint4 *>(sm + slot * PI + ((g ^ swz<K>(slot)) << 2)) =
                        make_uint4(q4[0], q4[1], q4[2], q4[3]);
                }
            }
        } else if (o.fast == 2) {
            // rows along z' are contiguous in the original cube (reversed when sz < 0)
            stage_rows<In, 8>(S * S, WIN, [&](int slot) {
                const int w1 = slot / S, w2 = slot % S;
                const long long b = o.off0 + (long long)(xb + w1) * o.sx + (long long)(yb + w2) * o.sy;
                RowSrc<In> r;
                if (o.sz > 0) { r.ptr = cube + b; r.st = z0; r.dir = 1; }
                else { r.ptr = cube + b - (N - 1); r.st = N - 1 - z0; r.dir = -1; }
                r.width = N;
                return r;
            }, put);
        } else {
            // the unit-stride axis is x' (fast 0) or y' (fast 1): stage runs of S voxels along it
            const bool fx = o.fast == 0;
            stage_rows<In, 8>(S * WIN, S, [&](int r) {
                const int other = r % S, e = r / S, z = z0 + e;
                const long long sf = fx ? o.sx : o.sy, so = fx ? o.sy : o.sx;
                const int fb = fx ? xb : yb, ob = fx ? yb : xb;
                const long long b = o.off0 + (long long)(ob + other) * so + (long long)z * o.sz;
                RowSrc<In> rr;
                if (sf > 0) { rr.ptr = cube + b; rr.st = fb; rr.dir = 1; }
                else { rr.ptr = cube + b - (N - 1); rr.st = N - 1 - fb; rr.dir = -1; }
                rr.width = ((unsigned)z < (unsigned)N) ? N : 0;
                return rr;
            }, [&](int r, int wf, uint32_t bits) {
                const int other = r % S, e = r / S;
                put(fx ? wf * S + other : other * S + wf, e, bits);
            });
        }
    } else {
        const In *inb = reinterpret_cast<const In *>(p.in) + (long long)li * p.in_inst_stride;
        const int nc = p.n - c;
        const long long rbase = (((long long)sg1 << c) + sg2) << (2 * nc);
        stage_rows<In, 8>(S * S, WIN, [&](int slot) {
            const int w1 = slot / S, w2 = slot % S;
            const long long row = rbase + ((long long)((V1 << K) + w1) << nc) + (V2 << K) + w2;
            RowSrc<In> r;
            r.ptr = inb + row * p.in_pitch;
            r.st = Dabs + sg1 * w1 + sg2 * w2 - p.in_base;
            r.dir = 1;
            r.width = p.in_width;
            return r;
        }, put);
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


// ===========================================================================
// Non-first passes.  The 4^K stage-c rows are staged in their storage type
// (u16 or 32-bit): each 16-byte SMEM chunk is built from two aligned 16-byte
// global loads and an in-register realignment by the row's runtime
// displacement (sigma1 w1 + sigma2 w2 is arbitrary, so neither TMA nor plain
// vector loads can place it directly).  X is written in place as 32-bit lanes
// with an XOR swizzle; sums use 3-input adds.
// ===========================================================================
template <int K, int R, int T, class MidIn>
struct DrtMidGeom {
    static constexpr int S = 1 << K;
    static constexpr int H = S - 1;
    static constexpr int WIN = T + 2 * H;
    static constexpr int EPC = 16 / (int)sizeof(MidIn);            // elements per 16-byte chunk
    static constexpr int NRX = (T + H + R - 1) / R;
    static constexpr int NRY = T / R;
    static constexpr int RD = (NRX - 1) * R + (R + H + EPC - 1) / EPC * EPC;   // input elements touched
    static constexpr int BOXW = ((WIN > RD ? WIN : RD) + EPC - 1) / EPC * EPC;  // staged elements per row
    static constexpr int NQ = BOXW / EPC;                           // staged chunks per row
    static constexpr int XW = ((NRX * R + 31) / 32) * 32;           // X words per slot (8-chunk groups)
    static constexpr int SLOT_IN = BOXW * (int)sizeof(MidIn);
    static constexpr int SP0 = (((SLOT_IN > XW * 4) ? SLOT_IN : XW * 4) + 15) / 16 * 16;
    static constexpr int SP = (SP0 % 128 == 0) ? SP0 + 16 : SP0;    // slot pitch (bytes), rotates banks across slots
    static constexpr int XT = S * NRX;
    static constexpr int YT = S * NRY;
    static constexpr int THREADS = ((XT > YT ? XT : YT) + 31) / 32 * 32;
    static constexpr int SMEM = S * S * SP;
    // two CTAs per SM: with W warps per CTA an SM sub-partition holds ceil(2W/4) warps of its
    // 16K-register file, which caps the registers per thread
    static constexpr int WARPS = THREADS / 32;
    static constexpr int MAXREG0 = 16384 / (((2 * WARPS + 3) / 4) * 32) / 8 * 8;
    static constexpr int MAXREG = MAXREG0 > 255 ? 255 : MAXREG0;
    static_assert(T % R == 0 && R % 4 == 0 && (R % EPC == 0 || EPC > R), "tile shape");
    static_assert((NRY - 1) * R + (R + H + 3) / 4 * 4 <= NRX * R, "y-step reads inside X");
};

// 16 bytes starting `b` bytes (0..15) into the 32-byte window lo:hi.
__device__ __forceinline__ uint4 realign16(const uint4 &lo, const uint4 &hi, int b) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const int ws = b >> 2, bs = (b & 3) * 8;
    uint32_t t[6], u[5];
#pragma unroll
    for (int i = 0; i < 6; ++i) t[i] = (ws & 2) ? w[i + 2] : w[i];
#pragma unroll
    for (int i = 0; i < 5; ++i) u[i] = (ws & 1) ? t[i + 1] : t[i];
    uint4 o;
    o.x = __funnelshift_r(u[0], u[1], bs);
    o.y = __funnelshift_r(u[1], u[2], bs);
    o.z = __funnelshift_r(u[2], u[3], bs);
    o.w = __funnelshift_r(u[3], u[4], bs);
    return o;
}

__device__ __forceinline__ int xswz(int c) { return c ^ ((c >> 3) & 1); }

// Load elements [0, NE) of a row starting at `row` (run-aligned), unpacked to 32-bit lanes.
template <class MidIn, int NE>
__device__ __forceinline__ void load_run(const unsigned char *row, uint32_t *buf) {
    if constexpr (sizeof(MidIn) == 2) {
#pragma unroll
        for (int i = 0; i < (NE + 7) / 8; ++i) {
            const uint4 v = *reinterpret_cast<const uint4 *>(row + 16 * i);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (8 * i + q < NE) buf[8 * i + q] = (q & 1) ? (w[q >> 1] >> 16) : (w[q >> 1] & 0xFFFFu);
        }
    } else {
#pragma unroll
        for (int i = 0; i < (NE + 3) / 4; ++i) {
            const uint4 v = *reinterpret_cast<const uint4 *>(row + 16 * i);
            buf[4 * i + 0] = v.x;
            if (4 * i + 1 < NE) buf[4 * i + 1] = v.y;
            if (4 * i + 2 < NE) buf[4 * i + 2] = v.z;
            if (4 * i + 3 < NE) buf[4 * i + 3] = v.w;
        }
    }
}

// acc[r][j] += sum_a row_a[j + l^K_r(a)]; rows taken two at a time so that the
// integer sums become 3-input adds.  LoadRow(integral_constant a, buf) fills
// buf[0, R + a) with the row's run.
template <int K, int R, class Acc, class LoadRow>
__device__ __forceinline__ void direct_sum2(LoadRow &&load_row, Acc (&acc)[1 << K][R]) {
    constexpr int S = 1 << K;
    if constexpr (S == 1) {
        uint32_t b0[R];
        load_row(std::integral_constant<int, 0>{}, b0);
#pragma unroll
        for (int j = 0; j < R; ++j) acc[0][j] = acc[0][j] + Lane<Acc>::get(b0[j]);
    } else {
        static_for<0, S / 2>([&](auto p_) {
            constexpr int a0 = 2 * decltype(p_)::value, a1 = a0 + 1;
            uint32_t b0[R + a0], b1[R + a1];
            load_row(std::integral_constant<int, a0>{}, b0);
            load_row(std::integral_constant<int, a1>{}, b1);
            static_for<0, S>([&](auto r_) {
                constexpr int r = decltype(r_)::value;
                constexpr int o0 = lk(K, r, a0), o1 = lk(K, r, a1);
#pragma unroll
                for (int j = 0; j < R; ++j)
                    acc[r][j] = acc[r][j] + Lane<Acc>::get(b0[j + o0]) + Lane<Acc>::get(b1[j + o1]);
            });
        });
    }
}

template <int K, int R, int T, class MidIn, class Acc, class Out, bool FINAL>
__global__ void __maxnreg__((DrtMidGeom<K, R, T, MidIn>::MAXREG))
drt_pass_mid_kernel(const DrtPass p) {
    using G = DrtMidGeom<K, R, T, MidIn>;
    constexpr int S = G::S, SP = G::SP, EPC = G::EPC, NQ = G::NQ;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;

    const int tid = threadIdx.x;
    const int tile = blockIdx.x, g = blockIdx.y, li = blockIdx.z;
    const int inst = p.inst0 + li;
    const int m = p.m, c = p.c, N = p.N, cK = c + K;
    const int V2 = g & ((1 << m) - 1);
    const int V1 = (g >> m) & ((1 << m) - 1);
    const int sig = g >> (2 * m);
    const int sg2 = sig & ((1 << c) - 1);
    const int sg1 = sig >> c;
    const int d0 = tile * T;
    const int Dabs = p.out_base + d0;

    auto out_row_index = [&](int r1, int r2) -> long long {
        const int s1 = (sg1 << K) + r1, s2 = (sg2 << K) + r2;
        return ((((long long)s1 << cK) + s2) << (2 * m)) + ((long long)V1 << m) + V2;
    };
    Out *outp = reinterpret_cast<Out *>(p.out);
    const long long out_inst = FINAL ? (long long)inst * p.out_inst_stride : (long long)li * p.out_inst_stride;
    const int mos_b = inst / p.ndod, mos_j = inst - mos_b * p.ndod;
    auto mosaic_row = [&](int r1, int r2) -> long long {
        const int b = mos_b, j = mos_j;
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

    // ---- zero tiles (support D >= 2N - s1 - s2)
    {
        const int s1max = (sg1 << K) + S - 1, s2max = (sg2 << K) + S - 1;
        if (Dabs + T <= 2 * N - s1max - s2max) {
            constexpr int EPV = 16 / (int)sizeof(Out);
            const bool vz = (!FINAL || p.layout == 0) && ((p.out_pitch * (int)sizeof(Out)) % 16 == 0) &&
                            ((d0 * (int)sizeof(Out)) % 16 == 0) && (d0 + T <= p.out_width);
            if (vz) {
                for (int i = tid; i < S * S * (T / EPV); i += blockDim.x) {
                    const int rr = i / (T / EPV), q = i - rr * (T / EPV);
                    Out *dst = outp + out_inst + out_row_index(rr / S, rr % S) * p.out_pitch + d0 + q * EPV;
                    if (FINAL) st_cs_v4(dst, 0u, 0u, 0u, 0u);
                    else *reinterpret_cast<uint4 *>(dst) = make_uint4(0u, 0u, 0u, 0u);
                }
            } else {
                for (int i = tid; i < S * S * T; i += blockDim.x) {
                    const int rr = i / T, e = i - rr * T;
                    store_scalar(rr / S, rr % S, e, Acc(0));
                }
            }
            return;
        }
    }

    // ---- stage: SMEM chunk q of slot (w1, w2) = elements [st + EPC q, st + EPC (q+1)) of the
    // stage-c row, st = displacement of the row (its pre-shift); out-of-row chunks read as 0
    // (the stored rows are zero-padded up to their pitch).
    {
        const MidIn *inb = reinterpret_cast<const MidIn *>(p.in) + (long long)li * p.in_inst_stride;
        const int nc = p.n - c;
        const long long rbase = (((long long)sg1 << c) + sg2) << (2 * nc);
        const int nchunk = p.in_width / EPC;                 // chunks per stored row (width = pitch)
        constexpr int ITEMS = 4;
        for (int base = tid; base < S * S * NQ; base += blockDim.x * ITEMS) {
            uint4 lo[ITEMS], hi[ITEMS];
            int bsh[ITEMS], dst[ITEMS];
#pragma unroll
            for (int u = 0; u < ITEMS; ++u) {
                const int it = base + u * blockDim.x;
                dst[u] = -1;
                lo[u] = hi[u] = make_uint4(0u, 0u, 0u, 0u);
                if (it < S * S * NQ) {
                    const int slot = it / NQ, q = it - slot * NQ;
                    const int w1 = slot / S, w2 = slot - w1 * S;
                    const long long row = rbase + ((long long)((V1 << K) + w1) << nc) + (V2 << K) + w2;
                    const int e0 = Dabs + sg1 * w1 + sg2 * w2 - p.in_base + EPC * q;
                    const int c0 = floor_div(e0, EPC);
                    bsh[u] = (e0 - c0 * EPC) * (int)sizeof(MidIn);
                    dst[u] = slot * SP + 16 * q;
                    const uint4 *src = reinterpret_cast<const uint4 *>(inb + row * p.in_pitch);
                    if (c0 >= 0 && c0 < nchunk) lo[u] = __ldg(src + c0);
                    if (bsh[u] != 0 && c0 + 1 >= 0 && c0 + 1 < nchunk) hi[u] = __ldg(src + c0 + 1);
                }
            }
#pragma unroll
            for (int u = 0; u < ITEMS; ++u)
                if (dst[u] >= 0) *reinterpret_cast<uint4 *>(sm + dst[u]) = realign16(lo[u], hi[u], bsh[u]);
        }
    }
    __syncthreads();

    // ---- x-step: thread (w2, run) over rows w1; X kept in registers, then in place
    Acc acc[S][R];
    const bool xact = tid < G::XT;
    const int xr = tid % G::NRX, xw2 = tid / G::NRX;
    if (xact) {
#pragma unroll
        for (int r = 0; r < S; ++r)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[r][j] = Acc(0);
        const unsigned char *base = sm + xw2 * SP + xr * R * (int)sizeof(MidIn);
        direct_sum2<K, R, Acc>([&](auto a_, uint32_t *buf) {
            constexpr int a = decltype(a_)::value;
            load_run<MidIn, R + a>(base + a * S * SP, buf);
        }, acc);
    }
    __syncthreads();
    if (xact) {
#pragma unroll
        for (int r = 0; r < S; ++r) {
            unsigned char *slot = sm + (r * S + xw2) * SP;
#pragma unroll
            for (int q = 0; q < R / 4; ++q) {
                uint4 v;
                v.x = Lane<Acc>::bits(acc[r][4 * q + 0]);
                v.y = Lane<Acc>::bits(acc[r][4 * q + 1]);
                v.z = Lane<Acc>::bits(acc[r][4 * q + 2]);
                v.w = Lane<Acc>::bits(acc[r][4 * q + 3]);
                *reinterpret_cast<uint4 *>(slot + 16 * xswz(xr * (R / 4) + q)) = v;
            }
        }
    }
    __syncthreads();

    // ---- y-step: thread (r1, run) over X rows w2; store
    if (tid < G::YT) {
        const int yr = tid % G::NRY, r1 = tid / G::NRY;
#pragma unroll
        for (int r = 0; r < S; ++r)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[r][j] = Acc(0);
        const unsigned char *base = sm + (r1 * S) * SP;
        const int c0 = yr * (R / 4);
        direct_sum2<K, R, Acc>([&](auto a_, uint32_t *buf) {
            constexpr int a = decltype(a_)::value;
            const unsigned char *slot = base + a * SP;
#pragma unroll
            for (int i = 0; i < (R + a + 3) / 4; ++i) {
                const uint4 v = *reinterpret_cast<const uint4 *>(slot + 16 * xswz(c0 + i));
                buf[4 * i + 0] = v.x;
                if (4 * i + 1 < R + a) buf[4 * i + 1] = v.y;
                if (4 * i + 2 < R + a) buf[4 * i + 2] = v.z;
                if (4 * i + 3 < R + a) buf[4 * i + 3] = v.w;
            }
        }, acc);

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
