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
// tile of width T; all 4^K rows stay in shared memory as 32-bit lanes.
//
// Storage of a stage-c buffer (per instance = one (cube, dodecant) pair):
//   rows  ((s1 2^c + s2) 2^(n-c) + v1) 2^(n-c) + v2,     (N^2 rows)
//   D' = D - base_c with base_c = floor16(2N - 2(2^c - 1)) (the support of
//   eq:3Dfm at stage c starts at 2N - 2(2^c - 1)), rows computed and
//   zero-padded up to their pitch.  Stage 0 is the oriented cube itself
//   (base 2N, width N); the final stage is the stacked output out[s1][s2][D],
//   D in [0, 3N), zero outside the support.
#pragma once
#include <cuda.h>
#include "common.cuh"

// -DD3_PROF_PASS: per-phase clock accounting of the u16 final pass (thread 0 of each CTA),
// summed into d3_pass_prof[] (debug builds only)
#ifdef D3_PROF_PASS
__device__ unsigned long long d3_pass_prof[16];
#define PP_MARK(i) pp_t[i] = clock64()
#define PP_ADD(slot, a, b) do { if (pp_on) atomicAdd(&d3_pass_prof[slot], (unsigned long long)(pp_t[b] - pp_t[a])); } while (0)
#else
#define PP_MARK(i)
#define PP_ADD(slot, a, b) do { } while (0)
#endif

#ifndef D3_PF_GROUPS
#define D3_PF_GROUPS 0
#endif

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
    int next_k;                     // non-final passes: radix bits of the pass that reads this output
    int inst_total;                 // instances (cubes x dodecants) of the whole call
    int tma_store;                  // final pass: emit the output tile with one TMA tensor store
    int reduce_sub;                 // final fp32 pass: out <- out - A f (TMA reduce-add of -acc; the
                                    // inverse's residual update, invert.cu), zero tiles add nothing
    double *sq_part;                // final fp32 pass: per-CTA sum of out^2 (fp64) at
                                    // sq_part[(inst * gridDim.y + y) * gridDim.x + x], count in sq_count
    int *sq_count;
    uint32_t one;                   // = 1; a runtime multiplier so some adds issue as IMAD (FMA pipe)
    // zero tiles of the final output written by the first pass (DESIGN.md §5 item 6): the first
    // pass (zf_T > 0) writes the final pass's tiles of width zf_T that lie wholly below the support
    // into zf_out; the final pass (zeros_by_first) then skips them
    int zf_T;
    void *zf_out;
    long long zf_inst_stride;
    int zeros_by_first;
    Orient ori[kMaxDod];            // first pass: per-dodecant-slot orientation
    int8_t out_order[kMaxDod][2];   // mosaic: OutOrder[k][0..1]
    int8_t coords[kMaxDod][2];      // mosaic: DodecantCoords[k]
};

template <int K, int R, int T, bool STAGE16 = false>
struct DrtGeom {
    static constexpr int S = 1 << K;
    static constexpr int H = S - 1;                       // max l^K_r(w) = w <= S-1
    static constexpr int WIN = T + 2 * H;                 // input elements a tile needs per row
    static constexpr int NRX = (T + H + R - 1) / R;       // x-step runs per row (X needs T + H)
    static constexpr int NRY = T / R;                     // y-step runs per row
    static constexpr int EPS = STAGE16 ? 8 : 4;           // staged elements per 16-byte chunk
    static constexpr int RD = (NRX - 1) * R + (R + H + EPS - 1) / EPS * EPS;   // staged elements the x-step touches
    static constexpr int BW = ((WIN > RD ? WIN : RD) + 15) / 16 * 16; // staged elements per row
    // slot layout (bytes): staged row (u16 when STAGE16, else 32-bit with XOR-swizzled chunks);
    // X (32-bit, NRX*R words, XOR-swizzled chunks) is written in place over it.
    static constexpr int STAGED = BW * (STAGE16 ? 2 : 4);
    static constexpr int XB = NRX * R * 4;
    static constexpr int SP0 = (STAGED > XB ? STAGED : XB);
    static constexpr int SP = (SP0 + 15) / 16 * 16 + 16;  // slot pitch; +16 rotates banks per slot
    static constexpr int XT = S * NRX;                    // x-step tasks
    static constexpr int YT = S * NRY;                    // y-step tasks
    static constexpr int THREADS = ((XT > YT ? XT : YT) + 31) / 32 * 32;
    static constexpr int SMEM = S * S * SP;
    // two CTAs per SM: with W warps per CTA one SM sub-partition holds ceil(2W/4) warps of its
    // 16K-register file, which caps the registers per thread
    static constexpr int WARPS = THREADS / 32;
    // CTAS resident CTAs per SM (shared memory bound); with W warps per CTA one SM sub-partition
    // holds ceil(CTAS W / 4) warps of its 16K-register file, which caps the registers per thread
    static constexpr int CTAS0 = (227 * 1024) / (SMEM + 1024);
#ifndef D3_CTAS_MAX
#define D3_CTAS_MAX 8      // small-SMEM 32-bit passes (N <= 64): more resident CTAs, fewer registers;
                           // swept 4 / 6 / 8 / 10 / 12: 8 best (cfg5 0.860 -> 0.825 ms, cfg2 -4%)
#endif
    static constexpr int CTAS = CTAS0 < 1 ? 1 : (CTAS0 > D3_CTAS_MAX ? D3_CTAS_MAX : CTAS0);
    static constexpr int MAXREG0 = 16384 / (((CTAS * WARPS + 3) / 4) * 32) / 8 * 8;
    static constexpr int MAXREG = MAXREG0 > 255 ? 255 : MAXREG0;
    static_assert(T % R == 0 && R % 8 == 0, "tile shape");
    static_assert((NRY - 1) * R + (R + H + 3) / 4 * 4 <= NRX * R, "y-step reads inside X");
};

// Per-warp output stores of the u16 final pass (Y8 task mapping, 4 warps, S = 16): warp w owns
// r1 in [4w, 4w + 4), i.e. X slots [64w, 64w + 64), which no other warp reads in the y-step; it
// writes its output rows densely over those slots and issues its own TMA store (box {T, S, 4}),
// with no CTA-wide barrier.  The host builds the matching tensor map (launch.cuh).
#ifndef D3_WARP_STORE
#define D3_WARP_STORE 0               // measured: 0.7266 ms per final pass vs 0.7206 with the single CTA-wide store
#endif
template <int K, int R, int T, bool STAGE16, bool FINAL>
__host__ __device__ constexpr bool drt_warp_store() {
    return D3_WARP_STORE && STAGE16 && FINAL && K == 4 && R == 8 && DrtGeom<K, R, T, STAGE16>::NRY < 8 &&
           DrtGeom<K, R, T, STAGE16>::THREADS == 128;
}

// Hybrid output of the u16 final pass (Y8 mapping, 4 warps, S = 16): warps 0-1 (r1 < 8) write their
// half of the tile to shared memory over their own X slots and leave it with one TMA store (box
// {T, S, 8}), warps 2-3 (r1 >= 8) store theirs directly with 16-byte streaming stores; no CTA-wide
// barrier after the y-step, and the TMA drain overlaps the direct stores.
#ifndef D3_HYBRID_STORE
#define D3_HYBRID_STORE 0              // measured: final pass 0.6847 vs 0.6766 ms (bit-exact; off)
#endif
template <int K, int R, int T, bool STAGE16, bool FINAL>
__host__ __device__ constexpr bool drt_hybrid_store() {
    return D3_HYBRID_STORE && !D3_WARP_STORE && STAGE16 && FINAL && K == 4 && R == 8 &&
           DrtGeom<K, R, T, STAGE16>::NRY < 8 && DrtGeom<K, R, T, STAGE16>::THREADS == 128;
}

// XOR swizzle of 16-byte chunks (flip bit 0 in every other 8-chunk group): lanes
// that read runs R = 8 words apart (chunk stride 2) hit 8 distinct bank groups.
__device__ __forceinline__ int xswz(int c) { return c ^ ((c >> 3) & 1); }

// acc[r][j] += sum_a row_a[j + l^K_r(a)] over the S staged rows slot(a) =
// slot0 + a * sstep; the thread's run starts at chunk c0.  Rows are taken two
// at a time so the integer sums become 3-input adds.
// FMA16 of every 16 output rows take their adds on the FMA pipe (evenly spread over r).
__host__ __device__ constexpr bool fma_row(int r, int fma16) { return ((r + 1) * fma16) / 16 > (r * fma16) / 16; }

// FMA16 = -1: the measured default, rows with r % 4 < 1 (1/4 of the rows; swept 0 .. 3/8).
// TR (transposed, the backprojection pass of adjoint_pass.cuh): output r, input a at offset
// (S - 1) - l^K_a(r), i.e. acc[w][j] += row_r[j + H - l^K_r(w)].
// PB / PE: the row pairs (a0, a1) = (2p, 2p + 1), p in [PB, PE), taken (default: all).
template <int K, int R, int SP, bool U16, class Acc, int FMA16 = -1, bool TR = false, int PB = 0, int PE = (1 << K) / 2>
__device__ __forceinline__ void drt_accumulate(const unsigned char *__restrict__ sm, int slot0, int sstep, int c0,
                                               uint32_t one, Acc (&acc)[1 << K][R]) {
    constexpr int S = 1 << K;
    // U16: unswizzled u16 rows, run start = chunk c0 (8 elements per chunk); else 32-bit
    // rows with XOR-swizzled chunks, run start = chunk c0 (4 elements per chunk).
    auto load = [&](int a, int ne, uint32_t *buf) {
        const unsigned char *row = sm + (slot0 + a * sstep) * SP;
        if constexpr (U16) {
#pragma unroll
            for (int i = 0; i < (ne + 7) / 8; ++i) {
                const uint4 v = *reinterpret_cast<const uint4 *>(row + 16 * (c0 + i));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (8 * i + q < ne) buf[8 * i + q] = (q & 1) ? (w[q >> 1] >> 16) : (w[q >> 1] & 0xFFFFu);
            }
        } else {
#pragma unroll
            for (int i = 0; i < (ne + 3) / 4; ++i) {
                const uint4 v = *reinterpret_cast<const uint4 *>(row + 16 * xswz(c0 + i));
                buf[4 * i + 0] = v.x;
                if (4 * i + 1 < ne) buf[4 * i + 1] = v.y;
                if (4 * i + 2 < ne) buf[4 * i + 2] = v.z;
                if (4 * i + 3 < ne) buf[4 * i + 3] = v.w;
            }
        }
    };
    if constexpr (S == 1) {
        uint32_t b0[R];
        load(0, R, b0);
#pragma unroll
        for (int j = 0; j < R; ++j) acc[0][j] = acc[0][j] + Lane<Acc>::get(b0[j]);
    } else {
        static_for<PB, PE>([&](auto p_) {
            constexpr int a0 = 2 * decltype(p_)::value, a1 = a0 + 1;
            // forward offsets l^K_r(a) <= a; transposed ones (S - 1) - l^K_a(r) reach S - 1
            constexpr int n0 = R + (TR ? S - 1 : a0), n1 = R + (TR ? S - 1 : a1);
            uint32_t b0[n0], b1[n1];
            load(a0, n0, b0);
            load(a1, n1, b1);
            static_for<0, S>([&](auto r_) {
                constexpr int r = decltype(r_)::value;
                constexpr int o0 = TR ? (S - 1) - lk(K, a0, r) : lk(K, r, a0);
                constexpr int o1 = TR ? (S - 1) - lk(K, a1, r) : lk(K, r, a1);
// rows r with r % D3_FMA_MOD < D3_FMA_LT take their adds on the FMA pipe (round 2 re-sweep on the
// cfg3 final pass: none 764 µs, 1/8 701, 1/4 689, 3/8 704, rows 0-1 mod 4 682, 5/8 687, 3/4 711,
// even rows 677 -- and the backprojection 1.945 -> 1.768 ms); the transposed (adjoint) passes
// have their own pair, D3_ADJ_FMA_MOD / LT
#ifndef D3_FMA_MOD
#define D3_FMA_MOD 2
#define D3_FMA_LT 1
#endif
#ifndef D3_ADJ_FMA_MOD
#define D3_ADJ_FMA_MOD 2
#define D3_ADJ_FMA_LT 1
#endif
                constexpr bool fma = FMA16 < 0 ? (TR ? (r % D3_ADJ_FMA_MOD) < D3_ADJ_FMA_LT : (r % D3_FMA_MOD) < D3_FMA_LT)
                                               : fma_row(r, FMA16);
#ifndef D3_FADD2
#define D3_FADD2 0                  // measured slower: cfg5 0.758 vs 0.741 ms, N=256 f32 2.03 vs 1.98 ms
#endif
                if constexpr (std::is_same<Acc, float>::value && D3_FADD2 && R % 2 == 0) {
                    // fp32: two outputs per instruction (sm_100 FADD2), same summation order as add2
#pragma unroll
                    for (int j = 0; j < R; j += 2) {
                        float2 a = make_float2(acc[r][j], acc[r][j + 1]);
                        a = __fadd2_rn(a, make_float2(__uint_as_float(b0[j + o0]), __uint_as_float(b0[j + o0 + 1])));
                        a = __fadd2_rn(a, make_float2(__uint_as_float(b1[j + o1]), __uint_as_float(b1[j + o1 + 1])));
                        acc[r][j] = a.x;
                        acc[r][j + 1] = a.y;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < R; ++j) acc[r][j] = add2<Acc>(acc[r][j], b0[j + o0], b1[j + o1], one, fma);
                }
            });
        });
    }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <int K, int R, int T, class In, class Acc, class Out, bool FIRST, bool FINAL>
__global__ void __maxnreg__((DrtGeom<K, R, T, !FIRST && sizeof(In) == 2>::MAXREG))
drt_pass_kernel(const DrtPass p, const __grid_constant__ CUtensorMap omap) {
    constexpr bool STAGE16 = !FIRST && sizeof(In) == 2;
    using G = DrtGeom<K, R, T, STAGE16>;
#ifndef D3_SPLIT_STAGE
#define D3_SPLIT_STAGE 0                 // measured: cfg3 final pass 0.703 vs 0.677 ms (the extra barrier costs more than the overlap)
#endif
    // u16 final passes: the staged rows arrive in two cp.async groups (rows w1 < S/2, then the rest);
    // the x-step takes the first half's row pairs while the second half is still in flight
    constexpr bool SPLIT = D3_SPLIT_STAGE && STAGE16 && FINAL && K >= 2;
    constexpr int S = G::S, SP = G::SP, BW = G::BW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;

    const int tid = threadIdx.x;
    const int tile = blockIdx.x, g = blockIdx.y, li = blockIdx.z;
    const int inst = p.inst0 + li;
    const int m = p.m, c = p.c;
#ifndef D3_PDL
#define D3_PDL 1
#endif
    // the next pass may be scheduled from now on (programmatic dependent launch, DESIGN.md §5 item 8)
    if constexpr (!FINAL && D3_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int V2 = g & ((1 << m) - 1);
    const int V1 = (g >> m) & ((1 << m) - 1);
    const int sig = g >> (2 * m);
    const int sg2 = sig & ((1 << c) - 1);
    const int sg1 = sig >> c;
    const int d0 = tile * T;                 // stored output coordinate of the tile
    const int Dabs = p.out_base + d0;        // absolute displacement D of the tile start
    const int N = p.N;
    const int cK = c + K;

    // ---- output addressing: row (r1, r2) = row0(r1) + r2 * 2^(2m)
    Out *outp = reinterpret_cast<Out *>(p.out);
    const long long out_inst = FINAL ? (long long)inst * p.out_inst_stride : (long long)li * p.out_inst_stride;
    const long long r2_stride = (long long)p.out_pitch << (2 * m);
    auto row_ptr = [&](int r1) -> Out * {
        const long long s1 = (sg1 << K) + r1, s2 = (long long)sg2 << K;
        const long long row = (((s1 << cK) + s2) << (2 * m)) + ((long long)V1 << m) + V2;
        return outp + out_inst + row * p.out_pitch + d0;
    };
    // mosaic placement of a final row (Alg. 2 OutOrder / DodecantCoords)
    auto store_mosaic = [&](int r1, int r2, int e, Acc v) {
        const int D = d0 + e;
        if (D < 2 || D >= p.out_width) return;
        const int b = inst / p.ndod, j = inst - b * p.ndod;
        const int s[2] = {(sg1 << K) + r1, (sg2 << K) + r2};
        const int o0 = p.out_order[j][0], o1 = p.out_order[j][1];
        int w0 = s[(o0 < 0 ? -o0 : o0) - 1], w1 = s[(o1 < 0 ? -o1 : o1) - 1];
        if (o0 < 0) w0 = N - 1 - w0;
        if (o1 < 0) w1 = N - 1 - w1;
        const long long rr = (long long)(p.coords[j][0] * N + w0) * (4 * N) + (p.coords[j][1] * N + w1);
        outp[(long long)b * 16 * N * N * (3 * N - 2) + rr * (3 * N - 2) + D - 2] = to_out<Out, Acc>(v);
    };
    const bool mosaic = FINAL && p.layout == 1;
    // mosaic row of slopes (r1, r2) of this group: [b][4N][4N][3N - 2], element d = D - 2 (8-byte
    // aligned: the row pitch 3N - 2 and the run starts D0 - 2 are even)
    auto mosaic_row = [&](int r1, int r2) -> Out * {
        const int b = inst / p.ndod, j = inst - b * p.ndod;
        const int s[2] = {(sg1 << K) + r1, (sg2 << K) + r2};
        const int o0 = p.out_order[j][0], o1 = p.out_order[j][1];
        int w0 = s[(o0 < 0 ? -o0 : o0) - 1], w1 = s[(o1 < 0 ? -o1 : o1) - 1];
        if (o0 < 0) w0 = N - 1 - w0;
        if (o1 < 0) w1 = N - 1 - w1;
        const long long rr = (long long)(p.coords[j][0] * N + w0) * (4 * N) + (p.coords[j][1] * N + w1);
        return outp + (long long)b * 16 * N * N * (3 * N - 2) + rr * (3 * N - 2);
    };
    // elements [D0, D0 + n) of a mosaic row from registers v[0..n) (n even, D0 even): pairs as 8-byte
    // stores, D < 2 and D >= 3N dropped
    auto mosaic_run = [&](Out *row, int D0, const uint32_t *v, int n) {
        if (n == 8 && D0 >= 2 && D0 + 8 <= p.out_width) {
            // interior run of 8: 16-byte stores where the address allows (it is 8-byte aligned)
            unsigned char *dst = reinterpret_cast<unsigned char *>(row + D0 - 2);
            if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                *reinterpret_cast<uint4 *>(dst) = make_uint4(v[0], v[1], v[2], v[3]);
                *reinterpret_cast<uint4 *>(dst + 16) = make_uint4(v[4], v[5], v[6], v[7]);
            } else {
                *reinterpret_cast<uint2 *>(dst) = make_uint2(v[0], v[1]);
                *reinterpret_cast<uint4 *>(dst + 8) = make_uint4(v[2], v[3], v[4], v[5]);
                *reinterpret_cast<uint2 *>(dst + 24) = make_uint2(v[6], v[7]);
            }
            return;
        }
        for (int q = 0; q < n; q += 2) {
            const int D = D0 + q;
            if (D >= 2 && D + 2 <= p.out_width)
                *reinterpret_cast<uint2 *>(row + D - 2) = make_uint2(v[q], v[q + 1]);
        }
    };

    // ---- final tiles entirely outside the support of all 4^K output rows: zeros
    // (support D >= 2N - s1 - s2).  Intermediate tiles are always computed so
    // that their pre-shifted chunks are written by exactly one pattern.
    if constexpr (FINAL) {
        const int s1max = (sg1 << K) + S - 1, s2max = (sg2 << K) + S - 1;
        if (Dabs + T <= 2 * N - s1max - s2max) {
            if (p.sq_part && tid == 0) {
                p.sq_part[((long long)inst * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = 0.0;
                if (blockIdx.x == 0 && blockIdx.y == 0 && li == 0) *p.sq_count = p.inst_total * (int)(gridDim.x * gridDim.y);
            }
            if (p.zeros_by_first) return;                // already written by the first pass
            if (p.reduce_sub) return;                    // out - 0 = out
#ifndef D3_ZERO_TMA
#define D3_ZERO_TMA 1
#endif
            if constexpr (sizeof(Out) == 4 && D3_ZERO_TMA && !drt_warp_store<K, R, T, STAGE16, FINAL>()) {
                if (p.tma_store) {
                    // a zeroed shared-memory image of the tile leaves with one TMA tensor store (the
                    // CTA is done once the TMA engine has read it) instead of S*S*T/4 16-byte stores
                    for (int i = tid; i < S * S * T / 4; i += blockDim.x)
                        reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncthreads();
                    if (tid == 0) {
                        const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
                        constexpr int NH = drt_hybrid_store<K, R, T, STAGE16, FINAL>() ? 2 : 1;   // box {T, S, S / NH}
#pragma unroll
                        for (int h = 0; h < NH; ++h)
                            asm volatile(
                                "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&omap),
                                "r"(d0), "r"(sg2 << K), "r"((sg1 << K) + h * (S / NH)), "r"(inst), "r"(src)
                                : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    }
                    return;
                }
            }
            constexpr int EPV = 16 / (int)sizeof(Out);
            const bool vz = !mosaic && ((p.out_pitch * (int)sizeof(Out)) % 16 == 0) &&
                            ((d0 * (int)sizeof(Out)) % 16 == 0) && (d0 + T <= p.out_width);
            if (vz) {
                for (int i = tid; i < S * S * (T / EPV); i += blockDim.x) {
                    const int rr = i / (T / EPV), q = i - rr * (T / EPV);
                    Out *dst = row_ptr(rr / S) + (rr % S) * r2_stride + q * EPV;
                    if (FINAL) st_cs_v4(dst, 0u, 0u, 0u, 0u);
                    else *reinterpret_cast<uint4 *>(dst) = make_uint4(0u, 0u, 0u, 0u);
                }
            } else {
                if (mosaic && (T % 2) == 0 && (d0 % 2) == 0) {
                    // zero runs of 8 (or the tile's tail) per mosaic row, 8-byte stores
                    constexpr int RUN = 8;
                    const uint32_t z[RUN] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                    for (int i = tid; i < S * S * ((T + RUN - 1) / RUN); i += blockDim.x) {
                        const int rr = i / ((T + RUN - 1) / RUN), q = i - rr * ((T + RUN - 1) / RUN);
                        const int n = T - RUN * q < RUN ? T - RUN * q : RUN;
                        mosaic_run(mosaic_row(rr / S, rr % S), d0 + RUN * q, z, n);
                    }
                    return;
                }
                for (int i = tid; i < S * S * T; i += blockDim.x) {
                    const int rr = i / T, e = i - rr * T;
                    if (mosaic) store_mosaic(rr / S, rr % S, e, Acc(0));
                    else if (d0 + e < p.out_width) row_ptr(rr / S)[(rr % S) * r2_stride + e] = to_out<Out, Acc>(Acc(0));
                }
            }
            return;
        }
    }

#ifdef D3_PROF_PASS
    const bool pp_on = tid == 0 && STAGE16 && FINAL;
    long long pp_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    // programmatic dependent launch (DESIGN.md §5 item 8): a final pass may be scheduled while the
    // pass that writes its input finishes; zero tiles (above) need nothing from it, the rest wait
    // here until that grid has completed and its writes are visible (a no-op without PDL)
    if constexpr (!FIRST && D3_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    PP_MARK(0);
    // ---- stage the 4^K input rows of the group (32-bit lanes, BW elements per slot)
    auto put = [&](int slot, int e, uint32_t bits) {
        *reinterpret_cast<uint32_t *>(sm + slot * SP + 16 * xswz(e >> 2) + 4 * (e & 3)) = bits;
    };
    auto put4 = [&](int slot, int chunk, uint4 v) {
        *reinterpret_cast<uint4 *>(sm + slot * SP + 16 * xswz(chunk)) = v;
    };
    if constexpr (FIRST) {
        const Orient o = p.ori[inst % p.ndod];
        const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
        const int z0 = Dabs - 2 * N;       // z' of element 0 (stage-0 rows: D = z' + 2N)
        const int xb = V1 << K, yb = V2 << K;
        if (sizeof(In) == 1 && p.vec_ok && o.fast == 2 && o.sz > 0 && (z0 & 15) == 0) {
            // u8 rows along z' (forward, 16-aligned): one LDG.128 = 16 voxels = 4 SMEM chunks
            constexpr int NQ16 = BW / 16;
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
#pragma unroll
                    for (int h = 0; h < 4; ++h)
                        put4(sl[u], 4 * qq[u] + h,
                             make_uint4(__byte_perm(w[h], 0, 0x4440), __byte_perm(w[h], 0, 0x4441),
                                        __byte_perm(w[h], 0, 0x4442), __byte_perm(w[h], 0, 0x4443)));
                }
            }
        } else if (sizeof(In) == 1 && K == 4 && p.vec_ok && o.fast != 2) {
            // u8, unit stride along x' (fast 0) or y' (fast 1): one LDG.128 = the 16 voxels of a
            // run along that axis; 4 consecutive z' per item are transposed in registers so every
            // SMEM write is a 16-byte chunk (4 consecutive e of one slot)
            const bool fx = o.fast == 0;
            const long long sf = fx ? o.sx : o.sy, so = fx ? o.sy : o.sx;
            const int fb = fx ? xb : yb, ob = fx ? yb : xb;
            constexpr int NG = BW / 4;
            for (int it = tid; it < S * NG; it += blockDim.x) {
                const int other = it % S, gq = it / S;
                uint4 v[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int z = z0 + 4 * gq + t;
                    v[t] = make_uint4(0u, 0u, 0u, 0u);
                    if ((unsigned)z < (unsigned)N) {
                        const long long b = o.off0 + (long long)(ob + other) * so + (long long)z * o.sz +
                                            (sf > 0 ? (long long)fb : -(long long)(fb + 15));
                        v[t] = __ldg(reinterpret_cast<const uint4 *>(cube + b));
                    }
                }
#pragma unroll
                for (int wf = 0; wf < 16; ++wf) {
                    const int byte = sf > 0 ? wf : 15 - wf;
                    uint32_t q4[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint32_t w[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
                        q4[t] = __byte_perm(w[byte >> 2], 0, 0x4440 | (byte & 3));
                    }
                    put4(fx ? wf * S + other : other * S + wf, gq, make_uint4(q4[0], q4[1], q4[2], q4[3]));
                }
            }
        } else if (sizeof(In) == 4 && K >= 2 && p.vec_ok && (z0 & 3) == 0 && (o.fast != 2 || o.sz > 0)) {
            // 32-bit voxels: LDG.128 = 4 voxels.  Along z' (forward) they are one staged chunk;
            // along x' or y' they are 4 rows at one z', so 4 consecutive z' are loaded per item
            // and transposed in registers (reversed axes: the 4 values in reverse order).
            constexpr int NQ4 = BW / 4;
            if (o.fast == 2) {
                // ITEMS independent loads in flight per thread before any is stored (one load per
                // iteration left each thread waiting a full L2 round trip per chunk)
                constexpr int ITEMS = 8;
                for (int base = tid; base < S * S * NQ4; base += blockDim.x * ITEMS) {
                    uint4 v[ITEMS];
#pragma unroll
                    for (int u = 0; u < ITEMS; ++u) {
                        const int it = base + u * blockDim.x;
                        const int slot = it / NQ4, q = it - slot * NQ4;
                        const int w1 = slot / S, w2 = slot - w1 * S, z = z0 + 4 * q;
                        v[u] = make_uint4(0u, 0u, 0u, 0u);
                        if (it < S * S * NQ4 && (unsigned)z < (unsigned)N)
                            v[u] = __ldg(reinterpret_cast<const uint4 *>(cube + o.off0 + (long long)(xb + w1) * o.sx +
                                                                         (long long)(yb + w2) * o.sy + z));
                    }
#pragma unroll
                    for (int u = 0; u < ITEMS; ++u) {
                        const int it = base + u * blockDim.x;
                        if (it < S * S * NQ4) put4(it / NQ4, it - (it / NQ4) * NQ4, v[u]);
                    }
                }
            } else {
                const bool fy = o.fast == 1;
                const long long sf = fy ? o.sy : o.sx, so = fy ? o.sx : o.sy;
                const int fb = fy ? yb : xb, ob = fy ? xb : yb;
                // two items (8 loads) in flight per thread before any is stored
                constexpr int ITEMS = 2;
                for (int base = tid; base < S * (S / 4) * NQ4; base += blockDim.x * ITEMS) {
                    uint4 a[ITEMS][4];
#pragma unroll
                    for (int u = 0; u < ITEMS; ++u) {
                        const int it = base + u * blockDim.x;
                        const int q = it % NQ4, rest = it / NQ4, g4 = rest % (S / 4), other = rest / (S / 4);
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const int z = z0 + 4 * q + t;
                            a[u][t] = make_uint4(0u, 0u, 0u, 0u);
                            if (it < S * (S / 4) * NQ4 && (unsigned)z < (unsigned)N) {
                                const long long b = o.off0 + (long long)(ob + other) * so + (long long)z * o.sz +
                                                    (sf > 0 ? (long long)(fb + 4 * g4) : -(long long)(fb + 4 * g4 + 3));
                                a[u][t] = __ldg(reinterpret_cast<const uint4 *>(cube + b));
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < ITEMS; ++u) {
                        const int it = base + u * blockDim.x;
                        if (it >= S * (S / 4) * NQ4) break;
                        const int q = it % NQ4, rest = it / NQ4, g4 = rest % (S / 4), other = rest / (S / 4);
                        uint32_t v[4][4];
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const uint32_t av[4] = {a[u][t].x, a[u][t].y, a[u][t].z, a[u][t].w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) v[t][j] = av[sf > 0 ? j : 3 - j];
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int f = 4 * g4 + j;
                            put4(fy ? other * S + f : f * S + other, q, make_uint4(v[0][j], v[1][j], v[2][j], v[3][j]));
                        }
                    }
                }
            }
        } else {
            // generic (any voxel type, any orientation, small N): element by element
            for (int i = tid; i < S * S * BW; i += blockDim.x) {
                const int e = i % BW, slot = i / BW;
                const int w1 = slot / S, w2 = slot % S, z = z0 + e;
                uint32_t bits = 0;
                if ((unsigned)z < (unsigned)N)
                    bits = Elem<In>::load_bits(cube + o.off0 + (long long)(xb + w1) * o.sx +
                                               (long long)(yb + w2) * o.sy + (long long)z * o.sz);
                put(slot, e, bits);
            }
        }
    } else {
        // stage-c rows, stored with the residual pre-shift (writer side, DESIGN.md "Aligned stage
        // buffers"): the slot's window starts at stored element
        //   (Dabs - in_base) + EPC * floor((s1 w1 + s2 w2) / EPC),
        // a chunk boundary, so staging is a plain aligned 16-byte copy (cp.async, zero-filled
        // outside the stored row).  Consecutive threads take consecutive chunks of one row.
        constexpr int EPC = 16 / (int)sizeof(In);          // stored elements per 16-byte chunk
        constexpr int LOG_EPC = EPC == 8 ? 3 : 2;
        constexpr int NCH = BW / EPC;                      // chunks per staged row
        static_assert(BW % EPC == 0, "staging chunks");
        const In *inb = reinterpret_cast<const In *>(p.in) + (long long)li * p.in_inst_stride;
        const int nc = p.n - c;
        const long long rbase = (((long long)sg1 << c) + sg2) << (2 * nc);
        const int nchunk = p.in_width >> LOG_EPC;          // chunks per stored row (width = pitch)
#if D3_PF_GROUPS > 0
        // L2 prefetch: the first D tile of each group pulls the rows of the group D3_PF_GROUPS ahead
        // (the tiles of one group run together; the intermediate may have left L2)
        if (tile == 0 && tid < S) {
            const int gp = g + D3_PF_GROUPS;
            if (gp < (int)gridDim.y) {
                const int mm = (1 << m) - 1;
                const int pV2 = gp & mm, pV1 = (gp >> m) & mm, psig = gp >> (2 * m);
                const long long prow = ((((long long)(psig >> c) << c) + (psig & ((1 << c) - 1))) << (2 * nc)) +
                                       ((long long)((pV1 << K) + tid) << nc) + (pV2 << K);
                const unsigned bytes = (unsigned)(S * p.in_pitch * (int)sizeof(In));
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(inb + prow * p.in_pitch), "r"(bytes)
                             : "memory");
            }
        }
#endif
        const int cb = (Dabs - p.in_base) >> LOG_EPC;      // exact: Dabs - in_base is a multiple of 16
        // thread (sub, q) copies chunk q of slots sub, sub + SUBS, ...: the per-copy work is the
        // slot's shift term and one address add
        constexpr int SUBS = G::THREADS / NCH;             // slots in flight per iteration
        const int q = tid % NCH, sub = tid / NCH;
#ifdef D3_BULK_STAGE
        if constexpr (STAGE16) {
            // one 1-D bulk copy (TMA engine, completes on an mbarrier) per staged row whose window
            // lies inside its stored row: NCH * 16 contiguous, 16-byte-aligned bytes each (rows are
            // pre-shifted); warp 0 issues them.  Rows reaching
            // past either end of the stored row take the zero-filling cp.async path below.
            __shared__ __align__(8) uint64_t stage_bar;
            const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&stage_bar));
            if (tid == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(32) : "memory");
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncthreads();
            const In *rb = inb + (rbase + ((long long)(V1 << K) << nc) + (V2 << K)) * p.in_pitch;
            if (tid < 32) {
                uint32_t bytes = 0;
                for (int slot = tid; slot < S * S; slot += 32) {
                    const int w1 = slot >> K, w2 = slot & (S - 1);
                    const int cc = cb + ((sg1 * w1 + sg2 * w2) >> LOG_EPC);
                    if (cc >= 0 && cc + NCH <= nchunk) {
                        const char *src = reinterpret_cast<const char *>(rb) +
                                          ((size_t)((w1 << nc) + w2) * p.in_pitch + (size_t)cc * EPC) * sizeof(In);
                        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sm + slot * SP));
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                            "l"(src), "r"(NCH * 16), "r"(bar)
                            : "memory");
                        bytes += NCH * 16;
                    }
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            }
            // edge rows: chunk-wise with zero fill
            for (int i = tid; i < S * S * NCH; i += G::THREADS) {
                const int slot = i / NCH, qq = i - slot * NCH;
                const int w1 = slot >> K, w2 = slot & (S - 1);
                const int c0r = cb + ((sg1 * w1 + sg2 * w2) >> LOG_EPC);
                if (c0r >= 0 && c0r + NCH <= nchunk) continue;
                const int cc = c0r + qq;
                const bool ok = (unsigned)cc < (unsigned)nchunk;
                const uint32_t off =
                    ((uint32_t)((w1 << nc) + w2) * (uint32_t)p.in_pitch + (uint32_t)(ok ? cc : 0) * EPC) * (uint32_t)sizeof(In);
                cp_async16(sm + slot * SP + 16 * qq, reinterpret_cast<const char *>(rb) + off, ok);
            }
            PP_MARK(1);
            cp_async_wait_all();
            asm volatile(
                "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(bar)
                : "memory");
        } else
#endif
        if (sub < SUBS) {
            const In *rb = inb + (rbase + ((long long)(V1 << K) << nc) + (V2 << K)) * p.in_pitch;
            unsigned char *dst = sm + sub * SP + 16 * (STAGE16 ? q : xswz(q));
            const int cq = cb + q;
            auto copy = [&](int slot) {
                const int w1 = slot >> K, w2 = slot & (S - 1);
                const int cc = cq + ((sg1 * w1 + sg2 * w2) >> LOG_EPC);
                const bool ok = (unsigned)cc < (unsigned)nchunk;
                const uint32_t off = ((uint32_t)((w1 << nc) + w2) * (uint32_t)p.in_pitch + (uint32_t)(ok ? cc : 0) * EPC) *
                                     (uint32_t)sizeof(In);
                cp_async16(dst, reinterpret_cast<const char *>(rb) + off, ok);
            };
            int slot = sub;
            if constexpr (SPLIT) {
                // rows w1 < S/2 (slots below S*S/2) in the first commit group, the rest in the second
#pragma unroll 4
                for (; slot < S * S / 2; slot += SUBS, dst += SUBS * SP) copy(slot);
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
#pragma unroll 4
            for (; slot < S * S; slot += SUBS, dst += SUBS * SP) copy(slot);
        }
        PP_MARK(1);
        if constexpr (SPLIT) {
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;\n" ::: "memory");
        } else {
            cp_async_wait_all();
        }
    }
    __syncthreads();
    PP_MARK(2);

    // ---- x-step (rows w1 of slot (w1, w2) -> X(r1, w2)), written in place over slot (r1, w2),
    // then y-step (rows w2 of X slot (r1, w2) -> out(r1, r2)); one code path, two iterations.
    Acc acc[S][R];
    int xb, xr;
    task_row_run(tid, G::NRX, S, xb, xr);
#ifndef D3_Y8
#define D3_Y8 1
#endif
    // y-step task (r1 = yb, run yr).  With fewer than 8 runs per row (T=48: 6) a quarter-warp of
    // the compact mapping spans two rows whose X slots sit 16 x 17 chunks = 0 (mod 8 bank groups)
    // apart, so their reads collide; giving each row 8 lanes (the last NRY..7 idle) keeps every
    // quarter-warp on one row and its chunk reads conflict-free.
    constexpr bool Y8 = D3_Y8 && STAGE16 && FINAL && G::NRY < 8 && G::THREADS >= 8 * S;
    const int yr = Y8 ? (tid & 7) : tid % G::NRY, yb = Y8 ? (tid >> 3) : tid / G::NRY;
    const bool yact = Y8 ? (yr < G::NRY) : (tid < G::YT);
    auto zero_acc = [&]() {
#pragma unroll
        for (int i = 0; i < S; ++i)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[i][j] = Acc(0);
    };
    auto write_x = [&]() {
#pragma unroll
        for (int i = 0; i < S; ++i) {
#pragma unroll
            for (int q = 0; q < R / 4; ++q)
                put4(i * S + xb, xr * (R / 4) + q,
                     make_uint4(Lane<Acc>::bits(acc[i][4 * q + 0]), Lane<Acc>::bits(acc[i][4 * q + 1]),
                                Lane<Acc>::bits(acc[i][4 * q + 2]), Lane<Acc>::bits(acc[i][4 * q + 3])));
        }
    };
    if constexpr (STAGE16) {
        // x-step reads the u16 staged rows, y-step the 32-bit X rows
        if constexpr (SPLIT) {
            if (tid < G::XT) {
                zero_acc();
                drt_accumulate<K, R, SP, true, Acc, -1, false, 0, S / 4>(sm, xb, S, xr * (R / 8), p.one, acc);
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();                                 // every thread's second-half rows have landed
            if (tid < G::XT) drt_accumulate<K, R, SP, true, Acc, -1, false, S / 4, S / 2>(sm, xb, S, xr * (R / 8), p.one, acc);
        } else if (tid < G::XT) {
            zero_acc();
            drt_accumulate<K, R, SP, true, Acc>(sm, xb, S, xr * (R / 8), p.one, acc);
        }
        PP_MARK(3);
        __syncthreads();
        PP_MARK(4);
        if (tid < G::XT) write_x();
        __syncthreads();
        PP_MARK(5);
        if (yact) {
            zero_acc();
            drt_accumulate<K, R, SP, false, Acc>(sm, yb * S, 1, yr * (R / 4), p.one, acc);
        }
        PP_MARK(6);
    } else {
        // both steps read 32-bit rows: one code path, two iterations
#pragma unroll 1
        for (int step = 0; step < 2; ++step) {
            const bool act = step ? yact : (tid < G::XT);
            const int r = step ? yr : xr, b = step ? yb : xb;
            if (act) {
                zero_acc();
                drt_accumulate<K, R, SP, false, Acc>(sm, step ? b * S : b, step ? 1 : S, r * (R / 4), p.one, acc);
            }
            if (step == 0) {
                __syncthreads();
                if (act) write_x();
                __syncthreads();
            }
        }
    }

    // ---- intermediate output: rows stored pre-shifted by rho (see common.cuh), realigned
    // across the NRY runs of a row with one shuffle per word
    if constexpr (!FINAL) {
        if (yact) {
            constexpr int E = 4 / (int)sizeof(Out);        // elements per 32-bit word
            constexpr int EPC = 4 * E;                     // elements per 16-byte chunk
            constexpr int NWO = R / E;                     // words per run
            constexpr int NCK = R / EPC;                   // chunks per run
            const int mK = (1 << p.next_k) - 1;
            const int r1 = yb, e0 = yr * R;
            const long long s1 = ((long long)sg1 << K) + r1;
            const long long wv1 = V1 & mK, wv2 = V2 & mK;
            Out *rowp = row_ptr(r1) + e0;
#pragma unroll
            for (int r2 = 0; r2 < S; ++r2, rowp += r2_stride) {
                const long long s2 = ((long long)sg2 << K) + r2;
                const int rho = (int)((s1 * wv1 + s2 * wv2) & (EPC - 1));
                uint32_t win[NWO + 4];
#pragma unroll
                for (int i = 0; i < NWO; ++i) {
                    if constexpr (E == 2) win[i] = __byte_perm(Lane<Acc>::bits(acc[r2][2 * i]), Lane<Acc>::bits(acc[r2][2 * i + 1]), 0x5410);
                    else win[i] = Lane<Acc>::bits(acc[r2][i]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) win[NWO + i] = __shfl_down_sync(0xffffffffu, win[i], 1, G::NRY);
#ifndef D3_STAGE_ST256
#define D3_STAGE_ST256 0          // measured slower: f32 N = 256 x12 2.004 vs 1.937 ms, i32 1.822 vs 1.784, N = 128 0.232 vs 0.220
#endif
                if constexpr (D3_STAGE_ST256 && NCK == 2) {
                    // a run's two chunks as one 32-byte store (STG.256, §5 item 9) except the row's last run
                    if (yr != G::NRY - 1 && d0 + e0 + EPC < p.out_width && (reinterpret_cast<unsigned long long>(rowp) & 31ull) == 0) {
                        uint32_t v0[4], v1[4];
                        window_chunk<E>(win, rho, 0, v0);
                        window_chunk<E>(win, rho, 1, v1);
                        const uint32_t v8[8] = {v0[0], v0[1], v0[2], v0[3], v1[0], v1[1], v1[2], v1[3]};
                        st_v8(rowp, v8);
                        goto stored;
                    }
                }
#pragma unroll
                for (int q = 0; q < NCK; ++q) {
                    uint32_t v[4];
                    window_chunk<E>(win, rho, q, v);
                    if (d0 + e0 + q * EPC < p.out_width) {
                        if (yr == G::NRY - 1 && q == NCK - 1) store_chunk_head<E>(rowp + q * EPC, v, EPC - rho);
                        else *reinterpret_cast<uint4 *>(rowp + q * EPC) = make_uint4(v[0], v[1], v[2], v[3]);
                    }
                }
            stored:;
                if (yr == 0 && rho > 0 && d0 >= EPC) {
                    // own elements [0, rho) end the previous chunk (whose head the previous tile wrote)
                    uint32_t tw[NWO + 4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) tw[i] = win[i];
#pragma unroll
                    for (int i = 0; i < NWO; ++i) tw[4 + i] = win[i];
                    uint32_t v[4];
                    window_chunk<E>(tw, rho, 0, v);
                    store_chunk_tail<E>(rowp - EPC, v, rho);
                }
            }
        }
        return;
    }

    // ---- final output via SMEM + one TMA tensor store (stacked layout, m = 0): the tile is the
    // box {T, S (s2), S (s1), 1} of out[inst][s1][s2][3N]
    if constexpr (FINAL && sizeof(Out) == 4 && drt_hybrid_store<K, R, T, STAGE16, FINAL>()) {
        if (p.tma_store) {
            static_assert(Y8 && R == 8 && S == 16, "hybrid stores: Y8 mapping");
            if (tid < 64) {
                // rows r1 < 8: their X slots [0, 8 S) are read only by warps 0-1
                asm volatile("bar.sync 1, 64;" ::: "memory");
                if (yact) {
                    unsigned char *row = sm + ((yb * S) * T + yr * R) * 4;
                    const bool sw = (yr & 4) != 0;
#pragma unroll
                    for (int r2 = 0; r2 < S; ++r2) {
                        const uint4 c0 = make_uint4(Lane<Acc>::bits(acc[r2][0]), Lane<Acc>::bits(acc[r2][1]),
                                                    Lane<Acc>::bits(acc[r2][2]), Lane<Acc>::bits(acc[r2][3]));
                        const uint4 c1 = make_uint4(Lane<Acc>::bits(acc[r2][4]), Lane<Acc>::bits(acc[r2][5]),
                                                    Lane<Acc>::bits(acc[r2][6]), Lane<Acc>::bits(acc[r2][7]));
                        *reinterpret_cast<uint4 *>(row + (r2 * T + (sw ? 4 : 0)) * 4) = sw ? c1 : c0;
                        *reinterpret_cast<uint4 *>(row + (r2 * T + (sw ? 0 : 4)) * 4) = sw ? c0 : c1;
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, 64;" ::: "memory");
                if (tid == 0) {
                    const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
                    asm volatile(
                        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&omap),
                        "r"(d0), "r"(sg2 << K), "r"(sg1 << K), "r"(inst), "r"(src)
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
            } else if (yact) {
                // rows r1 >= 8: 16-byte streaming stores straight from the registers
                Out *dst = row_ptr(yb) + yr * R;
#pragma unroll
                for (int r2 = 0; r2 < S; ++r2, dst += r2_stride) {
                    st_cs_v4(dst, Lane<Acc>::bits(acc[r2][0]), Lane<Acc>::bits(acc[r2][1]), Lane<Acc>::bits(acc[r2][2]),
                             Lane<Acc>::bits(acc[r2][3]));
                    st_cs_v4(dst + 4, Lane<Acc>::bits(acc[r2][4]), Lane<Acc>::bits(acc[r2][5]), Lane<Acc>::bits(acc[r2][6]),
                             Lane<Acc>::bits(acc[r2][7]));
                }
            }
            return;
        }
    } else if constexpr (FINAL && sizeof(Out) == 4 && drt_warp_store<K, R, T, STAGE16, FINAL>()) {
        if (p.tma_store) {
            static_assert(Y8 && R == 8 && S == 16, "per-warp stores: Y8 mapping");
            const int wq = tid >> 5;
            unsigned char *wbase = sm + wq * 64 * SP;         // this warp's X slots, 128-byte aligned
            __syncwarp();                                    // the warp's y-step reads of them are done
            if (yact) {
                unsigned char *row = wbase + (((yb & 3) * S) * T + yr * R) * 4;
                const bool sw = (yr & 4) != 0;               // runs 4..: chunks in swapped order (banks)
#pragma unroll
                for (int r2 = 0; r2 < S; ++r2) {
                    const uint4 c0 = make_uint4(Lane<Acc>::bits(acc[r2][0]), Lane<Acc>::bits(acc[r2][1]),
                                                Lane<Acc>::bits(acc[r2][2]), Lane<Acc>::bits(acc[r2][3]));
                    const uint4 c1 = make_uint4(Lane<Acc>::bits(acc[r2][4]), Lane<Acc>::bits(acc[r2][5]),
                                                Lane<Acc>::bits(acc[r2][6]), Lane<Acc>::bits(acc[r2][7]));
                    *reinterpret_cast<uint4 *>(row + (r2 * T + (sw ? 4 : 0)) * 4) = sw ? c1 : c0;
                    *reinterpret_cast<uint4 *>(row + (r2 * T + (sw ? 0 : 4)) * 4) = sw ? c0 : c1;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if ((tid & 31) == 0) {
                const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(wbase));
                asm volatile(
                    "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&omap),
                    "r"(d0), "r"(sg2 << K), "r"((sg1 << K) + 4 * wq), "r"(inst), "r"(src)
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
#ifdef D3_PROF_PASS
            PP_MARK(7);
            PP_ADD(0, 0, 1);
            PP_ADD(1, 1, 2);
            PP_ADD(2, 2, 3);
            PP_ADD(3, 3, 4);
            PP_ADD(4, 4, 5);
            PP_ADD(5, 5, 6);
            PP_ADD(6, 6, 7);
            if (pp_on) atomicAdd(&d3_pass_prof[7], 1ull);
#endif
            return;
        }
    } else if constexpr (FINAL && sizeof(Out) == 4) {
        if (p.tma_store) {
            __shared__ double sq_warp[32];
            double sq_thread = 0.0;
            __syncthreads();                                 // every y-step read of X is done
            if (yact) {
                unsigned char *row = sm + ((yb * S) * T + yr * R) * 4;
#ifndef D3_Y8_STORE_SWAP
#define D3_Y8_STORE_SWAP 1
#endif
                if constexpr (std::is_same<Acc, float>::value) {
                    if (p.sq_part) {                     // this thread's share of sum out^2 (fp64, fixed order)
                        double ss = 0.0;
#pragma unroll
                        for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                            for (int j = 0; j < R; ++j) ss += (double)acc[r2][j] * (double)acc[r2][j];
                        sq_thread = ss;
                    }
                    if (p.reduce_sub) {                  // the tile is added to out: -acc
#pragma unroll
                        for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                            for (int j = 0; j < R; ++j) acc[r2][j] = -acc[r2][j];
                    }
                }
                if constexpr ((Y8 || G::NRY == 8) && R == 8 && D3_Y8_STORE_SWAP) {
                    // runs 4.. write their two chunks in the opposite order: with runs 0..3 they
                    // then cover 8 distinct bank groups per store instruction of a quarter-warp
                    // (one row per quarter-warp: the Y8 mapping, or 8 runs per row at T = 64)
                    const bool sw = (yr & 4) != 0;
#pragma unroll
                    for (int r2 = 0; r2 < S; ++r2) {
                        const uint4 c0 = make_uint4(Lane<Acc>::bits(acc[r2][0]), Lane<Acc>::bits(acc[r2][1]),
                                                    Lane<Acc>::bits(acc[r2][2]), Lane<Acc>::bits(acc[r2][3]));
                        const uint4 c1 = make_uint4(Lane<Acc>::bits(acc[r2][4]), Lane<Acc>::bits(acc[r2][5]),
                                                    Lane<Acc>::bits(acc[r2][6]), Lane<Acc>::bits(acc[r2][7]));
                        *reinterpret_cast<uint4 *>(row + (r2 * T + (sw ? 4 : 0)) * 4) = sw ? c1 : c0;
                        *reinterpret_cast<uint4 *>(row + (r2 * T + (sw ? 0 : 4)) * 4) = sw ? c0 : c1;
                    }
                } else {
#pragma unroll
                    for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                        for (int q = 0; q < R / 4; ++q)
                            *reinterpret_cast<uint4 *>(row + (r2 * T + 4 * q) * 4) =
                                make_uint4(Lane<Acc>::bits(acc[r2][4 * q]), Lane<Acc>::bits(acc[r2][4 * q + 1]),
                                           Lane<Acc>::bits(acc[r2][4 * q + 2]), Lane<Acc>::bits(acc[r2][4 * q + 3]));
                }
            }
            if (std::is_same<Acc, float>::value && p.sq_part) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sq_thread += __shfl_xor_sync(0xffffffffu, sq_thread, o);
                if ((tid & 31) == 0) sq_warp[tid >> 5] = sq_thread;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (std::is_same<Acc, float>::value && p.sq_part && tid == 0) {
                double t = 0.0;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sq_warp[w];
                p.sq_part[((long long)inst * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
                if (blockIdx.x == 0 && blockIdx.y == 0 && li == 0) *p.sq_count = p.inst_total * (int)(gridDim.x * gridDim.y);
            }
            if (tid == 0) {
                const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
#ifdef D3_TMA_EVICT_FIRST
                uint64_t pol;
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                asm volatile(
                    "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], [%5], %6;" ::"l"(&omap),
                    "r"(d0), "r"(sg2 << K), "r"(sg1 << K), "r"(inst), "r"(src), "l"(pol)
                    : "memory");
#else
                if (std::is_same<Acc, float>::value && p.reduce_sub)
                    asm volatile(
                        "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&omap),
                        "r"(d0), "r"(sg2 << K), "r"(sg1 << K), "r"(inst), "r"(src)
                        : "memory");
                else
                    asm volatile(
                        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&omap),
                        "r"(d0), "r"(sg2 << K), "r"(sg1 << K), "r"(inst), "r"(src)
                        : "memory");
#endif
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
#ifdef D3_PROF_PASS
            if constexpr (STAGE16) {
                PP_MARK(7);
                PP_ADD(0, 0, 1);
                PP_ADD(1, 1, 2);
                PP_ADD(2, 2, 3);
                PP_ADD(3, 3, 4);
                PP_ADD(4, 4, 5);
                PP_ADD(5, 5, 6);
                PP_ADD(6, 6, 7);
                if (pp_on) atomicAdd(&d3_pass_prof[7], 1ull);
            }
#endif
            return;
        }
    }

    // ---- store out(r1 = yb, r2, run yr)
    if (yact) {
        const int r1 = yb, e0 = yr * R;
        if (mosaic) {
#pragma unroll
            for (int r2 = 0; r2 < S; ++r2) {
                if constexpr (R % 2 == 0) {
                    if ((d0 % 2) == 0) {
                        uint32_t v[R];
#pragma unroll
                        for (int j = 0; j < R; ++j) v[j] = Lane<Acc>::bits(acc[r2][j]);
                        mosaic_run(mosaic_row(r1, r2), d0 + e0, v, R);
                        continue;
                    }
                }
#pragma unroll
                for (int j = 0; j < R; ++j) store_mosaic(r1, r2, e0 + j, acc[r2][j]);
            }
            return;
        }
        const bool vec_ok = (d0 + e0 + R <= p.out_width) && ((p.out_pitch * (int)sizeof(Out)) % 16 == 0) &&
                            (((d0 + e0) * (int)sizeof(Out)) % 16 == 0);
        Out *dst = row_ptr(r1) + e0;
#pragma unroll
        for (int r2 = 0; r2 < S; ++r2, dst += r2_stride) {
            if (vec_ok) {
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
#ifndef D3_DRT_ST256
#define D3_DRT_ST256 0
#endif
                    if constexpr (D3_DRT_ST256 && R == 8) {
                        // an 8-element run of a 32-byte-aligned row position: one STG.256
                        if ((reinterpret_cast<unsigned long long>(dst) & 31ull) == 0) {
                            uint32_t v[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) v[j] = Lane<Acc>::bits(acc[r2][j]);
                            if (FINAL) st_cs_v8(dst, v);
                            else st_v8(dst, v);
                            continue;
                        }
                    }
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
                for (int j = 0; j < R; ++j)
                    if (d0 + e0 + j < p.out_width) dst[j] = to_out<Out, Acc>(acc[r2][j]);
            }
        }
    }
#ifdef D3_PROF_PASS
    if constexpr (STAGE16 && FINAL) {
        PP_MARK(7);
        PP_ADD(0, 0, 1);    // staging issue
        PP_ADD(1, 1, 2);    // staging wait + barrier
        PP_ADD(2, 2, 3);    // x-step
        PP_ADD(3, 3, 4);    // barrier after x
        PP_ADD(4, 4, 5);    // write X + barrier
        PP_ADD(5, 5, 6);    // y-step
        PP_ADD(6, 6, 7);    // stores
        if (pp_on) atomicAdd(&d3_pass_prof[7], 1ull);
    }
#endif
}

}  // namespace d3
