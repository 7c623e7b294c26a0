// drt_first_swar.cuh -- first DRT pass for u8 voxels with two 16-bit lanes per
// 32-bit register (SWAR; the paper's "narrow integer" idea).
//
// The first pass (stages 0..K-1, K <= 4) of a u8 cube produces stage-K sums of
// at most 255 * 4^K <= 65280 voxels' worth, and its x-step sums (16 voxels)
// at most 4080: both fit a 16-bit lane, and a 32-bit add of two packed words
// never carries between lanes.  With the pass identity of drt_kernels.cuh
//
//   X(r1, w2)[e]  = sum_{w1} f(w1, w2)[e + l^K_{r1}(w1)]           (x-step)
//   out(r1, r2)[e] = sum_{w2} X(r1, w2)[e + l^K_{r2}(w2)]          (y-step)
//
// the x-step offsets do not depend on w2 and the y-step offsets do not depend
// on r1.  So the x-step runs on rows packed as (w2, w2 + S/2) and the y-step
// on X rows packed as (r1, r1 + S/2); one lane swap between the steps turns
// the first packing into the second.  Each add instruction thus serves two
// outputs, at the same tile shape as the 32-bit kernel.
#pragma once
#include "drt_kernels.cuh"

namespace d3 {

// E > 0 (the TMA-staged K = 4 kernel): a tile computes TE = T + E outputs per row but still owns the
// T stored positions [d0, d0 + T).  Rows are stored shifted left by rho <= 7, so with E = 8 every one
// of the tile's T / 8 stored chunks is whole (elements [d0 + rho, d0 + T + rho) are all computed
// here): the copy-out has no partial head / tail stores, which were 3 of its 7 store instructions
// per row on the L1 data pipe that limits this pass.  The extra run per row is taken by threads
// that were idle (x-step 88 of 96, y-step 72 of 96 at T = 64).
template <int K, int R, int T, int E = 0>
struct SwarGeom {
    static constexpr int S = 1 << K;
    static constexpr int H2 = S / 2;                      // lane pairing distance
    static constexpr int H = S - 1;
    static constexpr int TE = T + E;                      // outputs computed per row
    static constexpr int WIN = TE + 2 * H;
    static constexpr int NRX = (TE + H + R - 1) / R;
    static constexpr int NRY = TE / R;
    static constexpr int RD = (NRX - 1) * R + (R + H + 3) / 4 * 4;
    static constexpr int BWG = E > 0 ? 8 : 16;            // E > 0 keeps the slots small enough for 4 CTAs per SM
    static constexpr int BW = ((WIN > RD ? WIN : RD) + BWG - 1) / BWG * BWG;   // staged words per slot
    static constexpr int BWI = (BW + 15) / 16 * 16;       // brick extent along a contiguous z' (whole 16-byte vectors)
    static constexpr int XB = NRX * R * 4;
    static constexpr int SP0 = (BW * 4 > XB ? BW * 4 : XB);
    static constexpr int SP = SP0 + 16;                   // slot pitch (bytes); +16 rotates banks
    static constexpr int NSLOT = S * H2;                  // packed slots
    static constexpr int XT = H2 * NRX;                   // x-step tasks
    static constexpr int YT = H2 * NRY;                   // y-step tasks
    static constexpr int THREADS = ((XT > YT ? XT : YT) + 31) / 32 * 32;
    static constexpr int ORW = TE / 2;                    // output staging: words per row
    static constexpr int ORP = (ORW + 1) * 4;             // odd word pitch: rows hit distinct banks
    static constexpr int SMEM0 = NSLOT * SP;
    static constexpr int SMEM = (SMEM0 > S * S * ORP ? SMEM0 : S * S * ORP);
#ifndef SWAR_CTAS
#define SWAR_CTAS 4
#endif
#ifndef SWAR_CTAS3
#define SWAR_CTAS3 12                 // swept 4 / 8 / 12 / 16 on cfg2: 12 best (0.048 -> 0.044 ms)
#endif
    // target CTAs per SM (register cap): K = 4 (96 threads, 51 KB) 4; K = 3 (64 threads, 11 KB) SWAR_CTAS3
    static constexpr int CTAS = K == 4 ? SWAR_CTAS : SWAR_CTAS3;
    static constexpr int MAXREG0 = 65536 / (CTAS * THREADS) / 8 * 8;
    static constexpr int MAXREG = MAXREG0 > 255 ? 255 : MAXREG0;
    static_assert(T % R == 0 && E % R == 0 && (R == 8 || R == 4), "tile shape");
    static_assert(NRY == 8 || NRY == 16 || E > 0, "y runs per row must be a shuffle width");
    static_assert(S * S * BWI <= SMEM0, "the cube brick fits the slots");
};

// word = lo | hi << 16 for the four byte pairs (a.b_i, b.b_i): 6 PRMT per 4 words
__device__ __forceinline__ void pair_bytes(uint32_t a, uint32_t b, uint32_t (&w)[4]) {
    const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
    w[0] = __byte_perm(t0, 0u, 0x4140);
    w[1] = __byte_perm(t0, 0u, 0x4342);
    w[2] = __byte_perm(t1, 0u, 0x4140);
    w[3] = __byte_perm(t1, 0u, 0x4342);
}
__device__ __forceinline__ uint4 rev16(uint4 v) {
    return make_uint4(__byte_perm(v.w, 0, 0x0123), __byte_perm(v.z, 0, 0x0123), __byte_perm(v.y, 0, 0x0123),
                      __byte_perm(v.x, 0, 0x0123));
}

// -DD3_PROF_SWAR: per-phase clock accounting (thread 0 of each CTA) into d3_swar_prof[]
#ifdef D3_PROF_SWAR
__device__ unsigned long long d3_swar_prof[16];
#define SW_MARK(i) sw_t[i] = clock64()
#else
#define SW_MARK(i)
#endif

// Output staging rows (r1, r2) start row_skew(r1) words after their 33-word slot (rows are
// 33 words apart; 16 rows of one r1 = 528 = 16 mod 32 banks).  Two access patterns must both be
// conflict-free:
//   - the unpack stores: a warp writes 4 consecutive r1 x 8 runs (4 words apart) of one r2, so
//     the 4 skews must differ mod 4;
//   - the copy-out reads: a warp reads 32 rows, two 16-row blocks whose bank ranges must not
//     overlap.  The copy-out pairs r1 with r1 + 4 (copy_row below), so skew(r1 + 4) - skew(r1)
//     must be 16 mod 32.
// skew = (r1 & 3) + 16 ((r1 >> 2) & 1) satisfies both; + 32 (r1 >> 3) (0 mod 32) keeps rows from
// overlapping where the skew drops.
// (S = 8, the K = 3 first pass: skew r1 and the plain order.)
#ifdef D3_SWAR_NO_SKEW
template <int S> __device__ __forceinline__ int row_skew(int) { return 0; }
template <int S> __device__ __forceinline__ int copy_row(int i) { return i; }
#else
template <int S> __device__ __forceinline__ int row_skew(int r1) {
    if constexpr (S == 16) return (r1 & 3) + 16 * ((r1 >> 2) & 1) + 32 * (r1 >> 3);
    else return r1;
}
// copy-out order: each 32-row block of the loop = rows (a, r2) and (a + 4, r2), r2 = 0..15
template <int S> __device__ __forceinline__ int copy_row(int i) {
    if constexpr (S == 16) {
        const int blk = i >> 5, half = (i >> 4) & 1, r2 = i & 15;
        const int r1 = ((blk >> 2) << 3) + (blk & 3) + 4 * half;
        return (r1 << 4) | r2;
    } else {
        return i;
    }
}
#endif

#ifndef SWAR_FMA16
#define SWAR_FMA16 0                                      // all adds IADD3 (measured fastest)
#endif

// TMA staging of the cube brick (D3_SWAR_TMA_STAGE, K = 4, N >= 128).  The first pass is limited by
// the L1 data pipe, and a fifth of its wavefronts were the scattered 16-byte cube loads (every lane
// a different line).  Instead one TMA tensor load brings the tile's 16 x 16 x BW voxel brick of the
// ORIGINAL cube into shared memory (zero-filled outside the cube), the threads read it into
// registers with LDS.128 and, after a barrier, pack over it.  Three maps of cube[batch][x][y][z],
// one per original axis a that z' runs along: a = 2 (z' along z): box {BW, 16, 16} over (z, y, x);
// a = 0 / 1: box {16, 16, BW} over (z, y, x) / (z, x, y), i.e. the BW-long side outermost, so the
// 16-byte vectors of one z' are contiguous.
// Chunk index of item (r, lane step d) on the packing diagonal: r's 8-chunk group is kept and only the
// position inside it rotates, so the 8 lanes of a quarter-warp write 8 distinct bank groups whether
// or not xswz flips that group's low bit.  (NE4 not a multiple of 8: plain rotation.)
#ifndef D3_SWAR_DIAG8
#define D3_SWAR_DIAG8 1
#endif
template <int NE4> __device__ __forceinline__ int diag_chunk(int r, int d) {
    if constexpr (D3_SWAR_DIAG8 && NE4 % 8 == 0) return (r & ~7) | ((r + d) & 7);
    else return (r + d) % NE4;
}

struct SwarCubeMaps {
    CUtensorMap m[3];
    CUtensorMap st;       // the stage-K rows this pass writes (D3_SWAR_TMA_OUT, the copy-out)
};
#ifndef D3_SWAR_TMA_STAGE
#define D3_SWAR_TMA_STAGE 1
#endif

template <int K, int R, int T, int E = 0>
__global__ void __launch_bounds__(SwarGeom<K, R, T, E>::THREADS) __maxnreg__((SwarGeom<K, R, T, E>::MAXREG))
drt_first_swar_kernel(const DrtPass p, const __grid_constant__ CUtensorMap zmap, const __grid_constant__ SwarCubeMaps cmap,
                      const int tma_in, const int tma_out) {
    using G = SwarGeom<K, R, T, E>;
    constexpr int S = G::S, H2 = G::H2, SP = G::SP, BW = G::BW;
    static_assert(E == 0 || (K == 4 && E == 8), "E = 8: the TMA-staged K = 4 kernel");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;

    const int tid = threadIdx.x;
    const int tile = blockIdx.x, g = blockIdx.y, li = blockIdx.z;
    const int inst = p.inst0 + li;
    const int m = p.m;                                    // c = 0: the group is (V1, V2) only
#ifndef D3_PDL
#define D3_PDL 1
#endif
    // the dependent final pass may be scheduled from now on (it waits for this grid's completion
    // before reading the stage buffer: griddepcontrol.wait in drt_pass_kernel)
    if (D3_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int V2 = g & ((1 << m) - 1);
    const int V1 = (g >> m) & ((1 << m) - 1);
    const int d0 = tile * T;
    const int Dabs = p.out_base + d0;
    const int N = p.N;

#ifdef D3_PROF_SWAR
    long long sw_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    SW_MARK(0);
    auto put4 = [&](int slot, int chunk, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
        *reinterpret_cast<uint4 *>(sm + slot * SP + 16 * xswz(chunk)) = make_uint4(a, b, c, d);
    };

    // ---- stage packed rows: slot (w1, pw), word e = f(w1, pw)[e] | f(w1, pw + H2)[e] << 16,
    // f(w1, w2)[e] = oriented voxel (xb + w1, yb + w2, z0 + e), 0 outside the cube.
    {
        const Orient o = p.ori[inst % p.ndod];
        const uint8_t *cube = reinterpret_cast<const uint8_t *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
        const int z0 = Dabs - 2 * N;                      // stage 0: D = z' + 2N
        const int xb = V1 << K, yb = V2 << K;
        auto vox = [&](int x, int y, int z) -> const uint8_t * {
            return cube + o.off0 + (long long)x * o.sx + (long long)y * o.sy + (long long)z * o.sz;
        };
        if (E > 0 && !(tma_in && (z0 & 15) == 0 && (o.fast != 2 || o.sz == 1))) __trap();   // host: E > 0 only with the brick load
        if (K == 4 && D3_SWAR_TMA_STAGE && tma_in && (z0 & 15) == 0 && (o.fast != 2 || o.sz == 1)) {
            if constexpr (K == 4) {
            // ---- brick by TMA, packed from shared memory (see SwarCubeMaps)
            uint64_t *bar = reinterpret_cast<uint64_t *>(sm + G::SMEM);
            const long long sv[3] = {o.sx, o.sy, o.sz};
            const int lo[3] = {xb, yb, z0}, ext[3] = {S, S, BW};
            int aj[3], start[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const long long a = sv[j] < 0 ? -sv[j] : sv[j];
                aj[j] = a == 1 ? 2 : (a == (long long)N ? 1 : 0);       // original axis of oriented axis j
            }
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if (aj[j] == a) start[a] = sv[j] > 0 ? lo[j] : N - lo[j] - ext[j];
            // dense brick, byte multiplier of each oriented axis (see SwarCubeMaps)
            const int kind = aj[2], other = 1 - kind;         // kind != 2: the 16-long non-inner original axis
            int ss[3], soff = 0;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int mm = kind == 2 ? (aj[j] == 2 ? 1 : (aj[j] == 1 ? G::BWI : S * G::BWI))
                                         : (aj[j] == 2 ? 1 : (j == 2 ? S * S : S));
                ss[j] = sv[j] > 0 ? mm : -mm;
                if (sv[j] < 0) soff += (ext[j] - 1) * mm;
            }
            const int c1 = kind == 2 ? start[1] : (other == 1 ? start[1] : start[0]);
            const int c2 = kind == 2 ? start[0] : start[kind == 0 ? 0 : 1];
            const uint32_t smb = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
            const uint32_t barb = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
            if (tid == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(barb), "r"(1) : "memory");
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(barb), "r"(S * S * (kind == 2 ? G::BWI : BW)) : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smb),
                    "l"(&cmap.m[kind]), "r"(start[2]), "r"(c1), "r"(c2), "r"(inst / p.ndod), "r"(barb)
                    : "memory");
            }
#ifndef D3_SWAR_ONE_WAITER
#define D3_SWAR_ONE_WAITER 0
#endif
            if (D3_SWAR_ONE_WAITER) {
                // thread 0 alone waits for the brick, the CTA barrier then orders everyone after it
                if (tid == 0)
                    asm volatile(
                        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(barb)
                        : "memory");
                __syncthreads();
            } else {
            __syncthreads();                                  // the barrier is initialised
            asm volatile(
                "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(barb)
                : "memory");
            }
            // 16-byte vector at brick offset `off` (a multiple of 16)
            auto lds16 = [&](int off) -> uint4 {
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(smb + (uint32_t)off));
                return v;
            };
            // Lane orders below keep a quarter-warp's 8 brick vectors AND its 8 packed chunks in
            // distinct 16-byte bank groups: the brick group depends on the 16-long axis index, the
            // packed group on (pw + chunk) mod 8 (slots are 25 chunks apart), hence the diagonals.
            if (o.fast == 2) {
                // z' contiguous: rows pw and pw + 8 of slot (w1, pw), 16 voxels = 4 packed chunks.
                // When x' runs along the brick's outer side (y), w1 advances with pw (rows 96 bytes apart)
                constexpr int NQ = G::BWI / 16, NIT = (G::NSLOT * NQ + G::THREADS - 1) / G::THREADS;
                const bool diag = (ss[0] < 0 ? -ss[0] : ss[0]) < (ss[1] < 0 ? -ss[1] : ss[1]);
                uint4 a[NIT], b[NIT];
#pragma unroll
                for (int u = 0; u < NIT; ++u) {
                    const int it = tid + u * G::THREADS;
                    const int sl = it & (G::NSLOT - 1), q = it / G::NSLOT;
                    const int pw = sl & (H2 - 1), w1 = ((sl / H2) + (diag ? pw : 0)) & (S - 1);
                    a[u] = make_uint4(0u, 0u, 0u, 0u);
                    b[u] = a[u];
                    if (it < G::NSLOT * NQ) {
                        const int off = soff + w1 * ss[0] + pw * ss[1] + 16 * q;
                        a[u] = lds16(off);
                        b[u] = lds16(off + H2 * ss[1]);
                    }
                }
                __syncthreads();                              // the brick is in registers: pack over it
#pragma unroll
                for (int u = 0; u < NIT; ++u) {
                    const int it = tid + u * G::THREADS;
                    if (it < G::NSLOT * NQ) {
                        const int sl = it & (G::NSLOT - 1), q = it / G::NSLOT;
                        const int pw = sl & (H2 - 1), w1 = ((sl / H2) + (diag ? pw : 0)) & (S - 1);
                        const uint32_t av[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, bv[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            uint32_t w[4];
                            pair_bytes(av[h], bv[h], w);
                            if (G::BWI == BW || 4 * q + h < BW / 4) put4(w1 * H2 + pw, 4 * q + h, w[0], w[1], w[2], w[3]);
                        }
                    }
                }
            } else if (o.fast == 1) {
                // y' contiguous: one vector = all 16 w2 of (w1, z'); item (w1, e4) = 4 consecutive z',
                // lanes along w1 with e4 on the diagonal
                const bool fwd = ss[1] > 0;
                const int yoff = soff + (fwd ? 0 : 15 * ss[1]);
                constexpr int NE4 = BW / 4, NI = (S * NE4 + G::THREADS - 1) / G::THREADS;
                uint4 v[NI][4];
#pragma unroll
                for (int u = 0; u < NI; ++u) {
                    const int it = tid + u * G::THREADS;
                    const int w1 = it & (S - 1), e4 = diag_chunk<NE4>(it / S, w1);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        v[u][t] = make_uint4(0u, 0u, 0u, 0u);
                        if (it < S * NE4) v[u][t] = lds16(yoff + w1 * ss[0] + (4 * e4 + t) * ss[2]);
                    }
                }
                __syncthreads();
#pragma unroll
                for (int u = 0; u < NI; ++u) {
                    const int it = tid + u * G::THREADS;
                    if (it >= S * NE4) break;
                    const int w1 = it & (S - 1), e4 = diag_chunk<NE4>(it / S, w1);
                    uint32_t wd[4][H2];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint4 x = fwd ? v[u][t] : rev16(v[u][t]);   // byte b <-> w2 = b
                        uint32_t l4[4], h4[4];
                        pair_bytes(x.x, x.z, l4);          // w2 = 0..3 with 8..11
                        pair_bytes(x.y, x.w, h4);          // w2 = 4..7 with 12..15
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            wd[t][j] = l4[j];
                            wd[t][4 + j] = h4[j];
                        }
                    }
#pragma unroll
                    for (int pw = 0; pw < H2; ++pw) put4(w1 * H2 + pw, e4, wd[0][pw], wd[1][pw], wd[2][pw], wd[3][pw]);
                }
            } else {
                // x' contiguous: one vector = all 16 w1 of (w2, z'); item (pw, e4): rows pw and pw + 8,
                // lanes along pw with e4 on the diagonal (step 2: (pw + chunk) mod 8 = 3 pw + const, diag_chunk)
                const bool fwd = ss[0] > 0;
                const int xoff = soff + (fwd ? 0 : 15 * ss[0]);
                constexpr int NE4 = BW / 4, NI = (H2 * NE4 + G::THREADS - 1) / G::THREADS;
                uint4 a[NI][4], b[NI][4];
#pragma unroll
                for (int u = 0; u < NI; ++u) {
                    const int it = tid + u * G::THREADS;
                    const int pw = it & (H2 - 1), e4 = diag_chunk<NE4>(it / H2, 2 * pw);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        a[u][t] = make_uint4(0u, 0u, 0u, 0u);
                        b[u][t] = a[u][t];
                        if (it < H2 * NE4) {
                            const int off = xoff + pw * ss[1] + (4 * e4 + t) * ss[2];
                            a[u][t] = lds16(off);
                            b[u][t] = lds16(off + H2 * ss[1]);
                        }
                    }
                }
                __syncthreads();
#pragma unroll
                for (int u = 0; u < NI; ++u) {
                    const int it = tid + u * G::THREADS;
                    if (it >= H2 * NE4) break;
                    const int pw = it & (H2 - 1), e4 = diag_chunk<NE4>(it / H2, 2 * pw);
                    uint32_t wd[4][S];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint4 xa = fwd ? a[u][t] : rev16(a[u][t]), xb4 = fwd ? b[u][t] : rev16(b[u][t]);
                        const uint32_t av[4] = {xa.x, xa.y, xa.z, xa.w}, bv[4] = {xb4.x, xb4.y, xb4.z, xb4.w};
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            uint32_t w[4];
                            pair_bytes(av[h], bv[h], w);
#pragma unroll
                            for (int j = 0; j < 4; ++j) wd[t][4 * h + j] = w[j];
                        }
                    }
#pragma unroll
                    for (int w1 = 0; w1 < S; ++w1) put4(w1 * H2 + pw, e4, wd[0][w1], wd[1][w1], wd[2][w1], wd[3][w1]);
                }
            }
            }
        } else if (K == 4 && p.vec_ok && o.fast == 2 && (z0 & 15) == 0) {
            // z' contiguous (forward): two LDG.128 (rows pw, pw + 8) -> 16 packed words.  Item
            // it = slot + NSLOT * q (consecutive lanes: consecutive slots, conflict-free STS); all of
            // a thread's loads are issued before any is consumed so their L2 latencies overlap.
            constexpr int NQ = BW / 16, NIT = (G::NSLOT * NQ + G::THREADS - 1) / G::THREADS;
            static_assert((G::NSLOT & (G::NSLOT - 1)) == 0, "slot count");
            const uint8_t *vb = vox(xb, yb, z0);
            uint4 a[NIT], b[NIT];
#pragma unroll
            for (int u = 0; u < NIT; ++u) {
                const int it = tid + u * G::THREADS;
                const int slot = it & (G::NSLOT - 1), q = it / G::NSLOT;
                const int w1 = slot / H2, pw = slot & (H2 - 1);
                const uint8_t *ra = vb + (long long)w1 * o.sx + (long long)pw * o.sy + 16 * q;
                a[u] = make_uint4(0u, 0u, 0u, 0u);
                b[u] = a[u];
                if (it < G::NSLOT * NQ && (unsigned)(z0 + 16 * q) < (unsigned)N) {
                    a[u] = __ldg(reinterpret_cast<const uint4 *>(ra));
                    b[u] = __ldg(reinterpret_cast<const uint4 *>(ra + (long long)H2 * o.sy));
                }
            }
#pragma unroll
            for (int u = 0; u < NIT; ++u) {
                const int it = tid + u * G::THREADS;
                if (it < G::NSLOT * NQ) {
                    const int slot = it & (G::NSLOT - 1), q = it / G::NSLOT;
                    const uint32_t av[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, bv[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        uint32_t w[4];
                        pair_bytes(av[h], bv[h], w);
                        put4(slot, 4 * q + h, w[0], w[1], w[2], w[3]);
                    }
                }
            }
        } else if (K == 4 && p.vec_ok && o.fast == 1) {
            // y' contiguous: one LDG.128 along y' = all 16 w2 of (w1, z'); 4 consecutive z' per item
            const bool fwd = o.sy > 0;
            const uint8_t *vb = vox(xb, yb + (fwd ? 0 : 15), z0);
            constexpr int NE4 = BW / 4, IT = 2;
            for (int base = tid; base < S * NE4; base += IT * blockDim.x) {
                uint4 v[IT][4];
#pragma unroll
                for (int u = 0; u < IT; ++u) {
                    const int it = base + u * blockDim.x;
                    const int w1 = it / NE4, e4 = it - w1 * NE4;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int z = z0 + 4 * e4 + t;
                        v[u][t] = make_uint4(0u, 0u, 0u, 0u);
                        if (it < S * NE4 && (unsigned)z < (unsigned)N)
                            v[u][t] = __ldg(reinterpret_cast<const uint4 *>(vb + (long long)w1 * o.sx + (long long)(4 * e4 + t) * o.sz));
                    }
                }
#pragma unroll
                for (int u = 0; u < IT; ++u) {
                    const int it = base + u * blockDim.x;
                    if (it >= S * NE4) break;
                    const int w1 = it / NE4, e4 = it - w1 * NE4;
                    uint32_t wd[4][H2];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint4 x = fwd ? v[u][t] : rev16(v[u][t]);   // byte b <-> w2 = b
                        uint32_t lo[4], hi[4];
                        pair_bytes(x.x, x.z, lo);          // w2 = 0..3 with 8..11
                        pair_bytes(x.y, x.w, hi);          // w2 = 4..7 with 12..15
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            wd[t][j] = lo[j];
                            wd[t][4 + j] = hi[j];
                        }
                    }
#pragma unroll
                    for (int pw = 0; pw < H2; ++pw) put4(w1 * H2 + pw, e4, wd[0][pw], wd[1][pw], wd[2][pw], wd[3][pw]);
                }
            }
        } else if (K == 4 && p.vec_ok && o.fast == 0) {
            // x' contiguous: LDG.128 along x' = all 16 w1 of (w2, z'); rows pw and pw + 8
            const bool fwd = o.sx > 0;
            const uint8_t *vb = vox(xb + (fwd ? 0 : 15), yb, z0);
            constexpr int NE4 = BW / 4;
            for (int it = tid; it < H2 * NE4; it += blockDim.x) {
                const int pw = it / NE4, e4 = it - pw * NE4;
                uint32_t wd[4][S];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int z = z0 + 4 * e4 + t;
                    uint4 a = make_uint4(0u, 0u, 0u, 0u), b = a;
                    if ((unsigned)z < (unsigned)N) {
                        const uint8_t *ra = vb + (long long)pw * o.sy + (long long)(4 * e4 + t) * o.sz;
                        a = __ldg(reinterpret_cast<const uint4 *>(ra));
                        b = __ldg(reinterpret_cast<const uint4 *>(ra + (long long)H2 * o.sy));
                    }
                    if (!fwd) {
                        a = rev16(a);
                        b = rev16(b);
                    }
                    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        uint32_t w[4];
                        pair_bytes(av[h], bv[h], w);
#pragma unroll
                        for (int j = 0; j < 4; ++j) wd[t][4 * h + j] = w[j];
                    }
                }
#pragma unroll
                for (int w1 = 0; w1 < S; ++w1) put4(w1 * H2 + pw, e4, wd[0][w1], wd[1][w1], wd[2][w1], wd[3][w1]);
            }
        } else {
            // generic (small N, any orientation): word by word
            for (int it = tid; it < G::NSLOT * BW; it += blockDim.x) {
                const int slot = it / BW, e = it - slot * BW;
                const int w1 = slot / H2, pw = slot - w1 * H2, z = z0 + e;
                uint32_t bits = 0;
                if ((unsigned)z < (unsigned)N)
                    bits = (uint32_t)__ldg(vox(xb + w1, yb + pw, z)) | ((uint32_t)__ldg(vox(xb + w1, yb + pw + H2, z)) << 16);
                *reinterpret_cast<uint32_t *>(sm + slot * SP + 16 * xswz(e >> 2) + 4 * (e & 3)) = bits;
            }
        }
    }
    __syncthreads();
    SW_MARK(1);

    // ---- x-step on (w2, w2 + H2) pairs, then y-step on (r1, r1 + H2) pairs; one code path.
    //   step 0: thread (pw, run)  -> acc[r1][j] = (X(r1, pw), X(r1, pw + H2))
    //   step 1: thread (q, run)   -> acc[r2][j] = (out(q, r2), out(q + H2, r2))
    uint32_t acc[S][R];
#pragma unroll 1
    for (int step = 0; step < 2; ++step) {
        int grp, run;
        task_row_run(tid, step ? G::NRY : G::NRX, H2, grp, run, true);
        const bool act = tid < (step ? G::YT : G::XT);
        if (act) {
#pragma unroll
            for (int i = 0; i < S; ++i)
#pragma unroll
                for (int j = 0; j < R; ++j) acc[i][j] = 0u;
            drt_accumulate<K, R, SP, false, uint32_t, SWAR_FMA16>(sm, step ? grp * S : grp, step ? 1 : H2, run * (R / 4),
                                                             p.one, acc);
        }
#ifdef D3_PROF_SWAR
        if (step == 0) SW_MARK(2); else SW_MARK(4);
#endif
#ifndef D3_SWAR_DIRECT
#define D3_SWAR_DIRECT 0                 // measured: first pass 0.691 ms vs 0.451 with the unpack + copy-out
#endif
        if constexpr (D3_SWAR_DIRECT && G::NRY == 8 && R == 8) {
            if (step == 1) {
                // y-step results straight to the stage-K rows (no unpack / copy-out round trip through
                // shared memory): rows (grp, r2) and (grp + H2, r2), run `run` (8 elements = one
                // 16-byte chunk), stored pre-shifted by rho (common.cuh) after a one-lane shuffle with
                // the next run; the 8 runs of a row are 8 consecutive lanes, all lanes of a warp active
                static_assert(G::YT % 32 == 0, "y-step tasks fill whole warps");
                if (act) {
                    uint16_t *outp = reinterpret_cast<uint16_t *>(p.out);
                    const long long out_inst = (long long)li * p.out_inst_stride;
                    const int mK = (1 << p.next_k) - 1;
                    const int wv1 = V1 & mK, wv2 = V2 & mK;
                    const int e0 = run * R;
#pragma unroll
                    for (int r2 = 0; r2 < S; ++r2) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t sel = h ? 0x7632u : 0x5410u;
                            const int r1 = grp + h * H2;
                            uint32_t win[8];
#pragma unroll
                            for (int i = 0; i < 4; ++i) win[i] = __byte_perm(acc[r2][2 * i], acc[r2][2 * i + 1], sel);
#pragma unroll
                            for (int i = 0; i < 4; ++i) win[4 + i] = __shfl_down_sync(0xffffffffu, win[i], 1, 8);
                            const int rho = (r1 * wv1 + r2 * wv2) & 7;
                            const long long row = ((((long long)r1 << K) + r2) << (2 * m)) + ((long long)V1 << m) + V2;
                            uint16_t *dst = outp + out_inst + row * p.out_pitch + d0 + e0;
                            uint32_t v[4];
                            window_chunk<2>(win, rho, 0, v);
                            if (d0 + e0 < p.out_width) {
                                if (run == G::NRY - 1) store_chunk_head<2>(dst, v, 8 - rho);
                                else *reinterpret_cast<uint4 *>(dst) = make_uint4(v[0], v[1], v[2], v[3]);
                            }
                            if (run == 0 && rho > 0 && d0 >= 8) {
                                // tile elements [0, rho) end the previous chunk (whose head the previous tile wrote)
                                uint32_t tw[8] = {0u, 0u, 0u, 0u, win[0], win[1], win[2], win[3]};
                                window_chunk<2>(tw, rho, 0, v);
                                store_chunk_tail<2>(dst - 8, v, rho);
                            }
                        }
                    }
                }
#ifdef D3_PROF_SWAR
                SW_MARK(5);
                SW_MARK(6);
                if (tid == 0) {
                    for (int i = 0; i < 6; ++i) atomicAdd(&d3_swar_prof[i], (unsigned long long)(sw_t[i + 1] - sw_t[i]));
                    atomicAdd(&d3_swar_prof[7], 1ull);
                }
#endif
                return;
            }
        }
        __syncthreads();
        if (act) {
            if (step == 0) {
                // lane swap: X slot (q, w2) = (X(q, w2), X(q + H2, w2)), written in place
#pragma unroll
                for (int q = 0; q < H2; ++q) {
#pragma unroll
                    for (int c = 0; c < R / 4; ++c) {
                        uint32_t lo[4], hi[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            lo[j] = __byte_perm(acc[q][4 * c + j], acc[q + H2][4 * c + j], 0x5410);
                            hi[j] = __byte_perm(acc[q][4 * c + j], acc[q + H2][4 * c + j], 0x7632);
                        }
                        put4(q * S + grp, run * (R / 4) + c, lo[0], lo[1], lo[2], lo[3]);
                        put4(q * S + grp + H2, run * (R / 4) + c, hi[0], hi[1], hi[2], hi[3]);
                    }
                }
            } else {
                // unpack to u16 output rows in SMEM: row (r1, r2) at ORP * (r1 * S + r2)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t sel = h ? 0x7632u : 0x5410u;
#pragma unroll
                    for (int r2 = 0; r2 < S; ++r2) {
                        uint32_t *o = reinterpret_cast<uint32_t *>(sm + G::ORP * ((grp + h * H2) * S + r2)) +
                                      row_skew<S>(grp + h * H2) + (R / 2) * run;
#pragma unroll
                        for (int i = 0; i < R / 2; ++i) o[i] = __byte_perm(acc[r2][2 * i], acc[r2][2 * i + 1], sel);
                    }
                }
            }
        }
        __syncthreads();
#ifdef D3_PROF_SWAR
        if (step == 0) SW_MARK(3); else SW_MARK(5);
#endif
    }

    // ---- copy-out, one row per thread: stage-K rows stored pre-shifted by rho (common.cuh).
    // Stored chunk k of the tile (elements d0 + 8k .. + 7) holds tile elements [8k + rho, 8k + rho + 8);
    // the last one is a head store when rho > 0, and the chunk before the tile gets a tail store of
    // tile elements [0, rho) (its head belongs to the previous tile).
    uint16_t *outp = reinterpret_cast<uint16_t *>(p.out);
    const long long out_inst = (long long)li * p.out_inst_stride;
#ifdef D3_STAGE_EVICT_LAST
    const uint64_t keep_pol = l2_evict_last();
#endif
    const int mK = (1 << p.next_k) - 1;
    const int wv1 = V1 & mK, wv2 = V2 & mK;
    constexpr int NCK = T / 8;
#ifndef D3_SWAR_COPY_CHUNK
#define D3_SWAR_COPY_CHUNK 0              // measured: first pass 0.4575 ms vs 0.4514 with one row per thread
#endif
#if D3_SWAR_COPY_CHUNK
    static_assert(E == 0, "chunk copy-out: E = 0 only");
    // one 16-byte chunk per item, 8 consecutive lanes per row: every store instruction of a warp
    // writes 4 whole 128-byte row segments; a lane reads its chunk's 5 words at the rho/2 word offset
    // (no select network) and the k = 0 lane also writes the tail chunk before the tile
    for (int it = tid; it < S * S * NCK; it += blockDim.x) {
        const int rr = it / NCK, k = it - rr * NCK;
        const int r1 = rr >> K, r2 = rr & (S - 1);
        const int rho = (r1 * wv1 + r2 * wv2) & 7;
        const long long row = ((((long long)r1 << K) + r2) << (2 * m)) + ((long long)V1 << m) + V2;
        uint16_t *dst = outp + out_inst + row * p.out_pitch + d0 + 8 * k;
        const uint32_t *srow = reinterpret_cast<const uint32_t *>(sm + G::ORP * rr) + row_skew<S>(r1);
        static_assert(G::SMEM0 >= S * S * G::ORP + 4 * 51 + 12, "skewed rows + chunk overrun");
        if (d0 + 8 * k < p.out_width) {
            const int w0 = 4 * k + (rho >> 1);
            uint32_t w[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) w[i] = srow[w0 + i];     // up to 3 words past the row: staging area
            const uint32_t sel = (rho & 1) ? 0x5432u : 0x3210u;
            uint32_t v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = __byte_perm(w[i], w[i + 1], sel);
            if (k == NCK - 1) store_chunk_head<2>(dst, v, 8 - rho);
#ifdef D3_STAGE_EVICT_LAST
            else st_hint_v4(dst, v[0], v[1], v[2], v[3], keep_pol);
#else
            else *reinterpret_cast<uint4 *>(dst) = make_uint4(v[0], v[1], v[2], v[3]);
#endif
        }
        if (k == 0 && rho > 0 && d0 >= 8) {
            // tile elements [0, rho) end the previous chunk: window (zeros, row words 0..3)
            uint32_t tw[8] = {0u, 0u, 0u, 0u, srow[0], srow[1], srow[2], srow[3]}, v[4];
            window_chunk<2>(tw, rho, 0, v);
            store_chunk_tail<2>(dst - 8, v, rho);
        }
    }
#else
#ifndef D3_SWAR_TMA_OUT
#define D3_SWAR_TMA_OUT 0     // measured (bit-exact): cfg3 first pass 0.365 ms vs 0.331 with the LSU copy-out
#endif
#ifndef D3_SWAR_TMA_OUT_FULLWAIT
#define D3_SWAR_TMA_OUT_FULLWAIT 1
#endif
    if constexpr (E > 0) {
        // every stored chunk of the tile is whole (SwarGeom): 32-byte stores, no head / tail
        static_assert(E == 8 && NCK % 2 == 0, "E covers the largest shift");
        const bool al32 = (p.out_pitch % 16 == 0) && (p.out_inst_stride % 16 == 0) &&
                          ((reinterpret_cast<unsigned long long>(outp) & 31ull) == 0);
        for (int ii = tid; ii < S * S; ii += blockDim.x) {
            const int rr = copy_row<S>(ii);
            const int r1 = rr >> K, r2 = rr & (S - 1);
            const int rho = (r1 * wv1 + r2 * wv2) & 7;
            const long long row = ((((long long)r1 << K) + r2) << (2 * m)) + ((long long)V1 << m) + V2;
            uint16_t *dst = outp + out_inst + row * p.out_pitch + d0;
            const uint32_t sel = (rho & 1) ? 0x5432u : 0x3210u;
            const uint32_t *srow = reinterpret_cast<const uint32_t *>(sm + G::ORP * rr) + row_skew<S>(r1);
            static_assert(G::ORW >= 4 * NCK + 4, "the row holds the shifted window");
            uint32_t w0[4 * NCK + 4], w[4 * NCK + 1];
#pragma unroll
            for (int i = 0; i < 4 * NCK + 4; ++i) w0[i] = srow[i];
            const int q = rho >> 1;
            const bool b0 = q & 1, b1 = (q & 2) != 0;
#pragma unroll
            for (int i = 0; i < 4 * NCK + 3; ++i) w0[i] = b0 ? w0[i + 1] : w0[i];
#pragma unroll
            for (int i = 0; i < 4 * NCK + 1; ++i) w[i] = b1 ? w0[i + 2] : w0[i];
#pragma unroll
            for (int k = 0; k < NCK; k += 2) {
                uint32_t v8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) v8[i] = __byte_perm(w[4 * k + i], w[4 * k + i + 1], sel);
                if (al32 && d0 + 8 * (k + 1) < p.out_width) {
                    st_v8(dst + 8 * k, v8);
                } else {
                    if (d0 + 8 * k < p.out_width) *reinterpret_cast<uint4 *>(dst + 8 * k) = make_uint4(v8[0], v8[1], v8[2], v8[3]);
                    if (d0 + 8 * (k + 1) < p.out_width)
                        *reinterpret_cast<uint4 *>(dst + 8 * (k + 1)) = make_uint4(v8[4], v8[5], v8[6], v8[7]);
                }
            }
        }
    } else if (K == 4 && D3_SWAR_TMA_OUT && tma_out) {
        // Chunks 0 .. NCK - 2 of every row (whole for any rho) leave with ONE TMA tensor store of a
        // dense 256-row image (smap: stage rows as [inst][r1 r2][V1 V2][D], box {8 (NCK - 1), 1, 256, 1});
        // only the last chunk (head) and the tail before the tile stay on the LSU (the L1 data pipe
        // is this pass's limiter).  The image is written over the unpacked rows, so every thread first
        // reads and shifts its rows into registers.
        constexpr int NRW = (S * S + G::THREADS - 1) / G::THREADS, IMGP = (NCK - 1) * 16;
        uint32_t w[NRW][4 * NCK + 1], tw4[NRW][4];
#pragma unroll
        for (int u = 0; u < NRW; ++u) {
            const int ii = tid + u * G::THREADS;
            if (ii < S * S) {
                const int rr = copy_row<S>(ii), r1 = rr >> K, r2 = rr & (S - 1);
                const int rho = (r1 * wv1 + r2 * wv2) & 7;
                const uint32_t *srow = reinterpret_cast<const uint32_t *>(sm + G::ORP * rr) + row_skew<S>(r1);
                uint32_t w0[4 * NCK + 4];
#pragma unroll
                for (int i = 0; i < 4 * NCK + 4; ++i) w0[i] = srow[i];
#pragma unroll
                for (int i = 0; i < 4; ++i) tw4[u][i] = w0[i];
                const int q = rho >> 1;
                const bool b0 = q & 1, b1 = (q & 2) != 0;
#pragma unroll
                for (int i = 0; i < 4 * NCK + 3; ++i) w0[i] = b0 ? w0[i + 1] : w0[i];
#pragma unroll
                for (int i = 0; i < 4 * NCK + 1; ++i) w[u][i] = b1 ? w0[i + 2] : w0[i];
            }
        }
        __syncthreads();                                      // every unpacked row is in registers
#pragma unroll
        for (int u = 0; u < NRW; ++u) {
            const int ii = tid + u * G::THREADS;
            if (ii < S * S) {
                const int rr = copy_row<S>(ii), r1 = rr >> K, r2 = rr & (S - 1);
                const int rho = (r1 * wv1 + r2 * wv2) & 7;
                const uint32_t sel = (rho & 1) ? 0x5432u : 0x3210u;
#pragma unroll
                for (int k = 0; k < NCK - 1; ++k)
                    *reinterpret_cast<uint4 *>(sm + rr * IMGP + 16 * k) =
                        make_uint4(__byte_perm(w[u][4 * k], w[u][4 * k + 1], sel), __byte_perm(w[u][4 * k + 1], w[u][4 * k + 2], sel),
                                   __byte_perm(w[u][4 * k + 2], w[u][4 * k + 3], sel), __byte_perm(w[u][4 * k + 3], w[u][4 * k + 4], sel));
                const long long row = ((((long long)r1 << K) + r2) << (2 * m)) + ((long long)V1 << m) + V2;
                uint16_t *dst = outp + out_inst + row * p.out_pitch + d0;
                if (d0 + 8 * (NCK - 1) < p.out_width) {
                    constexpr int k = NCK - 1;
                    uint32_t v[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) v[i] = __byte_perm(w[u][4 * k + i], w[u][4 * k + i + 1], sel);
                    store_chunk_head<2>(dst + 8 * k, v, 8 - rho);
                }
                if (rho > 0 && d0 >= 8) {
                    const uint32_t tw[8] = {0u, 0u, 0u, 0u, tw4[u][0], tw4[u][1], tw4[u][2], tw4[u][3]};
                    uint32_t v[4];
                    window_chunk<2>(tw, rho, 0, v);
                    store_chunk_tail<2>(dst - 8, v, rho);
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0 && d0 < p.out_width) {
            asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&cmap.st),
                         "r"(d0), "r"((V1 << m) + V2), "r"(0), "r"(li), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(sm)))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (D3_SWAR_TMA_OUT_FULLWAIT) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    } else
    for (int ii = tid; ii < S * S; ii += blockDim.x) {
        const int rr = copy_row<S>(ii);
        const int r1 = rr >> K, r2 = rr & (S - 1);
        const int rho = (r1 * wv1 + r2 * wv2) & 7;
        const long long row = ((((long long)r1 << K) + r2) << (2 * m)) + ((long long)V1 << m) + V2;
        uint16_t *dst = outp + out_inst + row * p.out_pitch + d0;
        const uint32_t sel = (rho & 1) ? 0x5432u : 0x3210u;
        uint32_t w[4 * NCK + 1];                          // the row's words from rho/2, loaded before any store
        {
            // every lane reads its row from word 0 (odd row pitch: conflict-free), the rho/2 word
            // offset is applied with selects (overruns the row by 3 words: inside the staging area)
            const uint32_t *srow = reinterpret_cast<const uint32_t *>(sm + G::ORP * rr) + row_skew<S>(r1);
            static_assert(G::SMEM0 >= S * S * G::ORP + 4 * 51 + 12, "skewed rows + copy-out overrun");
            uint32_t w0[4 * NCK + 4];
#pragma unroll
            for (int i = 0; i < 4 * NCK + 4; ++i) w0[i] = srow[i];
            const int q = rho >> 1;
#ifndef D3_SWAR_SEL4
            // barrel shift by q = rho/2 words: by 1 if bit 0, then by 2 if bit 1 (2 selects per
            // word instead of sel4's 3)
            const bool b0 = q & 1, b1 = (q & 2) != 0;
#pragma unroll
            for (int i = 0; i < 4 * NCK + 3; ++i) w0[i] = b0 ? w0[i + 1] : w0[i];
#pragma unroll
            for (int i = 0; i < 4 * NCK + 1; ++i) w[i] = b1 ? w0[i + 2] : w0[i];
#else
#pragma unroll
            for (int i = 0; i < 4 * NCK + 1; ++i) {
                const uint32_t c4[4] = {w0[i], w0[i + 1], w0[i + 2], w0[i + 3]};
                w[i] = sel4(c4, q);
            }
#endif
        }
#ifndef D3_SWAR_ST256
#define D3_SWAR_ST256 1      // measured: cfg3 first pass 0.452 -> 0.392 ms (the L1 data pipe is its limiter)
#endif
        auto store_chunk = [&](int k, const uint32_t (&v)[4]) {
            if (d0 + 8 * k < p.out_width) {
                if (k == NCK - 1) store_chunk_head<2>(dst + 8 * k, v, 8 - rho);
#ifdef D3_STAGE_EVICT_LAST
                else st_hint_v4(dst + 8 * k, v[0], v[1], v[2], v[3], keep_pol);
#else
                else *reinterpret_cast<uint4 *>(dst + 8 * k) = make_uint4(v[0], v[1], v[2], v[3]);
#endif
            }
        };
#if D3_SWAR_ST256
        // chunk pairs (2j, 2j + 1) below the head chunk leave as one 32-byte store (STG.256: a whole
        // sector per lane); al32 is uniform over the CTA
        static_assert(NCK % 2 == 0, "chunk pairs");
        const bool al32 = (p.out_pitch % 16 == 0) && (p.out_inst_stride % 16 == 0) &&
                          ((reinterpret_cast<unsigned long long>(outp) & 31ull) == 0);
#pragma unroll
        for (int k = 0; k < NCK; k += 2) {
            uint32_t va[4], vb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                va[i] = __byte_perm(w[4 * k + i], w[4 * k + i + 1], sel);
                vb[i] = __byte_perm(w[4 * k + 4 + i], w[4 * k + 5 + i], sel);
            }
            if (k + 1 < NCK - 1 && al32 && d0 + 8 * (k + 1) < p.out_width) {
                const uint32_t v8[8] = {va[0], va[1], va[2], va[3], vb[0], vb[1], vb[2], vb[3]};
                st_v8(dst + 8 * k, v8);
            } else {
                store_chunk(k, va);
                store_chunk(k + 1, vb);
            }
        }
#else
#pragma unroll
        for (int k = 0; k < NCK; ++k) {
            uint32_t v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = __byte_perm(w[4 * k + i], w[4 * k + i + 1], sel);
            store_chunk(k, v);
        }
#endif
        if (rho > 0 && d0 >= 8) {
            // tile elements [0, rho) end the previous chunk: window (zeros, row words 0..3)
            const uint32_t *r0 = reinterpret_cast<const uint32_t *>(sm + G::ORP * rr) + row_skew<S>(r1);
            uint32_t tw[8] = {0u, 0u, 0u, 0u, r0[0], r0[1], r0[2], r0[3]}, v[4];
            window_chunk<2>(tw, rho, 0, v);
            store_chunk_tail<2>(dst - 8, v, rho);
        }
    }
#endif
    // ---- zero tiles of the final output (DESIGN.md §5 item 6).  This pass leaves HBM mostly idle,
    // so it stores the final pass's all-zero tiles: its shared memory is free after the copy-out,
    // a zeroed S x S x zf_T image leaves with one TMA tensor store per tile (zmap: the final output
    // out[inst][s1][s2][3N], box {zf_T, S, S, 1}).  The final pass has one group per S x S slope
    // block (sg1, sg2) = (g >> K, g & (S - 1)) -- as many as this pass's column blocks, so this
    // CTA's g -- and tiles of zf_T along D (out_base 0); tile t is zero when (t + 1) zf_T <=
    // 2N - s1max - s2max (the final pass's test).  Tiles t = blockIdx.x, + gridDim.x, ... here.
    if (p.zf_T > 0) {
        const int gs2 = g & (S - 1), gs1 = g >> K;
        const int nz = (2 * N - ((gs1 << K) + S - 1) - ((gs2 << K) + S - 1)) / p.zf_T;
        if ((int)blockIdx.x < nz) {
            if constexpr (K == 4 && G::SMEM < S * S * D3_FINAL16_T * 4) {
                __trap();                                     // a zero tile image must fit (host checks zf_T)
            }
            __syncthreads();                                  // every copy-out read is done
            for (int i = tid; i < S * S * p.zf_T / 4; i += blockDim.x)
                reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
                for (int t = blockIdx.x; t < nz; t += gridDim.x)
                    asm volatile(
                        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&zmap),
                        "r"(t * p.zf_T), "r"(gs2 << K), "r"(gs1 << K), "r"(p.inst0 + li), "r"(src)
                        : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        }
    }
#ifdef D3_PROF_SWAR
    SW_MARK(6);
    if (tid == 0) {
        for (int i = 0; i < 6; ++i) atomicAdd(&d3_swar_prof[i], (unsigned long long)(sw_t[i + 1] - sw_t[i]));
        atomicAdd(&d3_swar_prof[7], 1ull);
    }
#endif
}

}  // namespace d3
