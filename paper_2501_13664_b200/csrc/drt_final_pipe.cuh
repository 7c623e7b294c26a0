// drt_final_pipe.cuh -- persistent, warp-specialised last DRT pass for u16
// stage-c rows (u8 voxels, the headline N=256 plan 4 | 4).
//
// Same arithmetic as drt_pass_kernel (pass identity): for each
// tile (D window of T outputs, one 2^K x 2^K group of stage-c rows)
//   X(r1, w2)[e]   = sum_{w1} f(w1, w2)[e + l^K_{r1}(w1)]        (x-step)
//   out(r1, r2)[e] = sum_{w2} X(r1, w2)[e + l^K_{r2}(w2)]       (y-step)
// but organised as a pipeline so that no warp waits on L2 latency or on the
// other step:
//   * one CTA per SM loops over the tiles of the launch (static round robin);
//   * X-team warps (one task per (w2, run)) sum the rows in two halves of w1;
//     each half lives in its own shared buffer and is refilled with cp.async
//     for the CTA's next tile as soon as it has been consumed, so the copy
//     overlaps the other half's arithmetic;
//   * X goes to one of two shared buffers; Y-team warps (one task per
//     (r1, run)) consume it and stream the output rows from registers while
//     the X-team already works on the next tile.
// Hand-off is by named barriers: FULL[b] (X arrives, Y waits) and EMPTY[b]
// (Y arrives, X waits), b = tile parity.  Tiles wholly below the support are
// written as zeros by the Y-team alone.
#pragma once
#include "drt_kernels.cuh"

namespace d3 {

template <int K, int R, int T>
struct PipeGeom {
    static constexpr int S = 1 << K;
    static constexpr int H = S - 1;
    static constexpr int NRX = (T + H + R - 1) / R;       // x-step runs per row
    static constexpr int NRY = T / R;                     // y-step runs per row
    static constexpr int RD = (NRX - 1) * R + (R + H + 7) / 8 * 8;
    static constexpr int WIN = T + 2 * H;
    static constexpr int BW = ((WIN > RD ? WIN : RD) + 15) / 16 * 16;   // staged u16 per row
    static constexpr int NCH = BW / 8;                    // 16-byte chunks per staged row
    static constexpr int RAWP = BW * 2;                   // raw slot pitch (bytes)
    static constexpr int HALF = S * S / 2;                // slots per w1 half
    static constexpr int RAW_BYTES = HALF * RAWP;
    static constexpr int XW = NRX * R;                    // X words per row
    static constexpr int XP = XW * 4 + 16;                // X slot pitch (bytes)
    static constexpr int X_BYTES = S * S * XP + 16 * S;  // + per-r1 rotation (xslot)
    static constexpr int NRAW = 4;                        // ring of raw half-buffers (2 tiles in flight)
    static constexpr int XOFF = NRAW * RAW_BYTES;
    static constexpr int MBAR_OFF = XOFF + 2 * X_BYTES;   // NRAW mbarriers (raw half landed)
    static constexpr int SMEM = MBAR_OFF + 8 * NRAW;
    static constexpr int XTASKS = S * NRX;
    static constexpr int YTASKS = S * NRY;
    static constexpr int XWARPS = (XTASKS + 31) / 32;
    static constexpr int YWARPS = (YTASKS + 31) / 32;
    static constexpr int XTHREADS = XWARPS * 32;
    static constexpr int YTHREADS = YWARPS * 32;
    static constexpr int PTHREADS = 32;                   // one producer warp (cp.async issue)
    static constexpr int THREADS = XTHREADS + YTHREADS + PTHREADS;
    static_assert(R == 8 && T % R == 0 && YTASKS % 32 == 0 && XTASKS % 32 == 0, "tile shape");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// mbarrier that completes when every producer lane's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_addr(bar)), "r"(parity) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// acc[r][j] += sum_{a in [A0, A1)} row_a[j + l^K_r(a)] over u16 rows (unswizzled) at
// slot0 + (a - A0) * sstep; run start = chunk c0.  Rows are taken two at a time (IADD3).
// byte offset of X slot (r1, w2): the r1 groups are rotated by one 16-byte chunk each so that a
// quarter-warp straddling two r1 groups (NRY not a multiple of 8) hits distinct banks
template <int S, int XP>
__device__ __forceinline__ int xslot(int r1, int w2) { return (r1 * S + w2) * XP + 16 * r1; }

// The u16 unpack runs on the FMA pipe (hi = umulhi(w, 2^16), lo = w - hi 2^16 with runtime
// constants), and FMA16 of 16 rows take their adds as IMAD pairs, so the ALU and FMA pipes
// share the work (each accepts one warp instruction every 2 cycles per SMSP).
template <int K, int R, int SP, int A0, int A1, int FMA16>
__device__ __forceinline__ void accumulate_u16_rows(const unsigned char *__restrict__ sm, int slot0, int sstep, int c0,
                                                    uint32_t one, uint32_t (&acc)[1 << K][R]) {
    constexpr int S = 1 << K;
    const uint32_t k16 = one << 16, m16 = 0u - k16;
    auto load = [&](int a, int ne, uint32_t *buf) {
        const unsigned char *row = sm + (slot0 + (a - A0) * sstep) * SP;
#pragma unroll
        for (int i = 0; i < (ne + 7) / 8; ++i) {
            const uint4 v = *reinterpret_cast<const uint4 *>(row + 16 * (c0 + i));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const uint32_t hi = __umulhi(w[h], k16);
                if (8 * i + 2 * h < ne) buf[8 * i + 2 * h] = w[h] + hi * m16;
                if (8 * i + 2 * h + 1 < ne) buf[8 * i + 2 * h + 1] = hi;
            }
        }
    };
    static_for<A0 / 2, A1 / 2>([&](auto p_) {
        constexpr int a0 = 2 * decltype(p_)::value, a1 = a0 + 1;
        uint32_t b0[R + a0], b1[R + a1];
        load(a0, R + a0, b0);
        load(a1, R + a1, b1);
        static_for<0, S>([&](auto r_) {
            constexpr int r = decltype(r_)::value;
            constexpr int o0 = lk(K, r, a0), o1 = lk(K, r, a1);
            constexpr bool fma = fma_row(r, FMA16);
#pragma unroll
            for (int j = 0; j < R; ++j) acc[r][j] = add2<uint32_t>(acc[r][j], b0[j + o0], b1[j + o1], one, fma);
        });
    });
}

// -DPIPE_PROF: per-role clock accounting (lane 0 of each role's first warp, summed over CTAs
// into d3_pipe_prof[], printed by CTA 0 at exit).  Debug builds only.
#ifdef PIPE_PROF
__device__ unsigned long long d3_pipe_prof[16];
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(slot, t0) do { if (prof_on) acc_prof[slot] += clock64() - (t0); } while (0)
#else
#define PROF_T(v)
#define PROF_ADD(slot, t0) do { } while (0)
#endif

// output store flavour (experiment): 0 = st.global.cs, 1 = L2::evict_first policy, 2 = plain
#ifndef PIPE_STORE_MODE
#define PIPE_STORE_MODE 0
#endif
__device__ __forceinline__ void st_out_v4(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t pol) {
#if PIPE_STORE_MODE == 0
    st_cs_v4(p, a, b, c, d);
#elif PIPE_STORE_MODE == 1
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
                 "l"(pol) : "memory");
#else
    *reinterpret_cast<uint4 *>(p) = make_uint4(a, b, c, d);
#endif
}

#ifndef PIPE_X_FMA16
#define PIPE_X_FMA16 3                                    // x-step: unpack on FMA + 3/16 of the add pairs
#endif
#ifndef PIPE_Y_FMA16
#define PIPE_Y_FMA16 5                                    // y-step: ~1/3 of the add pairs on FMA
#endif

template <int K, int R, int T>
__global__ void __launch_bounds__(PipeGeom<K, R, T>::THREADS, 1)
drt_final_pipe_kernel(const DrtPass p, int log_ntiles_d, int tiles_total) {
    using G = PipeGeom<K, R, T>;
    constexpr int S = G::S, HALF = G::HALF, NCH = G::NCH;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // raw ring buffer i at smem_raw + i * RAW_BYTES; X buffer b at XOFF + b * X_BYTES
    constexpr int XOFF = G::XOFF, NRAW = G::NRAW;
    constexpr int BAR_FULL = 2, BAR_EMPTY = 4, BAR_RAW_EMPTY = 6;   // + parity / ring slot (6..9)
    constexpr int NX = G::XTHREADS, NXY = G::XTHREADS + G::YTHREADS;

    const int tid = threadIdx.x;
    const int N = p.N, m = p.m, c = p.c, cK = c + K, nc = p.n - c;
#ifdef PIPE_PROF
    long long acc_prof[4] = {0, 0, 0, 0};
    const bool prof_on = (tid == 0 || tid == G::XTHREADS || tid == G::XTHREADS + G::YTHREADS);
    const int prof_base = tid == 0 ? 0 : (tid == G::XTHREADS ? 4 : 8);
    PROF_T(t_start);
#endif
    uint64_t *fullm = reinterpret_cast<uint64_t *>(smem_raw + G::MBAR_OFF);
    if (tid == 0) {
        for (int i = 0; i < G::NRAW; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(fullm + i)), "r"(32) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // tile tt -> (instance li, group g, D tile d); group g -> (sg1, sg2, V1, V2)
    struct Tile {
        int li, d0, sg1, sg2, V1, V2;
        bool zero;
    };
    const int log_per_inst = 2 * (c + m) + log_ntiles_d;
    auto tile_of = [&](int tt) {
        Tile t;
        t.li = tt >> log_per_inst;
        const int rem = tt & ((1 << log_per_inst) - 1);
        const int g = rem >> log_ntiles_d, d = rem & ((1 << log_ntiles_d) - 1);
        t.d0 = d * T;
        t.V2 = g & ((1 << m) - 1);
        t.V1 = (g >> m) & ((1 << m) - 1);
        const int sig = g >> (2 * m);
        t.sg2 = sig & ((1 << c) - 1);
        t.sg1 = sig >> c;
        const int s1max = (t.sg1 << K) + S - 1, s2max = (t.sg2 << K) + S - 1;
        t.zero = p.out_base + t.d0 + T <= 2 * N - s1max - s2max;   // support D >= 2N - s1 - s2
        return t;
    };

    auto next_nonzero = [&](int tt) {
        for (; tt < tiles_total; tt += gridDim.x)
            if (!tile_of(tt).zero) return tt;
        return tiles_total;
    };

    if (tid >= NXY) {
        // ============================ producer warp ============================
        // copies w1-half h of each non-zero tile into raw[h] once the X-team has released it;
        // both halves can be in flight; each half has an mbarrier that completes when it lands.
        const int lane = tid - NXY;
        const uint16_t *inb = reinterpret_cast<const uint16_t *>(p.in);
        const int nchunk = p.in_width >> 3;
        constexpr int SPI = 32 / NCH;                       // slots per iteration (lanes < SPI * NCH work)
        const int q = lane % NCH, sub = lane / NCH;
        int seq = 0;                                        // half-tiles issued so far
        // per half: wait until the X-team has released the buffer, issue the copies and let the
        // mbarrier of the half track their completion; both halves can be in flight.
        const int pitch = p.in_pitch;
        for (int tt = next_nonzero(blockIdx.x); tt < tiles_total; tt = next_nonzero(tt + gridDim.x)) {
            const Tile t = tile_of(tt);
            // the tile's 2^K x 2^K rows: row (a, w) = tile row base + (a << nc) + w (V folded in)
            const uint16_t *tb = inb + ((((long long)t.sg1 << c) + t.sg2) << (2 * nc)) * pitch +
                                 (long long)t.li * ((long long)N * N) * pitch +
                                 ((long long)(t.V1 << K) << nc) * pitch + (long long)(t.V2 << K) * pitch;
            const int cb = ((p.out_base + t.d0 - p.in_base) >> 3) + q;
#pragma unroll 1
            for (int h = 0; h < 2; ++h, ++seq) {
                const int bi = seq & (NRAW - 1);
                PROF_T(tp0);
                named_sync(BAR_RAW_EMPTY + bi, NX + 32);
                PROF_ADD(0, tp0);
                PROF_T(tp1);
                if (sub < SPI) {
                    unsigned char *dbase = smem_raw + bi * G::RAW_BYTES + 16 * q;
#pragma unroll 4
                    for (int slot = sub; slot < HALF; slot += SPI) {
                        const int a = (slot >> K) + h * (S / 2), ww = slot & (S - 1);   // slot = (a - h S/2) S + w2
                        const int cc = cb + ((t.sg1 * a + t.sg2 * ww) >> 3);
                        const bool ok = (unsigned)cc < (unsigned)nchunk;
                        const uint16_t *src = tb + ((a << nc) + ww) * pitch + 8 * cc;
                        cp_async16(dbase + slot * G::RAWP, ok ? (const void *)src : (const void *)inb, ok);
                    }
                }
                cp_async_arrive_noinc(fullm + bi);           // completes when this lane's copies land
                PROF_ADD(1, tp1);
            }
        }
    } else if (tid < NX) {
        // ============================ X-team ============================
        const int xt = tid;
        // quarter-warps take 8 consecutive runs of one row (conflict-free LDS.128)
        int w2, run;
        if constexpr (G::NRX == 8) {
            w2 = xt >> 3;
            run = xt & 7;
        } else {
            if (xt < S * 8) { w2 = xt >> 3; run = xt & 7; }
            else { const int u = xt - S * 8; w2 = u / (G::NRX - 8); run = 8 + u % (G::NRX - 8); }
        }
        const bool xact = xt < G::XTASKS;
        for (int i = 0; i < NRAW; ++i) named_arrive(BAR_RAW_EMPTY + i, NX + 32);
        int nz = 0;
        for (int cur = next_nonzero(blockIdx.x); cur < tiles_total; cur = next_nonzero(cur + gridDim.x)) {
            uint32_t acc[S][R];
#pragma unroll
            for (int i = 0; i < S; ++i)
#pragma unroll
                for (int j = 0; j < R; ++j) acc[i][j] = 0u;
            // half 0: w1 in [0, S/2), half 1: w1 in [S/2, S)
            const int b0 = (2 * nz) & (NRAW - 1), b1 = (2 * nz + 1) & (NRAW - 1);
            const uint32_t ph = ((2 * nz) / NRAW) & 1;      // ring round of this tile's halves
            PROF_T(tx0);
            mbar_wait_parity(fullm + b0, ph);
            PROF_ADD(0, tx0);
            PROF_T(tx1);
            if (xact) accumulate_u16_rows<K, R, G::RAWP, 0, S / 2, PIPE_X_FMA16>(smem_raw + b0 * G::RAW_BYTES, w2, S, run, p.one, acc);
            named_arrive(BAR_RAW_EMPTY + b0, NX + 32);
            PROF_ADD(1, tx1);
            PROF_T(tx2);
            mbar_wait_parity(fullm + b1, ph);
            PROF_ADD(0, tx2);
            PROF_T(tx3);
            if (xact) accumulate_u16_rows<K, R, G::RAWP, S / 2, S, PIPE_X_FMA16>(smem_raw + b1 * G::RAW_BYTES, w2, S, run, p.one, acc);
            named_arrive(BAR_RAW_EMPTY + b1, NX + 32);
            PROF_ADD(1, tx3);
            // X -> xb[nz & 1] once the Y-team has released it
            const int b = nz & 1;
            PROF_T(tx4);
            named_sync(BAR_EMPTY + b, NXY);
            PROF_ADD(2, tx4);
            PROF_T(tx5);
            if (xact) {
#pragma unroll
                for (int r = 0; r < S; ++r)
#pragma unroll
                    for (int q = 0; q < R / 4; ++q)
                        *reinterpret_cast<uint4 *>(smem_raw + XOFF + b * G::X_BYTES + xslot<S, G::XP>(r, w2) + 16 * xswz(run * (R / 4) + q)) =
                            make_uint4(acc[r][4 * q], acc[r][4 * q + 1], acc[r][4 * q + 2], acc[r][4 * q + 3]);
            }
            named_arrive(BAR_FULL + b, NXY);
            PROF_ADD(3, tx5);
            ++nz;
        }
        // drain: match the producer's two outstanding RAW_EMPTY waits and the Y-team's EMPTY arrivals
        named_sync(BAR_EMPTY + (nz & 1), NXY);
        named_sync(BAR_EMPTY + ((nz + 1) & 1), NXY);
    } else {
        // ============================ Y-team ============================
        const int yt = tid - NX;
        const int r1 = yt / G::NRY, run = yt - r1 * G::NRY;
        uint32_t *outp = reinterpret_cast<uint32_t *>(p.out);
        uint64_t pol_first;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        named_arrive(BAR_EMPTY + 0, NXY);
        named_arrive(BAR_EMPTY + 1, NXY);
        int nz = 0;
        for (int tt = blockIdx.x; tt < tiles_total; tt += gridDim.x) {
            const Tile t = tile_of(tt);
            const long long s1 = ((long long)t.sg1 << K) + r1;
            const long long out_inst = (long long)(p.inst0 + t.li) * p.out_inst_stride;
            uint32_t *dst = outp + out_inst +
                            ((((s1 << cK) + ((long long)t.sg2 << K)) << (2 * m)) + ((long long)t.V1 << m) + t.V2) * p.out_pitch +
                            t.d0 + run * R;
            const long long r2_stride = (long long)p.out_pitch << (2 * m);
            if (t.zero) {
#pragma unroll
                for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                    for (int q = 0; q < R / 4; ++q) st_out_v4(dst + r2 * r2_stride + 4 * q, 0u, 0u, 0u, 0u, pol_first);
                continue;
            }
            const int b = nz & 1;
            uint32_t acc[S][R];
#pragma unroll
            for (int i = 0; i < S; ++i)
#pragma unroll
                for (int j = 0; j < R; ++j) acc[i][j] = 0u;
            PROF_T(ty0);
            named_sync(BAR_FULL + b, NXY);
            PROF_ADD(0, ty0);
            PROF_T(ty1);
            drt_accumulate<K, R, G::XP, false, uint32_t, PIPE_Y_FMA16>(smem_raw + XOFF + b * G::X_BYTES + 16 * r1, r1 * S, 1,
                                                                 run * (R / 4), p.one, acc);
            named_arrive(BAR_EMPTY + b, NXY);
            PROF_ADD(1, ty1);
            PROF_T(ty2);
            ++nz;
#pragma unroll
            for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                for (int q = 0; q < R / 4; ++q)
                    st_out_v4(dst + r2 * r2_stride + 4 * q, acc[r2][4 * q], acc[r2][4 * q + 1], acc[r2][4 * q + 2],
                              acc[r2][4 * q + 3], pol_first);
            PROF_ADD(2, ty2);
        }
    }
#ifdef PIPE_PROF
    if (prof_on) {
        acc_prof[3] += 0;
        for (int i = 0; i < 4; ++i) atomicAdd(&d3_pipe_prof[prof_base + i], (unsigned long long)acc_prof[i]);
        atomicAdd(&d3_pipe_prof[12 + prof_base / 4], (unsigned long long)(clock64() - t_start));
    }
#endif
}

}  // namespace d3
