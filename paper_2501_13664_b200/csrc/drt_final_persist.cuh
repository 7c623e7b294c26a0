// drt_final_persist.cuh -- persistent last DRT pass for u16 stage-c rows -> int32 stacked
// output (u8 voxels, the headline N=256 plan 4 | 4).
//
// Same arithmetic as drt_pass_kernel (pass identity).  Two CTAs per SM loop
// over the tiles of the launch (static round robin); per tile:
//   1. wait for the tile's staged rows (cp.async, issued during the previous tile);
//   2. x-step from the staged rows -> registers;
//   3. issue the cp.async staging of the CTA's next tile (overlaps steps 4-8);
//   4. wait until the previous tile's TMA store has read the X/output region;
//   5. write X;  6. y-step -> registers;
//   7. write the output tile (dense [r1][r2][T]) over X;  8. one TMA tensor store, not waited for.
// So neither the staging latency nor the output drain is exposed.  Tiles wholly below the
// support are written as zeros with plain stores.  Shared memory per CTA: staged rows
// (S^2 x BW u16) + X (S^2 x XP bytes) ~ 110 KB at T = 48.
#pragma once
#include "drt_kernels.cuh"

namespace d3 {

template <int K, int R, int T>
struct PersistGeom {
    static constexpr int S = 1 << K;
    static constexpr int H = S - 1;
    static constexpr int NRX = (T + H + R - 1) / R;       // x-step runs per row
    static constexpr int NRY = T / R;                     // y-step runs per row
    static constexpr int RD = (NRX - 1) * R + (R + H + 7) / 8 * 8;
    static constexpr int WIN = T + 2 * H;
    static constexpr int BW = ((WIN > RD ? WIN : RD) + 15) / 16 * 16;   // staged u16 per row
    static constexpr int NCH = BW / 8;                    // 16-byte chunks per staged row
    static constexpr int SPS = BW * 2;                    // staged slot pitch (bytes)
    static constexpr int STAGED_BYTES = S * S * SPS;
    static constexpr int XW = NRX * R;                    // X words per row
    static constexpr int XP = XW * 4 + 16;                // X slot pitch (bytes)
    static constexpr int X_BYTES = S * S * XP;
    static constexpr int OUT_BYTES = S * S * T * 4;       // dense output tile (TMA store source)
    static constexpr int SMEM = STAGED_BYTES + X_BYTES;
    static constexpr int XTASKS = S * NRX;
    static constexpr int YTASKS = S * NRY;
    static constexpr int THREADS = ((XTASKS > YTASKS ? XTASKS : YTASKS) + 31) / 32 * 32;
    static_assert(OUT_BYTES <= X_BYTES, "output tile overlays X");
    static_assert(R == 8 && T % R == 0, "tile shape");
};

template <int K, int R, int T>
__global__ void __launch_bounds__(PersistGeom<K, R, T>::THREADS, 2)
drt_final_persist_kernel(const DrtPass p, const __grid_constant__ CUtensorMap omap, int log_ntiles_d, int tiles_total) {
    using G = PersistGeom<K, R, T>;
    constexpr int S = G::S, NCH = G::NCH;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *stg = smem_raw;                        // staged u16 rows, slot (w1, w2) = w1 S + w2
    unsigned char *xo = smem_raw + G::STAGED_BYTES;       // X slots (r1, w2) / then the output tile

    const int tid = threadIdx.x;
    const int N = p.N, m = p.m, c = p.c, nc = p.n - c;
    const int log_per_inst = 2 * (c + m) + log_ntiles_d;
    struct Tile {
        int li, d0, sg1, sg2, V1, V2;
        bool zero;
    };
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

    // ---- staging of one tile: thread (sub, q) copies chunk q of slots sub, sub + SUBS, ...
    const uint16_t *inb = reinterpret_cast<const uint16_t *>(p.in);
    const int nchunk = p.in_width >> 3;
    constexpr int SUBS = G::THREADS / NCH;
    const int q = tid % NCH, sub = tid / NCH;
    auto stage = [&](const Tile &t) {
        if (sub < SUBS) {
            const uint16_t *rb = inb + ((((long long)t.sg1 << c) + t.sg2) << (2 * nc)) * p.in_pitch +
                                 (long long)t.li * p.in_inst_stride +
                                 (((long long)(t.V1 << K) << nc) + (t.V2 << K)) * p.in_pitch;
            const int cq = ((p.out_base + t.d0 - p.in_base) >> 3) + q;
            unsigned char *dst = stg + sub * G::SPS + 16 * q;
#pragma unroll 4
            for (int slot = sub; slot < S * S; slot += SUBS, dst += SUBS * G::SPS) {
                const int w1 = slot >> K, w2 = slot & (S - 1);
                const int cc = cq + ((t.sg1 * w1 + t.sg2 * w2) >> 3);
                const bool ok = (unsigned)cc < (unsigned)nchunk;
                const uint32_t off = ((uint32_t)((w1 << nc) + w2) * (uint32_t)p.in_pitch + (uint32_t)(ok ? cc : 0) * 8u) * 2u;
                cp_async16(dst, reinterpret_cast<const char *>(rb) + off, ok);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto next_nonzero = [&](int tt) {
        for (; tt < tiles_total; tt += gridDim.x)
            if (!tile_of(tt).zero) return tt;
        return tiles_total;
    };

    uint32_t *outp = reinterpret_cast<uint32_t *>(p.out);
    const int xr = tid % G::NRX, xb = tid / G::NRX;       // x task (w2 = xb, run xr)
    const int yr = tid % G::NRY, yb = tid / G::NRY;       // y task (r1 = yb, run yr)
    uint32_t acc[S][R];
    auto zero_acc = [&]() {
#pragma unroll
        for (int i = 0; i < S; ++i)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[i][j] = 0u;
    };

    int cur = next_nonzero(blockIdx.x);
    if (cur < tiles_total) stage(tile_of(cur));
    for (int tt = blockIdx.x; tt < tiles_total; tt += gridDim.x) {
        const Tile t = tile_of(tt);
        if (t.zero) {
            // zeros, straight from registers (no shared memory involved)
            if (tid < G::YTASKS) {
                const long long s1 = ((long long)t.sg1 << K) + yb;
                uint32_t *dst = outp + (long long)(p.inst0 + t.li) * p.out_inst_stride +
                                (((s1 << (c + K)) + ((long long)t.sg2 << K)) << (2 * m)) * p.out_pitch +
                                (((long long)t.V1 << m) + t.V2) * p.out_pitch + t.d0 + yr * R;
                const long long r2_stride = (long long)p.out_pitch << (2 * m);
#pragma unroll
                for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                    for (int qq = 0; qq < R / 4; ++qq) st_cs_v4(dst + r2 * r2_stride + 4 * qq, 0u, 0u, 0u, 0u);
            }
            continue;
        }
        // 1. this tile's staged rows
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        // 2. x-step
        if (tid < G::XTASKS) {
            zero_acc();
            drt_accumulate<K, R, G::SPS, true, uint32_t>(stg, xb, S, xr * (R / 8), p.one, acc);
        }
        __syncthreads();
        // 3. next tile's staging overlaps the rest of this tile
        const int nxt = next_nonzero(tt + gridDim.x);
        if (nxt < tiles_total) stage(tile_of(nxt));
        // 4. the previous TMA store must have read the X/output region
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        // 5. X
        if (tid < G::XTASKS) {
#pragma unroll
            for (int r = 0; r < S; ++r)
#pragma unroll
                for (int qq = 0; qq < R / 4; ++qq)
                    *reinterpret_cast<uint4 *>(xo + (r * S + xb) * G::XP + 16 * xswz(xr * (R / 4) + qq)) =
                        make_uint4(acc[r][4 * qq], acc[r][4 * qq + 1], acc[r][4 * qq + 2], acc[r][4 * qq + 3]);
        }
        __syncthreads();
        // 6. y-step
        if (tid < G::YTASKS) {
            zero_acc();
            drt_accumulate<K, R, G::XP, false, uint32_t>(xo, yb * S, 1, yr * (R / 4), p.one, acc);
        }
        __syncthreads();
        // 7. dense output tile [r1][r2][T] over X
        if (tid < G::YTASKS) {
            unsigned char *row = xo + ((yb * S) * T + yr * R) * 4;
#pragma unroll
            for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                for (int qq = 0; qq < R / 4; ++qq)
                    *reinterpret_cast<uint4 *>(row + (r2 * T + 4 * qq) * 4) =
                        make_uint4(acc[r2][4 * qq], acc[r2][4 * qq + 1], acc[r2][4 * qq + 2], acc[r2][4 * qq + 3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        // 8. one TMA tensor store of the box {T, S (s2), S (s1), 1}; drained later (step 4)
        if (tid == 0) {
            const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(xo));
            asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&omap),
                         "r"(t.d0), "r"(t.sg2 << K), "r"(t.sg1 << K), "r"(p.inst0 + t.li), "r"(src)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace d3
