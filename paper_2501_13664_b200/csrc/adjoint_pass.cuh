// adjoint_pass.cuh -- backprojection of one radix-2^K DRT pass.
//
// The forward pass (drt_kernels.cuh) computes, with s' = s 2^K + r and v = V 2^K + w,
//   f^{c+K}(s', V)[D] = sum_w f^c(s, v)[D + s1 w1 + s2 w2 + l^K_{r1}(w1) + l^K_{r2}(w2)].
// Its transpose -- K consecutive stages of eq:invmap3Dsummation run in
// reversed order -- is
//   g^c(s, v)[E] = sum_r g^{c+K}(s', V)[E - s1 w1 - s2 w2 - l^K_{r1}(w1) - l^K_{r2}(w2)]
//               = Z_w[E - s1 w1 - s2 w2],   Z_w[e] = sum_r g^{c+K}(s', V)[e - l^K_{r1}(w1) - l^K_{r2}(w2)].
// Z is the forward's separable direct sum with the roles of r and w exchanged and offsets
// H - l^K_r(w) (compile-time, register indexing: drt_accumulate<..., TR = true>), read from
// rows staged with NO runtime shift; the runtime shift s.w moves to the store: output row w
// of the tile is written at E = e + s1 w1 + s2 w2, realigned in registers (one shuffle with the
// neighbouring run), partial 16-byte chunks at the tile ends, exactly like the forward's
// pre-shifted intermediate stores.  Each output row's E range is covered by the tiles once.
//
// Level storage (adjoint only): level c rows ((s1 2^c + s2) 2^(n-c) + v1) 2^(n-c) + v2 (the
// forward's stage-c order), element p <-> E = base + p.  Only E in [lo_c, 3N) is needed
// (lo_c = 2N - 2(2^c - 1), the support argument: a needed output reads only needed inputs);
// other stored positions may hold anything.  Level n is the caller's coefficients (base 0).
#pragma once
#include "drt_kernels.cuh"

namespace d3 {

struct AdjPass {
    const void *in;
    void *out;
    int N, n, c, m;                 // output level c; m = n - c - K position bits per axis of the inputs
    long long in_inst_stride, out_inst_stride;
    int in_pitch, in_base, in_width;
    int out_pitch, out_base, out_width;
    int lo;                         // lowest needed E of the output level
    int ebase;                      // e of tile 0 (e0 - 2H - in_base is a multiple of 4)
    uint32_t one;
};

template <int K, int R, int T, class Acc>
__global__ void __launch_bounds__(DrtGeom<K, R, T, false>::THREADS) __maxnreg__((DrtGeom<K, R, T, false>::MAXREG))
drt_adj_pass_kernel(const AdjPass p) {
    using G = DrtGeom<K, R, T, false>;
    constexpr int S = G::S, SP = G::SP, BW = G::BW, H = G::H;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;

    const int tid = threadIdx.x;
    const int tile = blockIdx.x, g = blockIdx.y, li = blockIdx.z;
    const int m = p.m, c = p.c, n = p.n, N = p.N;
    const int V2 = g & ((1 << m) - 1);
    const int V1 = (g >> m) & ((1 << m) - 1);
    const int sig = g >> (2 * m);
    const int sg2 = sig & ((1 << c) - 1);
    const int sg1 = sig >> c;
    const int e0 = p.ebase + tile * T;
    if (e0 + T + H * (sg1 + sg2) <= p.lo || e0 >= 3 * N) return;     // no needed output in this tile

    // ---- stage the 4^K input rows (r1, r2) of level c+K over e in [e0 - 2H, e0 - 2H + BW):
    // plain aligned 16-byte copies (cp.async, zero-filled outside the stored row)
    {
        const uint32_t *inb = reinterpret_cast<const uint32_t *>(p.in) + (long long)li * p.in_inst_stride;
        const int cK = c + K;
        const int cc0 = (e0 - 2 * H - p.in_base) >> 2;                 // exact (multiple of 4), may be < 0
        const int nchunk = p.in_width >> 2;
        constexpr int NCH = BW / 4;
        constexpr int SUBS = G::THREADS / NCH;
        const int q = tid % NCH, sub = tid / NCH;
        if (sub < SUBS) {
            const int cc = cc0 + q;
            const bool ok = (unsigned)cc < (unsigned)nchunk;
            for (int slot = sub; slot < S * S; slot += SUBS) {
                const int r1 = slot >> K, r2 = slot & (S - 1);
                const long long row = ((((long long)((sg1 << K) + r1) << cK) + ((sg2 << K) + r2)) << (2 * m)) +
                                      ((long long)V1 << m) + V2;
                cp_async16(sm + slot * SP + 16 * xswz(q), inb + row * p.in_pitch + (ok ? cc : 0) * 4, ok);
            }
        }
        cp_async_wait_all();
    }
    __syncthreads();

    // ---- x-step: X(w1, r2)[e'] = sum_r1 in(r1, r2)[e' - l_r1(w1)], written in place over slot
    // (w1, r2); y-step: Z(w1, w2)[e] = sum_r2 X(w1, r2)[e - l_r2(w2)]
    Acc acc[S][R];
    int xb, xr;
    task_row_run(tid, G::NRX, S, xb, xr);
    const int yr = tid % G::NRY, yb = tid / G::NRY;
    auto zero_acc = [&]() {
#pragma unroll
        for (int i = 0; i < S; ++i)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[i][j] = Acc(0);
    };
    if (tid < G::XT) {
        zero_acc();
        drt_accumulate<K, R, SP, false, Acc, -1, true>(sm, xb, S, xr * (R / 4), p.one, acc);
    }
    __syncthreads();
    if (tid < G::XT) {
#pragma unroll
        for (int i = 0; i < S; ++i)
#pragma unroll
            for (int q = 0; q < R / 4; ++q)
                *reinterpret_cast<uint4 *>(sm + (i * S + xb) * SP + 16 * xswz(xr * (R / 4) + q)) =
                    make_uint4(Lane<Acc>::bits(acc[i][4 * q + 0]), Lane<Acc>::bits(acc[i][4 * q + 1]),
                               Lane<Acc>::bits(acc[i][4 * q + 2]), Lane<Acc>::bits(acc[i][4 * q + 3]));
    }
    __syncthreads();
    if (tid < G::YT) {
        zero_acc();
        drt_accumulate<K, R, SP, false, Acc, -1, true>(sm, yb * S, 1, yr * (R / 4), p.one, acc);
    }

    // ---- store: row (w1 = yb, w2), tile element t at E = e0 + t + sg1 w1 + sg2 w2
    if (tid < G::YT) {
        static_assert(R == 8, "epilogue: two chunks per run");
        constexpr int NW = R;                                           // words per run (32-bit)
        const int w1 = yb;
        const int nc = n - c;
        uint32_t *outb = reinterpret_cast<uint32_t *>(p.out) + (long long)li * p.out_inst_stride;
        const long long rbase = ((((long long)sg1 << c) + sg2) << (2 * nc)) + ((long long)((V1 << K) + w1) << nc) +
                                ((long long)V2 << K);
#pragma unroll
        for (int w2 = 0; w2 < S; ++w2) {
            uint32_t win[NW + 4];
#pragma unroll
            for (int i = 0; i < NW; ++i) win[i] = Lane<Acc>::bits(acc[w2][i]);
#pragma unroll
            for (int i = 0; i < 4; ++i) win[NW + i] = __shfl_down_sync(0xffffffffu, win[i], 1, G::NRY);
            const int P0 = e0 - p.out_base + sg1 * w1 + sg2 * w2;      // stored position of t = 0
            const int rho = P0 & 3, A = P0 - rho;                       // A: chunk-aligned
            const int rp = (4 - rho) & 3, kb = rho ? 1 : 0;
            uint32_t *row = outb + (rbase + w2) * p.out_pitch;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int pos = A + 4 * (2 * yr + kb + q);
                uint32_t v[4];
                window_chunk<1>(win, rp, q, v);
                if (pos >= 0 && pos + 4 <= p.out_width) {
                    if (q == 1 && rho && yr == G::NRY - 1) store_chunk_head<1>(row + pos, v, rho);
                    else *reinterpret_cast<uint4 *>(row + pos) = make_uint4(v[0], v[1], v[2], v[3]);
                }
            }
            if (yr == 0 && rho && A >= 0 && A + 4 <= p.out_width) {
                // tile elements [0, 4 - rho) fill positions [rho, 4) of chunk A (the previous tile
                // wrote the others)
                uint32_t tw[NW + 4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int i = 0; i < NW; ++i) tw[4 + i] = win[i];
                uint32_t v[4];
                window_chunk<1>(tw, rp, 0, v);
                store_chunk_tail<1>(row + A, v, 4 - rho);
            }
        }
    }
}

}  // namespace d3
