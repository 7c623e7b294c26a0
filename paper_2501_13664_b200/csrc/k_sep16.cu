// k_sep16.cu -- the DRT at N = 16 with every stage of one (cube, dodecant) instance in one CTA
// (SURVEY §8 rows A-1..A-6 at BASELINE cfg1's size, and A-10 for batches of N = 16 cubes).
//
// The separable form of k_sep32.cu: a digital plane is the sum of two digital lines
// (eq:3DfDRT; eq:digitalLine PAPER.md:133-137), so
//
//   out(s1, s2)[D] = sum_y P(s1, y)[D - 2N + l^4_{s2}(y)],   P(s1, y)[t] = sum_x f(x, y, t + l^4_{s1}(x)),
//
// and by the pass identity (c = 2, K = 2) l^4_{4 sig + rho}(4 V + w) = l^2_sig(w) + sig V + l^2_rho(V)
// each factor is two radix-4 steps:
//
//   X1  Q(sig1, V1, y)[t]      = sum_{w1 < 4} f(4 V1 + w1, y, t + l^2_{sig1}(w1))
//   X2  P(4 sig1 + rho1, y)[t] = sum_{V1 < 4} Q(sig1, V1, y)[t + sig1 V1 + l^2_{rho1}(V1)]
//   Y1  U(s1; sig2, V2)[t]     = sum_{w2 < 4} P(s1, 4 V2 + w2)[t + l^2_{sig2}(w2)]
//   Y2  out(s1, 4 sig2 + rho2)[D] = sum_{V2 < 4} U(s1; sig2, V2)[D - 2N + sig2 V2 + l^2_{rho2}(V2)]
//
// f is the oriented cube (Alg. 2 permute/flip as an index remap), D = z + 2N
// (eq:map3D).  At N = 16 everything fits one CTA (92 KB, two CTAs per SM): one
// launch per call, no stage buffer, HBM sees the cube and the stacked output only.
#include "dispatch.h"
#include "sep_common.cuh"

namespace d3 {
namespace sep16 {
using namespace sep;

constexpr int N = 16, R = 4;
// Shared memory, 16-byte chunks; odd row pitches keep lanes on consecutive rows conflict-free.
//  A: cube rows (x', y') = 16 x' + y' of 9 chunks: z' = 4c .. 4c + 3 (c in [0, 4)) at chunk c + 1,
//     zero chunks at c = -1, 4, 5 (X1 reads z' in [-4, 24)); after X1, U rows
//     ((s1 * 4 + sig2) * 4 + V2) of 9 chunks, u = t + 20 in [0, 36)
//  B: Q rows ((sig1 * 4 + V1) * 16 + y) of 5 chunks, q = t + 4 in [0, 20)
//  C: P rows (s1 * 16 + y) of 9 chunks (8 used), p = t + 16 in [0, 32)
constexpr int AP = 9, QP = 5, PP = 9;
constexpr int SMA = 256 * AP * 16, SMB = 256 * QP * 16, SMC = 256 * PP * 16;
constexpr int SMEM = SMA + SMB + SMC + 16;                // + one zero chunk

// THREADS: 256 (two CTAs per SM); the loops are written for any block size
template <class In, class Acc, int THREADS>
__global__ void __launch_bounds__(THREADS, THREADS <= 256 ? 2 : 1) drt_sep16_kernel(const DrtPass p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *smA = smem_raw, *smB = smem_raw + SMA, *smC = smem_raw + SMA + SMB, *zero = smC + SMC;
    const int inst = p.inst0 + blockIdx.x;
    const int tid = threadIdx.x;
    const Orient o = p.ori[inst % p.ndod];
    const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
    auto cube_chunk = [&](int row, int c) -> unsigned char * { return smA + (row * AP + c + 1) * 16; };
    if (tid == 0) *reinterpret_cast<uint4 *>(zero) = make_uint4(0u, 0u, 0u, 0u);
#if D3_PDL
    // the next launch on the stream may be scheduled now (programmatic dependent launch)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif

    // ---- stage the oriented cube: f(x', y', z') = cube[off0 + x' sx + y' sy + z' sz]
    for (int i = tid; i < 256 * 3; i += THREADS) {           // zero chunks -1, 4, 5 of every row
        const int row = i / 3, c = i - 3 * row;
        *reinterpret_cast<uint4 *>(cube_chunk(row, c == 0 ? -1 : c + 3)) = make_uint4(0u, 0u, 0u, 0u);
    }
    if (o.fast == 2) {
        // z' along the unit-stride axis: one vector load = one chunk (reversed axis: reversed order)
        constexpr int IT = (1024 + THREADS - 1) / THREADS;
        uint32_t v[IT][4];
#pragma unroll
        for (int u = 0; u < IT; ++u) {
            const int it = tid + u * THREADS, row = (it & 1023) >> 2, c = it & 3;
            const long long base = o.off0 + (long long)(row >> 4) * o.sx + (long long)(row & 15) * o.sy;
            load4<In>(cube + base + (o.sz > 0 ? 4 * c : -(4 * c + 3)), v[u]);
        }
#pragma unroll
        for (int u = 0; u < IT; ++u) {
            const int it = tid + u * THREADS, row = it >> 2, c = it & 3;
            if (it >= 1024) break;
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = o.sz > 0 ? v[u][q] : v[u][3 - q];
            *reinterpret_cast<uint4 *>(cube_chunk(row, c)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    } else {
        // x' (fast 0) or y' (fast 1) along the unit-stride axis: 4 loads at z' = 4c .. 4c + 3 of 4
        // consecutive coordinates 4g .. 4g + 3 of that axis, transposed in registers into 4 chunks
        const bool fy = o.fast == 1;
        const long long sf = fy ? o.sy : o.sx, so = fy ? o.sx : o.sy;
        for (int it = tid; it < 256; it += THREADS) {
            const int other = it >> 4, g = (it >> 2) & 3, c = it & 3;
            const long long base = o.off0 + (long long)other * so + (sf > 0 ? 4 * g : -(4 * g + 3));
            uint32_t v[4][4];
#pragma unroll
            for (int t = 0; t < 4; ++t) load4<In>(cube + base + (long long)(4 * c + t) * o.sz, v[t]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int jj = sf > 0 ? j : 3 - j;
                const int row = fy ? other * 16 + 4 * g + j : (4 * g + j) * 16 + other;
                *reinterpret_cast<uint4 *>(cube_chunk(row, c)) = make_uint4(v[0][jj], v[1][jj], v[2][jj], v[3][jj]);
            }
        }
    }
    __syncthreads();

    // ---- X1: task (V1, run, y), lanes on y; Q(sig1, V1, y)[q = 4 run + j], q = t + 4 in [0, 20):
    // f at z' = q - 4 + l^2_sig1(w1) (cube chunks run - 1 .., zero chunks outside 0..3)
    for (int t = tid; t < 4 * 5 * 16; t += THREADS) {
        const int y = t & 15, vr = t >> 4, V1 = vr / 5, run = vr - 5 * V1;
        Acc acc[4][R];
        radix4<0, R, Acc>([&](int w1, int c) -> const unsigned char * { return cube_chunk((4 * V1 + w1) * 16 + y, c); },
                          run - 1, p.one, acc);
#pragma unroll
        for (int s = 0; s < 4; ++s)
            *reinterpret_cast<uint4 *>(smB + (((s * 4 + V1) * 16 + y) * QP + run) * 16) =
                make_uint4(Lane<Acc>::bits(acc[s][0]), Lane<Acc>::bits(acc[s][1]), Lane<Acc>::bits(acc[s][2]),
                           Lane<Acc>::bits(acc[s][3]));
    }
    __syncthreads();

    // ---- X2: task (sig1, run, y), each warp on one sig1; P(4 sig1 + rho1, y)[p = 4 run + j],
    // p = t + 16 in [0, 32): Q at q = p - 12 + sig1 V1 + l^2_rho1(V1) (chunks run - 3 + .., valid 0..4)
    for (int t = tid; t < 4 * 8 * 16; t += THREADS) {
        const int y = t & 15, run = (t >> 4) & 7, sig1 = t >> 7;
        Acc acc[4][R];
        if (4 * run + 4 > N - (4 * sig1 + 3)) {              // else below the support of all 4 slopes
            auto rc = [&](int V1, int c) -> const unsigned char * {
                return (unsigned)c < (unsigned)QP ? smB + (((sig1 * 4 + V1) * 16 + y) * QP + c) * 16 : zero;
            };
            with_const8<0>(sig1, [&](auto S_) {
                constexpr int SG = decltype(S_)::value;
                if constexpr (SG < 4) radix4<SG, R, Acc>(rc, run - 3, p.one, acc);
            });
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < R; ++j) acc[i][j] = Acc(0);
        }
#pragma unroll
        for (int rho = 0; rho < 4; ++rho)
            *reinterpret_cast<uint4 *>(smC + (((4 * sig1 + rho) * 16 + y) * PP + run) * 16) =
                make_uint4(Lane<Acc>::bits(acc[rho][0]), Lane<Acc>::bits(acc[rho][1]), Lane<Acc>::bits(acc[rho][2]),
                           Lane<Acc>::bits(acc[rho][3]));
    }
    __syncthreads();

    // ---- Y1: task (s1, V2, run), lanes on run; U(s1; sig2, V2)[u = 4 run + j], u = t + 20 in [0, 36):
    // P(s1, 4 V2 + w2) at p = u - 4 + l^2_sig2(w2) (chunks run - 1 + .., valid 0..7)
    for (int t = tid; t < 16 * 4 * 9; t += THREADS) {
        const int rest = t / 9, run = t - 9 * rest, V2 = rest & 3, s1 = rest >> 2;
        Acc acc[4][R];
        radix4<0, R, Acc>([&](int w2, int c) -> const unsigned char * {
            return (unsigned)c < 8u ? smC + ((s1 * 16 + 4 * V2 + w2) * PP + c) * 16 : zero;
        }, run - 1, p.one, acc);
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2)
            *reinterpret_cast<uint4 *>(smA + (((s1 * 4 + s2) * 4 + V2) * AP + run) * 16) =
                make_uint4(Lane<Acc>::bits(acc[s2][0]), Lane<Acc>::bits(acc[s2][1]), Lane<Acc>::bits(acc[s2][2]),
                           Lane<Acc>::bits(acc[s2][3]));
    }
    __syncthreads();

    // ---- Y2: task (sig2, s1, run), each warp on one sig2 (192 tasks = 6 warps per sig2);
    // out(s1, 4 sig2 + rho2)[D = 4 run + j]: U at u = D - 12 + sig2 V2 + l^2_rho2(V2)
    // (chunks run - 3 + .., valid 0..8)
    Acc *outp = reinterpret_cast<Acc *>(p.out) + (long long)inst * N * N * 3 * N;
    for (int t = tid; t < 4 * 16 * 12; t += THREADS) {
        const int sig2 = t / 192, rest = t - 192 * sig2, s1 = rest / 12, run = rest - 12 * s1;
        Acc acc[4][R];
        if (4 * run + 4 > 2 * N - s1 - (4 * sig2 + 3)) {
            auto rc = [&](int V2, int c) -> const unsigned char * {
                return (unsigned)c < 9u ? smA + (((s1 * 4 + sig2) * 4 + V2) * AP + c) * 16 : zero;
            };
            with_const8<0>(sig2, [&](auto S_) {
                constexpr int SG = decltype(S_)::value;
                if constexpr (SG < 4) radix4<SG, R, Acc>(rc, run - 3, p.one, acc);
            });
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < R; ++j) acc[i][j] = Acc(0);
        }
        Acc *orow = outp + ((long long)s1 * N + 4 * sig2) * (3 * N) + 4 * run;
#pragma unroll
        for (int rho = 0; rho < 4; ++rho)
            st_cs_v4(orow + rho * (3 * N), Lane<Acc>::bits(acc[rho][0]), Lane<Acc>::bits(acc[rho][1]),
                     Lane<Acc>::bits(acc[rho][2]), Lane<Acc>::bits(acc[rho][3]));
    }
}

template <class In, class Acc, int THREADS>
drt3d_status launch_t(const DrtPass &prm, int ninst, cudaStream_t st) {
    auto kern = drt_sep16_kernel<In, Acc, THREADS>;
    static std::atomic<uint32_t> smem_done{0};
    if (!set_smem_once(kern, SMEM, smem_done)) return DRT3D_ERR_CUDA;
    kern<<<dim3((unsigned)ninst), THREADS, SMEM, st>>>(prm);
    return DRT3D_OK;
}
// 256 threads (two CTAs per SM).  Measured: 768 threads for up to one instance per SM (every phase
// one round of tasks) does not shorten the single-instance call (cfg1 0.0102 vs 0.0092 ms).
template <class In, class Acc>
drt3d_status launch(const DrtPass &prm, int ninst, cudaStream_t st) {
    return launch_t<In, Acc, 256>(prm, ninst, st);
}

}  // namespace sep16

drt3d_status dispatch_drt_sep16(int in_dtype, const DrtPass &prm, int ninst, cudaStream_t st) {
    if (prm.N != sep16::N) return DRT3D_ERR_UNSUPPORTED;
    if (in_dtype == DRT3D_U8) return sep16::launch<uint8_t, uint32_t>(prm, ninst, st);
    if (in_dtype == DRT3D_I32) return sep16::launch<uint32_t, uint32_t>(prm, ninst, st);
    return sep16::launch<float, float>(prm, ninst, st);
}

}  // namespace d3
