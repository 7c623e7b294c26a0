// k_small.cu -- the batched small-cube DRT (the paper's real-time case,
// PAPER.md:670): every stage of one (cube, dodecant) instance at N = 32 runs on
// chip, in one thread-block cluster, so HBM sees only the cube (read once per instance from L2)
// and the stacked output -- no intermediate stage buffer.
//
// N = 32 is n = 5 stages, split as in make_plan into a radix-8 pass (stages 0..2, K = 3) and a
// radix-4 pass (stages 3..4, K = 2), each a direct sum by the pass identity of drt_kernels.cuh
// (DESIGN.md §5):
//   phase 1, column block V = (V1, V2) (8 x 8 columns), slope r = (r1, r2) in 8 x 8:
//     f3(r | V)[z] = sum_{w1,w2 < 8} f(8 V1 + w1, 8 V2 + w2, z + l^3_{r1}(w1) + l^3_{r2}(w2)),
//   phase 2, slope group sigma (= the phase-1 r), final slope s = 4 sigma + rho:
//     out(s)[z] = sum_{V1,V2 < 4} f3(sigma | V)[z + sigma1 V1 + sigma2 V2 + l^2_{rho1}(V1) + l^2_{rho2}(V2)],
// with D = z + 2N (Alg. 1's displacement, eq:map3D PAPER.md:213-227, eq:3DfDRT PAPER.md:193-198).
//
// Phase 1 is an all-to-all into phase 2 (every column block feeds every slope group), so one
// instance is a cluster of 8 CTAs exchanging through distributed shared memory: CTA q computes
// column blocks 2q, 2q+1 and owns the slope groups sigma1 = q (8 groups x 16 rows).  Each f3 row
// is written straight into its owner's shared memory as aligned 16-byte chunks (realigned with
// one warp shuffle), at a residual shift that makes the runtime part of the phase-2 offsets,
// sigma1 V1 + sigma2 V2, a whole number of chunks: phase 2 adds a per-row chunk offset to its
// shared-memory addresses and keeps compile-time register offsets for the rest.  Both phases are
// separable direct sums (x-step then y-step) over register-blocked runs of R outputs on 32-bit
// lanes: integer sums mod 2^32, or fp32.
#include <cooperative_groups.h>

#include "dispatch.h"

namespace cg = cooperative_groups;

namespace d3 {
namespace small32 {

constexpr int N = 32, CL = 8, THREADS = 256;
// ---- phase 1: one column block at a time (two per CTA), 64 slots (w1, w2) of SP1 bytes; slot
// element e holds z' = e - 16.  The x-step output X covers e in [0, 56) (14 runs of R1 = 4), f3
// e in [0, 48) (12 runs): z in [-16, 32) -- f3 vanishes below z = -14, the support start of
// stage 3.
constexpr int R1 = 4, NB = 16 / CL, NRX1 = 14, NRY1 = 12;
constexpr int SP1 = 64 * 4 + 16;              // 64 staged words (X needs 56); +16 rotates banks
constexpr int SMA = NB * 64 * SP1;            // area A: phase-1 staging (both blocks), later phase-2 X2 rows
// ---- phase 2 input, area B: 8 groups (sigma2) x 16 rows (V = 4 V1 + V2) of 14 chunks.  Row
// (sigma, V) stores f3(sigma | V)[z] at element k = z + 16 + shift, shift = A - u in [0, 4),
// u = 16 + zb + sigma1 V1 + sigma2 V2, A = 4 ceil(u / 4), zb = -(4 sigma1 + 4 sigma2 + 8): the
// reader of output element p (z = zb + p) then needs element p + l + A, i.e. chunk offset A / 4.
// Chunks outside [0, 14) read as zero (one zero chunk).
constexpr int NCHB = 14, RB = NCHB * 16 + 16;
constexpr int SMB = 8 * 16 * RB;
// ---- phase 2: group sigma = (q, g) has the output window z in [zb, 32), Wout = 40 + 4 (q + g)
// <= 96 elements, D = p + 56 - 4 (q + g) (a multiple of 4: 16-byte stores); X2 rows (rho1, V2)
// in area A, two groups at a time.
constexpr int R2 = 8, NRX2 = 13, NRY2 = 12;   // runs for the widest group (Wout = 96, +3 halo)
constexpr int SPX = 104 * 4 + 16;
constexpr int GP = 4;                         // phase-2 groups at a time
static_assert(GP * 16 * SPX <= SMA, "X2 rows of GP groups fit area A");
constexpr int SMEM = SMA + SMB + 16;

// acc[r][j] += sum_a row_a[c0 chunks + co[a] chunks + j + l^K_r(a)] over the S rows `row[a]` of
// area B (NCHB chunks each, XOR-swizzled); chunks outside [0, NCHB) read the zero chunk.
template <int K, int R, class Acc>
__device__ __forceinline__ void acc_rows_b(const unsigned char *const (&row)[1 << K], const int (&co)[1 << K], int c0,
                                           const unsigned char *zero, uint32_t one, Acc (&acc)[1 << K][R]) {
    constexpr int S = 1 << K;
    auto load = [&](int a, int ne, uint32_t *buf) {
#pragma unroll
        for (int i = 0; i < (ne + 3) / 4; ++i) {
            const int c = co[a] + c0 + i;
            const unsigned char *src = (unsigned)c < (unsigned)NCHB ? row[a] + 16 * xswz(c) : zero;
            const uint4 v = *reinterpret_cast<const uint4 *>(src);
            buf[4 * i + 0] = v.x;
            if (4 * i + 1 < ne) buf[4 * i + 1] = v.y;
            if (4 * i + 2 < ne) buf[4 * i + 2] = v.z;
            if (4 * i + 3 < ne) buf[4 * i + 3] = v.w;
        }
    };
    static_for<0, S / 2>([&](auto p_) {
        constexpr int a0 = 2 * decltype(p_)::value, a1 = a0 + 1;
        uint32_t b0[R + a0], b1[R + a1];
        load(a0, R + a0, b0);
        load(a1, R + a1, b1);
        static_for<0, S>([&](auto r_) {
            constexpr int r = decltype(r_)::value;
            constexpr int o0 = lk(K, r, a0), o1 = lk(K, r, a1);
#pragma unroll
            for (int j = 0; j < R; ++j) acc[r][j] = add2<Acc>(acc[r][j], b0[j + o0], b1[j + o1], one, (r & 3) == 0);
        });
    });
}

template <class In, class Acc>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(THREADS, 3)
drt_small32_kernel(const DrtPass p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *smA = smem_raw, *smB = smem_raw + SMA, *zero = smem_raw + SMA + SMB;
    cg::cluster_group cluster = cg::this_cluster();
    const int q = (int)cluster.block_rank();                 // owns sigma1 = q
    const int li = blockIdx.x / CL;                          // instance of this launch
    const int inst = p.inst0 + li;
    const int tid = threadIdx.x;
    const Orient o = p.ori[inst % p.ndod];
    const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;

    // stage-0 rows of column block b into area A: slot (w1, w2), chunk c holds z' = 4 (c - 4) .. + 3
    // (zeros outside the cube); orientation as an index remap (reading A)
    auto stage = [&]() {
        for (int it = tid; it < NB * 64 * 16; it += THREADS) {
            const int slot = it >> 4, c = it & 15, w1 = (slot >> 3) & 7, w2 = slot & 7;
            const int b = NB * q + (slot >> 6), V1 = b >> 2, V2 = b & 3;
            uint32_t v[4] = {0u, 0u, 0u, 0u};
            if (c >= 4 && c < 12) {
                const int z4 = 4 * (c - 4);
                const long long base = o.off0 + (long long)(8 * V1 + w1) * o.sx + (long long)(8 * V2 + w2) * o.sy;
                if (o.fast == 2) {
                    // z' contiguous: the 4 voxels are one aligned vector (reversed axis: reversed order)
                    const In *src = cube + base + (o.sz > 0 ? (long long)z4 : -(long long)(z4 + 3));
                    uint32_t t[4];
                    if constexpr (sizeof(In) == 1) {
                        const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(src));
#pragma unroll
                        for (int k = 0; k < 4; ++k) t[k] = (w >> (8 * k)) & 0xFFu;
                    } else {
                        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(src));
                        t[0] = w.x; t[1] = w.y; t[2] = w.z; t[3] = w.w;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[k] = o.sz > 0 ? t[k] : t[3 - k];
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[k] = Elem<In>::load_bits(cube + base + (long long)(z4 + k) * o.sz);
                }
            }
            *reinterpret_cast<uint4 *>(smA + slot * SP1 + 16 * xswz(c)) = make_uint4(v[0], v[1], v[2], v[3]);
        }
    };

    // zero area B (f3 rows land on part of it) and the zero chunk; stage block 0; then a cluster
    // barrier: every CTA of the cluster has started and zeroed before any remote write
    for (int i = tid; i < SMB / 16 + 1; i += THREADS) reinterpret_cast<uint4 *>(smB)[i] = make_uint4(0u, 0u, 0u, 0u);
    stage();
    cluster.sync();

    Acc acc[8][R1];
    {
        // x-step: task (blk, w2, run) -> X(r1, w2) for all 8 r1, written in place over slot (r1, w2)
        {
            const int blk = tid / (8 * NRX1), rest = tid % (8 * NRX1), w2 = rest / NRX1, run = rest % NRX1;
            const bool act = tid < NB * 8 * NRX1;
            unsigned char *base = smA + blk * 64 * SP1;
            if (act) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < R1; ++j) acc[i][j] = Acc(0);
                drt_accumulate<3, R1, SP1, false, Acc>(base, w2, 8, run, p.one, acc);
            }
            __syncthreads();
            if (act) {
#pragma unroll
                for (int r1 = 0; r1 < 8; ++r1)
                    *reinterpret_cast<uint4 *>(base + (r1 * 8 + w2) * SP1 + 16 * xswz(run)) =
                        make_uint4(Lane<Acc>::bits(acc[r1][0]), Lane<Acc>::bits(acc[r1][1]),
                                   Lane<Acc>::bits(acc[r1][2]), Lane<Acc>::bits(acc[r1][3]));
            }
            __syncthreads();
        }
        // y-step: task (blk, r1, run), 16 lanes per r1 (12 active) -> f3(r1, r2 | V) for all 8 r2, sent
        // to CTA r1 as chunks: lane `run` holds f3 elements e = 4 run .. + 3, which land at k = e + shift
        {
            const int blk = tid >> 7, r1 = (tid >> 4) & 7, run = tid & 15;
            const int b = NB * q + blk, V1 = b >> 2, V2 = b & 3;
            const bool act = run < NRY1;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < R1; ++j) acc[i][j] = Acc(0);
            if (act) drt_accumulate<3, R1, SP1, false, Acc>(smA + blk * 64 * SP1, r1 * 8, 1, run, p.one, acc);
            unsigned char *dst = cluster.map_shared_rank(smB, r1) + (V1 * 4 + V2) * RB;
#pragma unroll
            for (int r2 = 0; r2 < 8; ++r2) {
                uint32_t w[7];
#pragma unroll
                for (int i = 0; i < 4; ++i) w[i] = Lane<Acc>::bits(acc[r2][i]);
#pragma unroll
                for (int i = 0; i < 3; ++i) w[4 + i] = __shfl_down_sync(0xffffffffu, w[i], 1, 16);
                if (!act) continue;
                if (run == NRY1 - 1) w[4] = w[5] = w[6] = 0u;        // past e = 48: zeros
                const int u = 8 - r1 * (4 - V1) - r2 * (4 - V2);
                const int shift = (4 - (u & 3)) & 3;
                unsigned char *row = dst + r2 * 16 * RB;
                if (shift == 0) {
                    *reinterpret_cast<uint4 *>(row + 16 * xswz(run)) = make_uint4(w[0], w[1], w[2], w[3]);
                } else {
                    // chunk run + 1 = elements 4 - shift .. of the window w (own tail, next lane's head)
                    uint32_t c[4];
                    const int s = 4 - shift;                                    // 1..3
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t a1 = (s & 1) ? w[i + 1] : w[i];
                        const uint32_t a3 = (s & 1) ? w[i + 3] : w[i + 2];
                        c[i] = (s & 2) ? a3 : a1;
                    }
                    *reinterpret_cast<uint4 *>(row + 16 * xswz(run + 1)) = make_uint4(c[0], c[1], c[2], c[3]);
                    if (run == 0) {
                        // chunk 0: `shift` zeros, then the first 4 - shift elements
                        uint32_t h[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int src = i - shift;
                            h[i] = src == 0 ? w[0] : src == 1 ? w[1] : src == 2 ? w[2] : 0u;
                        }
                        *reinterpret_cast<uint4 *>(row) = make_uint4(h[0], h[1], h[2], h[3]);
                    }
                }
            }
        }
    }
    cluster.sync();                                          // every f3 row has arrived

    // ---- phase 2: groups sigma = (q, g), GP at a time
    Acc *outp = reinterpret_cast<Acc *>(p.out) + (long long)inst * N * N * 3 * N;
    Acc acc2[4][R2];
    for (int g0 = 0; g0 < 8; g0 += GP) {
        {
            // x-step: task (group of the pair, V2, run) -> X2(rho1, V2), area A
            const int gp = tid / (4 * NRX2), rest = tid % (4 * NRX2), V2 = rest / NRX2, run = rest % NRX2;
            const int g = g0 + gp;
            const int wout = 40 + 4 * (q + g);
            if (tid < GP * 4 * NRX2 && R2 * run < wout + 3) {
                const unsigned char *rows[4];
                int co[4];
#pragma unroll
                for (int V1 = 0; V1 < 4; ++V1) {
                    const int u = 8 - q * (4 - V1) - g * (4 - V2);
                    co[V1] = (u + ((4 - (u & 3)) & 3)) >> 2;               // A / 4 (exact)
                    rows[V1] = smB + (g * 16 + V1 * 4 + V2) * RB;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < R2; ++j) acc2[i][j] = Acc(0);
                acc_rows_b<2, R2, Acc>(rows, co, 2 * run, zero, p.one, acc2);
                unsigned char *xb = smA + gp * 16 * SPX;
#pragma unroll
                for (int rho1 = 0; rho1 < 4; ++rho1)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        *reinterpret_cast<uint4 *>(xb + (rho1 * 4 + V2) * SPX + 16 * xswz(2 * run + h)) =
                            make_uint4(Lane<Acc>::bits(acc2[rho1][4 * h]), Lane<Acc>::bits(acc2[rho1][4 * h + 1]),
                                       Lane<Acc>::bits(acc2[rho1][4 * h + 2]), Lane<Acc>::bits(acc2[rho1][4 * h + 3]));
            }
            __syncthreads();
        }
        {
            // y-step: task (group of the pair, rho1, run) -> out(4q + rho1, 4g + rho2), rho2 = 0..3
            const int gp = tid / (4 * NRY2), rest = tid % (4 * NRY2), rho1 = rest / NRY2, run = rest % NRY2;
            const int g = g0 + gp;
            const int ssum = q + g, wout = 40 + 4 * ssum, dz = 56 - 4 * ssum;   // D of p = 0
            if (tid < GP * 4 * NRY2) {
                Acc *orow = outp + ((long long)(4 * q + rho1) * N + 4 * g) * (3 * N);
                if (R2 * run < wout) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < R2; ++j) acc2[i][j] = Acc(0);
                    drt_accumulate<2, R2, SPX, false, Acc>(smA + gp * 16 * SPX, rho1 * 4, 1, 2 * run, p.one, acc2);
                    const bool two = R2 * run + 4 < wout;              // wout is a multiple of 4, not of 8
#pragma unroll
                    for (int rho2 = 0; rho2 < 4; ++rho2) {
                        Acc *d = orow + rho2 * (3 * N) + dz + R2 * run;
                        st_cs_v4(d, Lane<Acc>::bits(acc2[rho2][0]), Lane<Acc>::bits(acc2[rho2][1]),
                                 Lane<Acc>::bits(acc2[rho2][2]), Lane<Acc>::bits(acc2[rho2][3]));
                        if (two)
                            st_cs_v4(d + 4, Lane<Acc>::bits(acc2[rho2][4]), Lane<Acc>::bits(acc2[rho2][5]),
                                     Lane<Acc>::bits(acc2[rho2][6]), Lane<Acc>::bits(acc2[rho2][7]));
                    }
                }
                // D below the group's window (below the support of every row): zeros
                for (int c = run; c < dz / 4; c += NRY2)
#pragma unroll
                    for (int rho2 = 0; rho2 < 4; ++rho2) st_cs_v4(orow + rho2 * (3 * N) + 4 * c, 0u, 0u, 0u, 0u);
            }
            __syncthreads();                                 // area A is rewritten by the next pair
        }
    }
}

template <class In, class Acc>
drt3d_status launch(const DrtPass &prm, int ninst, cudaStream_t st) {
    auto kern = drt_small32_kernel<In, Acc>;
    static std::atomic<uint32_t> smem_done{0};
    if (!set_smem_once(kern, SMEM, smem_done)) return DRT3D_ERR_CUDA;
    kern<<<dim3((unsigned)(CL * ninst)), THREADS, SMEM, st>>>(prm);
    return DRT3D_OK;
}

}  // namespace small32

drt3d_status dispatch_drt_small32(int in_dtype, const DrtPass &prm, int ninst, cudaStream_t st) {
    if (prm.N != small32::N) return DRT3D_ERR_UNSUPPORTED;
    if (in_dtype == DRT3D_U8) return small32::launch<uint8_t, uint32_t>(prm, ninst, st);
    if (in_dtype == DRT3D_I32) return small32::launch<uint32_t, uint32_t>(prm, ninst, st);
    return small32::launch<float, float>(prm, ninst, st);
}

}  // namespace d3
