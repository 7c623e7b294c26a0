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
// is written straight into its owner's shared memory, pre-shifted by sigma1 V1 + sigma2 V2 (the
// runtime part of the phase-2 offsets), so phase 2's sums use compile-time register offsets
// only.  Both phases use drt_accumulate (separable x-step then y-step, register-blocked runs of
// R = 8 outputs) on 32-bit lanes: integer sums mod 2^32, or fp32.
#include <cooperative_groups.h>

#include "dispatch.h"

namespace cg = cooperative_groups;

namespace d3 {
namespace small32 {

constexpr int N = 32, CL = 8, R = 8, THREADS = 128;
// phase 1: a column block = 64 slots (w1, w2); slot element e holds z' = e - 16
// (the x-step output X covers e in [0, 56), f3 e in [0, 48): z in [-16, 32) -- f3 vanishes
// below z = -14, the support start of stage 3).
constexpr int E0 = 16;
constexpr int NB = 16 / CL;                   // column blocks per CTA
constexpr int NRX1 = 7, NRY1 = 6;
constexpr int SP1 = 64 * 4 + 16;              // 64 staged words (X needs 56); +16 rotates banks
constexpr int SM1 = NB * 64 * SP1;
// phase 2: 8 groups (sigma2) x 16 rows (V1, V2) of stored f3.  Stored element p of row
// (sigma, V) holds f3(sigma | V) at z = zb + p + sigma1 V1 + sigma2 V2, zb = -(4 sigma1 +
// 4 sigma2 + 8): the group's output window z in [zb, 32) has Wout = 40 + 4 (sigma1 + sigma2)
// <= 96 elements (D = p + 56 - 4 (sigma1 + sigma2), a multiple of 4: 16-byte stores).
constexpr int NRX2 = 13, NRY2 = 12;           // runs for the widest group (Wout = 96, +3 halo)
constexpr int SP2 = 112 * 4 + 16;             // x-step reads < 108 elements, X2 is 104 words
constexpr int GROUP_BYTES = 16 * SP2;
constexpr int SM2 = 8 * GROUP_BYTES;
constexpr int SMEM = SM1 + SM2;

__device__ __forceinline__ int elem_off(int p) { return 16 * xswz(p >> 2) + 4 * (p & 3); }

template <class In, class Acc>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(THREADS)
drt_small32_kernel(const DrtPass p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm1 = smem_raw, *sm2 = smem_raw + SM1;
    cg::cluster_group cluster = cg::this_cluster();
    const int q = (int)cluster.block_rank();                 // owns sigma1 = q
    const int li = blockIdx.x / CL;                          // instance of this launch
    const int inst = p.inst0 + li;
    const int tid = threadIdx.x;

    // ---- zero this CTA's phase-2 rows (f3 lands on its support only), then a cluster barrier:
    // every CTA of the cluster has started and zeroed before any remote write
    for (int i = tid; i < SM2 / 16; i += THREADS) reinterpret_cast<uint4 *>(sm2)[i] = make_uint4(0u, 0u, 0u, 0u);

    // ---- phase 1 staging: slots (blk, w1, w2), stage-0 rows of column blocks 2q, 2q+1
    // (orientation as an index remap, reading A: element (x', y', z') at off0 + x' sx + y' sy + z' sz)
    {
        const Orient o = p.ori[inst % p.ndod];
        const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
        // item = (slot, chunk c of 16): chunks 4..11 hold z' = 4 (c - 4) .. + 3, the rest zeros
        for (int it = tid; it < NB * 64 * 16; it += THREADS) {
            const int slot = it >> 4, c = it & 15;
            const int blk = slot >> 6, w1 = (slot >> 3) & 7, w2 = slot & 7;
            const int b = NB * q + blk, V1 = b >> 2, V2 = b & 3;
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
            *reinterpret_cast<uint4 *>(sm1 + slot * SP1 + 16 * xswz(c)) = make_uint4(v[0], v[1], v[2], v[3]);
        }
    }
    cluster.sync();

    Acc acc[8][R], acc2[4][R];
    auto zero_acc = [&]() {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < R; ++j) acc[i][j] = Acc(0);
    };
    auto zero_acc2 = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < R; ++j) acc2[i][j] = Acc(0);
    };

    // ---- phase 1 x-step: task (blk, w2, run) -> X(r1, w2) for all 8 r1, written in place
    {
        const int blk = tid / (8 * NRX1), rest = tid % (8 * NRX1), w2 = rest / NRX1, run = rest % NRX1;
        const bool act = tid < NB * 8 * NRX1;
        unsigned char *base = sm1 + blk * 64 * SP1;
        if (act) {
            zero_acc();
            drt_accumulate<3, R, SP1, false, Acc>(base, w2, 8, 2 * run, p.one, acc);
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int r1 = 0; r1 < 8; ++r1)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    *reinterpret_cast<uint4 *>(base + (r1 * 8 + w2) * SP1 + 16 * xswz(2 * run + h)) =
                        make_uint4(Lane<Acc>::bits(acc[r1][4 * h]), Lane<Acc>::bits(acc[r1][4 * h + 1]),
                                   Lane<Acc>::bits(acc[r1][4 * h + 2]), Lane<Acc>::bits(acc[r1][4 * h + 3]));
        }
        __syncthreads();
    }
    // ---- phase 1 y-step: task (blk, r1, run) -> f3(r1, r2 | V) for all 8 r2, sent to CTA r1
    {
        const int blk = tid / (8 * NRY1), rest = tid % (8 * NRY1), r1 = rest / NRY1, run = rest % NRY1;
        if (tid < NB * 8 * NRY1) {
            const int b = NB * q + blk, V1 = b >> 2, V2 = b & 3;
            zero_acc();
            drt_accumulate<3, R, SP1, false, Acc>(sm1 + blk * 64 * SP1, r1 * 8, 1, 2 * run, p.one, acc);
            unsigned char *dst = cluster.map_shared_rank(sm2, r1) + (V1 * 4 + V2) * SP2;
#pragma unroll
            for (int r2 = 0; r2 < 8; ++r2) {
                // p = e - 8 + r1 (4 - V1) + r2 (4 - V2) >= 0 wherever f3 can be non-zero (z >= -(r1 + r2))
                const int p0 = R * run - 8 + r1 * (4 - V1) + r2 * (4 - V2);
                unsigned char *row = dst + r2 * GROUP_BYTES;
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (p0 + j >= 0) *reinterpret_cast<uint32_t *>(row + elem_off(p0 + j)) = Lane<Acc>::bits(acc[r2][j]);
            }
        }
    }
    cluster.sync();                                          // every f3 row has arrived

    // ---- phase 2: groups sigma = (q, g), two at a time (task = (group of the pair, V2 | rho1, run))
    Acc *outp = reinterpret_cast<Acc *>(p.out) + (long long)inst * N * N * 3 * N;
    for (int g0 = 0; g0 < 8; g0 += 2) {
        {
            const int gp = tid / (4 * NRX2), rest = tid % (4 * NRX2), V2 = rest / NRX2, run = rest % NRX2;
            const int g = g0 + gp;
            const int wout = 40 + 4 * (q + g);
            const bool act = tid < 2 * 4 * NRX2 && R * run < wout + 3;
            unsigned char *base = sm2 + g * GROUP_BYTES;
            if (act) {
                zero_acc2();
                drt_accumulate<2, R, SP2, false, Acc>(base, V2, 4, 2 * run, p.one, acc2);
            }
            __syncthreads();
            if (act) {
#pragma unroll
                for (int rho1 = 0; rho1 < 4; ++rho1)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        *reinterpret_cast<uint4 *>(base + (rho1 * 4 + V2) * SP2 + 16 * xswz(2 * run + h)) =
                            make_uint4(Lane<Acc>::bits(acc2[rho1][4 * h]), Lane<Acc>::bits(acc2[rho1][4 * h + 1]),
                                       Lane<Acc>::bits(acc2[rho1][4 * h + 2]), Lane<Acc>::bits(acc2[rho1][4 * h + 3]));
            }
            __syncthreads();
        }
        {
            const int gp = tid / (4 * NRY2), rest = tid % (4 * NRY2), rho1 = rest / NRY2, run = rest % NRY2;
            const int g = g0 + gp;
            const int ssum = q + g, wout = 40 + 4 * ssum, dz = 56 - 4 * ssum;   // D of stored p = 0
            if (tid < 2 * 4 * NRY2) {
                const int s1 = 4 * q + rho1;
                Acc *orow = outp + ((long long)s1 * N + 4 * g) * (3 * N);
                if (R * run < wout) {
                    zero_acc2();
                    drt_accumulate<2, R, SP2, false, Acc>(sm2 + g * GROUP_BYTES, rho1 * 4, 1, 2 * run, p.one, acc2);
                    const bool two = R * run + 4 < wout;                // wout is a multiple of 4, not of 8
#pragma unroll
                    for (int rho2 = 0; rho2 < 4; ++rho2) {
                        Acc *d = orow + rho2 * (3 * N) + dz + R * run;
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
