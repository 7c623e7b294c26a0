// k_sep32.cu -- the batched small-cube DRT at N = 32 (the paper's real-time
// case), every stage on chip: one 4-CTA cluster per instance, one
// exchange of x-partial sums through distributed shared memory, no stage buffer in HBM.
//
// The digital plane of slope (s1, s2) is the sum of two digital lines (eq:3DfDRT, PAPER.md:193-198,
// with eq:digitalLine PAPER.md:133-137), so the transform is separable:
//
//   out(s1, s2)[D] = sum_y P(s1, y)[D - 2N + l^n_{s2}(y)],   P(s1, y)[t] = sum_x f(x, y, t + l^n_{s1}(x)),
//
// f the oriented cube (Alg. 2 permute/flip as an index remap) and D = z + 2N
// (Alg. 1's displacement, eq:map3D PAPER.md:213-227).  Each direction is the recursion of Alg. 1
// restricted to one axis, regrouped (DESIGN.md §5 "Pass identity" with c = 3, K = 2) through
//   l^5_{4 sig + rho}(8 V + w) = l^3_sig(w) + sig V + l^2_rho(V):
//
//   X1  Q(sig1, V1, y)[t]      = sum_{w1 < 8} f(8 V1 + w1, y, t + l^3_{sig1}(w1))          (radix 8)
//   X2  P(4 sig1 + rho1, y)[t] = sum_{V1 < 4} Q(sig1, V1, y)[t + sig1 V1 + l^2_{rho1}(V1)] (radix 4)
//   Y1  U(s1; sig2, V2)[t]     = sum_{w2 < 8} P(s1, 8 V2 + w2)[t + l^3_{sig2}(w2)]           (radix 8)
//   Y2  out(s1, 4 sig2 + rho2)[D] = sum_{V2 < 4} U(s1; sig2, V2)[D - 2N + sig2 V2 + l^2_{rho2}(V2)]
//
// CTA k of the cluster stages the oriented slab x' in [8k, 8k + 8) (32 KB as 32-bit lanes) and runs
// X1 for all 8 sig1 on it; each Q row goes (16-byte stores, local or remote) to the CTA that owns
// sig1, CTA sig1 / 2.  After one cluster barrier CTA k holds Q(sig1 in {2k, 2k+1}, all V1) and
// finishes the slopes s1 in [8k, 8k + 8) alone: X2, then Y1 / Y2 for 4 slopes at a time.  Shared
// memory: Q 44 KB | slab 52 KB -> P 64 KB; U (4 slopes, 38 KB) over Q -- 108 KB, two CTAs per SM.
// The sums are direct register-blocked sums (compile-time offsets l^K_r(w) as register indices,
// runs of R = 8 outputs, rows two at a time: IADD3 for integer lanes, exact mod 2^32).
#include <cooperative_groups.h>

#include "dispatch.h"
#include "sep_common.cuh"

namespace cg = cooperative_groups;

namespace d3 {
namespace sep32 {
using namespace sep;

constexpr int N = 32, CL = 4, THREADS = 256, R = 8;
// -DD3_SEP_ABL=mask (ablation builds, wrong results): 1 no Y2 stores, 2 no remote Q stores,
// 4 no y part, 8 no x part
#ifndef D3_SEP_ABL
#define D3_SEP_ABL 0
#endif

// -DD3_PROF_SEP32: per-phase clock accounting (lane 0 of warps 0 and 7) into d3_sep_prof[]
#ifdef D3_PROF_SEP32
__device__ unsigned long long d3_sep_prof[32];
#define SP_MARK(i) sp_t[i] = clock64()
#else
#define SP_MARK(i)
#endif
// region Q (offset 0): rows (sl * 4 + V1) * 32 + y (sl = sig1 & 1) of QP chunks, q = t + 8 in
// [0, 40) (10 chunks; the odd pitch keeps lanes on consecutive y conflict-free)
constexpr int QP = 11, QCH = 10;
constexpr int SMQ = 2 * 4 * 32 * QP * 16;
// region S/P (offset SMQ): slab rows w1 * 32 + y of SLP chunks (z' = 4c .. 4c + 3 for c in [0, 8) at
// c + 2, zero chunks at -2, -1, 8, 9; the odd pitch keeps lanes on consecutive y conflict-free);
// after X1, P rows s1l * 32 + y (s1 = 8k + s1l) of 16 chunks, p = t + 32 in [0, 64), chunk c at
// pswz(c, y) = (c + y) mod 16 (lanes on consecutive y at one chunk, and lanes on consecutive chunks of
// one row, are both conflict-free)
constexpr int SLP = 13;
constexpr int SMP = 8 * 32 * 16 * 16;
static_assert(8 * 32 * SLP * 16 <= SMP, "padded slab fits region P");
// region U (offset 0, over Q after X2): rows (sb * 8 + sig2) * 4 + V2 of UP chunks, u = t + 40 in
// [0, 72) (18 chunks; lanes on consecutive runs touch chunks 1 or 3 apart: conflict-free unswizzled);
// sb = s1l - 4 b for the slopes of batch b
constexpr int UP = 19, UCH = 18;
static_assert(4 * 8 * 4 * UP * 16 <= SMQ, "U rows of 4 slopes fit region Q");
constexpr int ZB = 3 * N * 4;                  // zero region: one output row (the first chunk = the zero chunk)
constexpr int SMEM = SMQ + SMP + ZB;

__device__ __forceinline__ int pswz(int c, int y) { return (c + y) & 15; }

template <class Acc>
__device__ __forceinline__ void put_run(unsigned char *row, int c0, const Acc (&a)[R]) {
    *reinterpret_cast<uint4 *>(row + 16 * c0) =
        make_uint4(Lane<Acc>::bits(a[0]), Lane<Acc>::bits(a[1]), Lane<Acc>::bits(a[2]), Lane<Acc>::bits(a[3]));
    *reinterpret_cast<uint4 *>(row + 16 * (c0 + 1)) =
        make_uint4(Lane<Acc>::bits(a[4]), Lane<Acc>::bits(a[5]), Lane<Acc>::bits(a[6]), Lane<Acc>::bits(a[7]));
}

template <class In, class Acc>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(THREADS, 2) drt_sep32_kernel(const DrtPass p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *smQ = smem_raw, *smP = smem_raw + SMQ, *zero = smem_raw + SMQ + SMP;
    cg::cluster_group cluster = cg::this_cluster();
    const int k = (int)cluster.block_rank();               // slab x' in [8k, 8k + 8); slopes s1 in [8k, 8k + 8)
    const int li = blockIdx.x / CL;
    const int inst = p.inst0 + li;
    const int tid = threadIdx.x;
    const Orient o = p.ori[inst % p.ndod];
    const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
    // slab row (w1, y) = w1 * 32 + y: chunk c in [-2, 10) at (c + 2) of SLP (z' = 4c .. 4c + 3; chunks
    // outside [0, 8) are zero)
    auto slab_chunk = [&](int row, int c) -> unsigned char * { return smP + (row * SLP + c + 2) * 16; };
#ifdef D3_PROF_SEP32
    long long sp_t[8];
#endif
    SP_MARK(0);
    if (tid < ZB / 16) {
        reinterpret_cast<uint4 *>(zero)[tid] = make_uint4(0u, 0u, 0u, 0u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");     // read by the bulk zero stores
    }
    // cluster barrier, phase 1: this CTA has started (its shared memory may receive remote stores);
    // the matching wait comes right before the first remote store (X1)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

    // ---- stage the oriented slab: f(x', y', z') = cube[off0 + x' sx + y' sy + z' sz], x' = 8k + w1
    for (int i = tid; i < 8 * 32 * 4; i += THREADS) {        // zero pads: chunks -2, -1, 8, 9 of every row
        const int row = i >> 2, c = i & 3;
        *reinterpret_cast<uint4 *>(slab_chunk(row, c < 2 ? c - 2 : c + 6)) = make_uint4(0u, 0u, 0u, 0u);
    }
    if (o.fast == 2) {
        // z' along the unit-stride axis: one vector load = one chunk (reversed axis: reversed order)
        constexpr int IT = 8;
        uint32_t v[IT][4];
#pragma unroll
        for (int u = 0; u < IT; ++u) {
            const int it = tid + u * THREADS, row = it >> 3, c = it & 7;
            const long long base = o.off0 + (long long)(8 * k + (row >> 5)) * o.sx + (long long)(row & 31) * o.sy;
            load4<In>(cube + base + (o.sz > 0 ? 4 * c : -(4 * c + 3)), v[u]);
        }
#pragma unroll
        for (int u = 0; u < IT; ++u) {
            const int it = tid + u * THREADS, row = it >> 3, c = it & 7;
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = o.sz > 0 ? v[u][q] : v[u][3 - q];
            *reinterpret_cast<uint4 *>(slab_chunk(row, c)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    } else {
        // x' (fast 0) or y' (fast 1) along the unit-stride axis: 4 loads at z' = 4c .. 4c + 3 of 4
        // consecutive coordinates 4g .. 4g + 3 of that axis, transposed in registers into 4 chunks
        const bool fy = o.fast == 1;
        const long long sf = fy ? o.sy : o.sx, so = fy ? o.sx : o.sy;
#ifndef D3_SEP_LD256
#define D3_SEP_LD256 1
#endif
        bool wide = false;
        if constexpr (D3_SEP_LD256 && sizeof(In) == 4) wide = (reinterpret_cast<unsigned long long>(cube) & 31ull) == 0;
        if (wide) {
            // 32-bit voxels: one 32-byte load (LDG.256) = 8 consecutive coordinates of the unit-stride
            // axis, half the load instructions and L1 wavefronts of the 16-byte version (every lane
            // reads its own line here); item (other, g2, c): coordinates 8 g2 .. 8 g2 + 7 at z' = 4c .. 4c + 3
            const int it = tid, c = it & 7;
            const int other = fy ? (it >> 5) : (it >> 3), g2 = fy ? ((it >> 3) & 3) : 0;
            const int f0 = fy ? 8 * g2 : 8 * k;
            const long long base = o.off0 + (long long)(fy ? 8 * k + other : other) * so + (sf > 0 ? f0 : -(f0 + 7));
            uint32_t v[4][8];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const In *src = cube + base + (long long)(4 * c + t) * o.sz;
                asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                             : "=r"(v[t][0]), "=r"(v[t][1]), "=r"(v[t][2]), "=r"(v[t][3]), "=r"(v[t][4]), "=r"(v[t][5]),
                               "=r"(v[t][6]), "=r"(v[t][7])
                             : "l"(src));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int jj = sf > 0 ? j : 7 - j;
                const int row = fy ? other * 32 + 8 * g2 + j : j * 32 + other;
                *reinterpret_cast<uint4 *>(slab_chunk(row, c)) = make_uint4(v[0][jj], v[1][jj], v[2][jj], v[3][jj]);
            }
        } else
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int it = tid + u * THREADS, c = it & 7;
            // fast 1: other = w1 (it >> 6), g = (it >> 3) & 7; fast 0: other = y (it >> 4), g = (it >> 3) & 1
            const int other = fy ? (it >> 6) : (it >> 4), g = fy ? ((it >> 3) & 7) : ((it >> 3) & 1);
            const int f0 = fy ? 4 * g : 8 * k + 4 * g;
            const long long base = o.off0 + (long long)(fy ? 8 * k + other : other) * so + (sf > 0 ? f0 : -(f0 + 3));
            uint32_t v[4][4];
#pragma unroll
            for (int t = 0; t < 4; ++t) load4<In>(cube + base + (long long)(4 * c + t) * o.sz, v[t]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int jj = sf > 0 ? j : 3 - j;
                const int row = fy ? other * 32 + 4 * g + j : (4 * g + j) * 32 + other;
                *reinterpret_cast<uint4 *>(slab_chunk(row, c)) = make_uint4(v[0][jj], v[1][jj], v[2][jj], v[3][jj]);
            }
        }
    }
    __syncthreads();                                         // slab staged
    SP_MARK(1);

    // ---- X1 (threads 0..159): task (run, y), lanes on y; Q(sig1, k, y)[q = 8 run + j] for all 8 sig1,
    // q = t + 8 in [0, 40): f at z' = q - 8 + l, i.e. slab chunks 2 run - 2 .. (zero pads outside 0..7);
    // row sig1 goes to CTA sig1 / 2 (distributed shared memory).  Threads 160..255 meanwhile write the
    // output runs of Y2 (12 wide) that lie wholly below the support: 12 run + 12 <= 2N - s1 - (4 sig2 + 3)
    // for all 4 rows of a Y2 task (which Y2 then skips).
    Acc *outp = reinterpret_cast<Acc *>(p.out) + (long long)inst * N * N * 3 * N;
    if (tid < 5 * 32) {
        const int y = tid & 31, run = tid >> 5;
        Acc acc[8][R];
        auto rc = [&](int a, int c) -> const unsigned char * { return slab_chunk(a * 32 + y, c); };
        if (!(D3_SEP_ABL & 8)) radix8<8, 0, R, Acc>(rc, 2 * run - 2, p.one, acc);
        // every CTA of the cluster has started (arrive at entry) before any remote store
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            unsigned char *q = cluster.map_shared_rank(smQ, (D3_SEP_ABL & 2) ? k : (s >> 1)) + (((s & 1) * 4 + k) * 32 + y) * QP * 16;
            put_run<Acc>(q, 2 * run, acc[s]);
        }
    } else {
#ifndef D3_SEP_ZERO
#define D3_SEP_ZERO 0        // 0: one bulk copy (TMA) per row prefix here, overlapping X1 (default); measured:
                             // 1 16-byte stores here (f32 0.760 ms vs 0.713), 3 Y2 stores whole rows, zeros
                             // included (0.729); 2 none (ablation)
#endif
        if constexpr (D3_SEP_ZERO == 0) {
            // one bulk copy (TMA engine) of the zero region per output row prefix
            const uint32_t zsrc = static_cast<uint32_t>(__cvta_generic_to_shared(zero));
            for (int row = tid - 5 * 32; row < 8 * 32; row += THREADS - 5 * 32) {     // row = s1l * 32 + s2
                const int s1 = 8 * k + (row >> 5), s2 = row & 31;
                const int lim = 2 * N - s1 - (4 * (s2 >> 2) + 3), nz = lim > 0 ? lim / 12 : 0;
                if (nz > 0)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                     outp + ((long long)s1 * N + s2) * (3 * N)),
                                 "r"(zsrc), "r"(48 * nz)
                                 : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        } else if constexpr (D3_SEP_ZERO == 1) {
            for (int row = tid - 5 * 32; row < 8 * 32; row += THREADS - 5 * 32) {
                const int s1 = 8 * k + (row >> 5), s2 = row & 31;
                const int lim = 2 * N - s1 - (4 * (s2 >> 2) + 3), nz = lim > 0 ? lim / 12 : 0;
                Acc *d = outp + ((long long)s1 * N + s2) * (3 * N);
                for (int r = 0; r < 3 * nz; ++r) st_cs_v4(d + 4 * r, 0u, 0u, 0u, 0u);
            }
        }
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    }
    // every Q row has arrived (release / acquire at cluster scope)
    SP_MARK(2);
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    SP_MARK(3);

    // ---- X2: task (sl, run, y), lanes on y; P(s1 = 4 sig1 + rho1, y)[p = 8 run + j], sig1 = 2k + sl,
    // p = t + 32 in [0, 64): Q at q = p - 24 + sig1 V1 + l^2_rho1(V1) (chunks 2 run - 6 + .., valid 0..9)
    for (int t = tid; t < ((D3_SEP_ABL & 8) ? 0 : 2 * 8 * 32); t += THREADS) {
        const int y = t & 31, run = (t >> 5) & 7, sl = t >> 8, sig1 = 2 * k + sl;
        Acc acc[4][R];
        if (8 * run + 8 > 32 - (4 * sig1 + 3)) {            // else below the support of all 4 slopes
            auto rc = [&](int V1, int c) -> const unsigned char * {
                return (unsigned)c < (unsigned)QCH ? smQ + (((sl * 4 + V1) * 32 + y) * QP + c) * 16 : zero;
            };
            with_const8<0>(sig1, [&](auto S_) { radix4<decltype(S_)::value, R, Acc>(rc, 2 * run - 6, p.one, acc); });
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < R; ++j) acc[i][j] = Acc(0);
        }
#pragma unroll
        for (int rho = 0; rho < 4; ++rho) {
            unsigned char *row = smP + (32 * (4 * sl + rho) + y) * 256;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
                *reinterpret_cast<uint4 *>(row + 16 * pswz(2 * run + hh, y)) =
                    make_uint4(Lane<Acc>::bits(acc[rho][4 * hh]), Lane<Acc>::bits(acc[rho][4 * hh + 1]),
                               Lane<Acc>::bits(acc[rho][4 * hh + 2]), Lane<Acc>::bits(acc[rho][4 * hh + 3]));
        }
    }
    __syncthreads();
    SP_MARK(4);

    // ---- y part, 2 batches of 4 slopes s1 (U over region Q).  U(sb; sig2, V2) is needed for
    // t >= -(s1 + sig2): u = t + 40 in [8, 72) (16 runs of 4) for s1 < 24, [0, 72) (18 runs) above.
    const int ulo = k == 3 ? 0 : 2, nrun1 = 18 - ulo;
#pragma unroll 1
    for (int b = 0; b < ((D3_SEP_ABL & 4) ? 0 : 2); ++b) {
        // Y1: task (sb, V2, run), lanes on run; U(sb; sig2, V2)[u = 4 run + j]: P(s1, 8 V2 + w2) at
        // p = u - 8 + l^3_sig2(w2) (chunks run - 2 + .., valid 0..15)
        for (int t = tid; t < 4 * 4 * nrun1; t += THREADS) {
            constexpr int R1 = 4;
            const int rest = t / nrun1, run = ulo + t - rest * nrun1, V2 = rest & 3, sb = rest >> 2;
            const int s1l = 4 * b + sb;
            Acc acc[8][R1];
            const int cb = run - 2;
            auto rc = [&](int w2, int c) -> const unsigned char * {
                const int y = 8 * V2 + w2;
                return (unsigned)c < 16u ? smP + ((32 * s1l + y) * 16 + pswz(c, y)) * 16 : zero;
            };
            radix8<8, 0, R1, Acc>(rc, cb, p.one, acc);
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2)
                *reinterpret_cast<uint4 *>(smQ + (((sb * 8 + s2) * 4 + V2) * UP + run) * 16) =
                    make_uint4(Lane<Acc>::bits(acc[s2][0]), Lane<Acc>::bits(acc[s2][1]), Lane<Acc>::bits(acc[s2][2]),
                               Lane<Acc>::bits(acc[s2][3]));
        }
        __syncthreads();
        // Y2: warp = sig2, lane = (sb, run); out(s1, 4 sig2 + rho2)[D = 12 run + j]: U at
        // u = D - 24 + sig2 V2 + l^2_rho2(V2) (chunks 3 run - 6 + .., valid ulo..17)
        {
            constexpr int R2 = 12;
            const int sig2 = tid >> 5, sb = (tid >> 3) & 3, run = tid & 7;
            const int s1 = 8 * k + 4 * b + sb;
            bool skip = false;
            Acc acc[4][R2];
            if (12 * run + 12 > 2 * N - s1 - (4 * sig2 + 3)) {
                auto rc = [&](int V2, int c) -> const unsigned char * {
                    return (unsigned)(c - ulo) < (unsigned)(UCH - ulo) ? smQ + (((sb * 8 + sig2) * 4 + V2) * UP + c) * 16
                                                                       : zero;
                };
                with_const8<0>(sig2, [&](auto S_) { radix4<decltype(S_)::value, R2, Acc>(rc, 3 * run - 6, p.one, acc); });
            } else {
                // wholly below the support of the 4 rows: zeros (written by the block's own stores unless the
                // X1-phase zero writer did, D3_SEP_ZERO < 3)
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int j = 0; j < R2; ++j) acc[q][j] = Acc(0);
                if (D3_SEP_ZERO < 3) skip = true;
            }
            Acc *orow = outp + ((long long)s1 * N + 4 * sig2) * (3 * N) + R2 * run;
            if (D3_SEP_ABL & 1) {
                if (Lane<Acc>::bits(acc[0][0]) == 0x7f7f7f7fu) orow[0] = acc[3][11];   // keep the sums live
            } else if (!skip) {
#ifndef D3_SEP_ST256
#define D3_SEP_ST256 1       // measured: cfg5 0.731 -> 0.684 ms, 256 u8 cubes 0.651 -> 0.590
#endif
#if D3_SEP_ST256
                // a 48-byte run = one 32-byte store (STG.256) + one 16-byte store; runs start 32-byte
                // aligned on even lanes and 16 bytes past on odd ones (rows are 384 bytes)
                if ((reinterpret_cast<unsigned long long>(outp) & 31ull) == 0) {
                    const bool odd = run & 1;
#pragma unroll
                    for (int rho = 0; rho < 4; ++rho) {
                        uint32_t v8[8], v4[4];
#pragma unroll
                        for (int j = 0; j < 8; ++j) v8[j] = odd ? Lane<Acc>::bits(acc[rho][4 + j]) : Lane<Acc>::bits(acc[rho][j]);
#pragma unroll
                        for (int j = 0; j < 4; ++j) v4[j] = odd ? Lane<Acc>::bits(acc[rho][j]) : Lane<Acc>::bits(acc[rho][8 + j]);
                        Acc *o = orow + rho * (3 * N);
                        st_cs_v8(o + (odd ? 4 : 0), v8);
                        st_cs_v4(o + (odd ? 0 : 8), v4[0], v4[1], v4[2], v4[3]);
                    }
                } else
#endif
#pragma unroll
                for (int rho = 0; rho < 4; ++rho)
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        st_cs_v4(orow + rho * (3 * N) + 4 * q, Lane<Acc>::bits(acc[rho][4 * q]), Lane<Acc>::bits(acc[rho][4 * q + 1]),
                                 Lane<Acc>::bits(acc[rho][4 * q + 2]), Lane<Acc>::bits(acc[rho][4 * q + 3]));
            }
        }
        __syncthreads();                                     // U is rewritten by the next batch
#ifdef D3_PROF_SEP32
        sp_t[5 + b] = clock64();
#endif
    }
    // the zero region must outlive the bulk zero stores' shared-memory reads
    if (D3_SEP_ZERO == 0 && tid >= 5 * 32) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#ifdef D3_PROF_SEP32
    sp_t[7] = clock64();
    if ((tid & 31) == 0 && (tid == 0 || tid == 224)) {
        const int bb = tid == 0 ? 0 : 16;
        for (int i = 0; i < 7; ++i) atomicAdd(&d3_sep_prof[bb + i], (unsigned long long)(sp_t[i + 1] - sp_t[i]));
        atomicAdd(&d3_sep_prof[bb + 15], 1ull);
    }
#endif
}

template <class In, class Acc>
drt3d_status launch(const DrtPass &prm, int ninst, cudaStream_t st) {
    auto kern = drt_sep32_kernel<In, Acc>;
    static std::atomic<uint32_t> smem_done{0};
    if (!set_smem_once(kern, SMEM, smem_done)) return DRT3D_ERR_CUDA;
    kern<<<dim3((unsigned)(CL * ninst)), THREADS, SMEM, st>>>(prm);
    return DRT3D_OK;
}

}  // namespace sep32

drt3d_status dispatch_drt_sep32(int in_dtype, const DrtPass &prm, int ninst, cudaStream_t st) {
    if (prm.N != sep32::N) return DRT3D_ERR_UNSUPPORTED;
    if (in_dtype == DRT3D_U8) return sep32::launch<uint8_t, uint32_t>(prm, ninst, st);
    if (in_dtype == DRT3D_I32) return sep32::launch<uint32_t, uint32_t>(prm, ninst, st);
    return sep32::launch<float, float>(prm, ninst, st);
}

}  // namespace d3

#ifdef D3_PROF_SEP32
extern "C" int d3_sep_prof_read(unsigned long long *out32) {
    if (cudaMemcpyFromSymbol(out32, d3::sep32::d3_sep_prof, 32 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    unsigned long long z[32] = {0};
    return cudaMemcpyToSymbol(d3::sep32::d3_sep_prof, z, sizeof(z)) != cudaSuccess;
}
#endif
