// djt_kernels.cuh -- 3D DJT of lines: one "radix-2^K pass" kernel.
//
// Alg. 3 (eq:map3DJ PAPER.md:425-437) regrouped into passes
// of K stages.  From the stage-c partial transform (eq:3DJfm)
// the stage-(c+K) value is a direct sum over 2^K consecutive rows along the
// driving axis:
//
//   f^{c+K}(V | s1' | s2' | D1 | D2) = sum_{w < 2^K} f^c(V 2^K + w | s1 | s2 |
//               D1 + s1 w + l^K_{r1}(w) | D2 + s2 w + l^K_{r2}(w)),   s' = s 2^K + r.
//
// Storage of a stage-c buffer (per instance):
//   rows ((s1 2^c + s2) 2^(n-c) + v), each a plane [D1'][D2'],
//   Di' = Di - base_c, base_c = N - (2^c - 1), valid width N + 2^c - 1.
// Stage 0 is the oriented cube (x' = v, D1 = y' + N, D2 = z' + N), the final
// stage is out[s1][s2][D1][D2] with Di in [0, 2N) (Alg. 3 + separateS1S2).
#pragma once
#include <cuda.h>
#include "common.cuh"
#ifndef D3_FADD2
#define D3_FADD2 0
#endif
#ifndef D3_PDL
#define D3_PDL 1
#endif

namespace d3 {

struct DjtPass {
    const void *in;
    void *out;
    int N, n, c, m;
    long long in_inst_stride, in_plane;    // elements between instances / rows (planes)
    int in_pitch, in_base, in_width;
    long long out_inst_stride, out_plane;
    int out_pitch, out_base, out_width;
    int nt2;                               // tiles along D2
    int inst0, ndod;
    int vec_ok;                            // first pass: 16-byte chunked cube loads are aligned
    int zero_tma;                          // final pass: zero tiles leave as TMA stores (zmap)
    int inst_total;                        // instances of the whole call
    Orient ori[kMaxDod];
};

template <int K, int R, int T1, int T2>
struct DjtGeom {
    static constexpr int S = 1 << K;
    static constexpr int H = S - 1;
    static constexpr int WR = T1 + H;                     // staged rows per plane
    static constexpr int WC = T2 + H;                     // staged columns
    static constexpr int NR = T2 / R;
    static constexpr int NEED = ((T2 + H + 3) / 4) * 4;   // furthest column touched
    static constexpr int PJ0 = ((NEED > WC ? NEED : WC) + 3) / 4 * 4;
    static constexpr int PJ = ((PJ0 / 4) % 2 == 1) ? PJ0 : PJ0 + 4;   // pitch/4 odd: no bank conflicts across rows
    static constexpr int TASKS = S * T1 * NR;
#ifndef D3_DJT_THREADS
#define D3_DJT_THREADS 128    // 4 CTAs per SM at ~100 registers; 256 (2 per SM) is 1.7% slower on cfg4
#endif
    static constexpr int THREADS = D3_DJT_THREADS;
    static constexpr int SMEM_STAGE = S * WR * PJ * 4;
    // final passes with TMA output stores (D3_DJT_OUT_TMA): one S x T1 x T2 32-bit image per warp
    // behind the staged planes; a warp's 32 tasks of one iteration are exactly one r1
#ifndef D3_DJT_OUT_TMA
#define D3_DJT_OUT_TMA 0                  // measured: cfg4 0.0891 vs 0.0860 ms with the direct 16-byte stores
#endif
    static constexpr bool OUT_TMA = D3_DJT_OUT_TMA && T1 * NR == 32 && THREADS % 32 == 0 && R == 8;
    // final passes (D3_DJT_OUT_SMEM): a warp's tasks (one r1, T1 = 8 rows x T2 = 32 columns, S planes)
    // go through a per-warp XOR-swizzled shared-memory image, so that every 16-byte store instruction
    // writes 4 whole 128-byte row segments (direct stores from the task registers put 16 bytes in
    // each of 32 sectors of 8 lines per instruction: the L1 data pipe was at 81% on cfg4)
#ifndef D3_DJT_OUT_SMEM
#define D3_DJT_OUT_SMEM 1
#endif
    // D3_DJT_ST256: final 32-bit outputs leave the task registers as 32-byte stores (STG.256): a
    // lane's 8 columns fill one whole sector, 4 lanes one 128-byte line, so each instruction writes
    // 8 whole lines with no shared-memory image
#ifndef D3_DJT_ST256
#define D3_DJT_ST256 0
#endif
    static constexpr bool OUT_SMEM =
        D3_DJT_OUT_SMEM && !D3_DJT_ST256 && !OUT_TMA && T1 == 8 && T2 == 32 && R == 8 && THREADS % 32 == 0;
    static constexpr int IMG = S * T1 * T2 * 4;
    static constexpr int SMEM = SMEM_STAGE + ((OUT_TMA || OUT_SMEM) ? (THREADS / 32) * IMG : 0);
    static_assert(T2 % R == 0 && R % 4 == 0, "tile shape");
};

#ifndef D3_DJT_MINB
#define D3_DJT_MINB 1
#endif
template <int K, int R, int T1, int T2, class In, class Acc, class Out, bool FIRST, bool FINAL>
__global__ void __launch_bounds__(D3_DJT_THREADS, D3_DJT_MINB)
djt_pass_kernel(const DjtPass p, const __grid_constant__ CUtensorMap zmap) {
    using G = DjtGeom<K, R, T1, T2>;
    constexpr int S = G::S, WR = G::WR, WC = G::WC, PJ = G::PJ, NR = G::NR;
    extern __shared__ uint4 smem_u4[];
    uint32_t *sm = reinterpret_cast<uint32_t *>(smem_u4);

    const int tid = threadIdx.x;
    const int t1 = blockIdx.x / p.nt2, t2 = blockIdx.x - t1 * p.nt2;
    const int g = blockIdx.y, li = blockIdx.z, inst = p.inst0 + li;
    const int m = p.m, c = p.c, N = p.N, cK = c + K;
    const int V = g & ((1 << m) - 1);
    const int sig = g >> m;
    const int sg2 = sig & ((1 << c) - 1), sg1 = sig >> c;
    const int d10 = t1 * T1, d20 = t2 * T2;                 // stored output coords of the tile
    if constexpr (FIRST && D3_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int D1abs = p.out_base + d10, D2abs = p.out_base + d20;

    Out *outp = reinterpret_cast<Out *>(p.out);
    const long long out_inst = FINAL ? (long long)inst * p.out_inst_stride : (long long)li * p.out_inst_stride;
    auto out_plane_ptr = [&](int r1, int r2) -> Out * {
        const int s1 = (sg1 << K) + r1, s2 = (sg2 << K) + r2;
        const long long row = ((((long long)s1 << cK) + s2) << m) + V;
        return outp + out_inst + row * p.out_plane;
    };

    // ---- zero tiles: outputs need Di >= N - si (line support)
    {
        const int s1max = (sg1 << K) + S - 1, s2max = (sg2 << K) + S - 1;
        if (D1abs + T1 <= N - s1max || D2abs + T2 <= N - s2max) {
            if constexpr (FINAL && sizeof(Out) == 4) {
                if (p.zero_tma) {
                    // S TMA tensor stores of one zeroed S x T1 x T2 shared-memory image (zmap: the final
                    // output [inst][s1][s2][D1][D2], box {T2, T1, S, 1, 1}); the CTA is done once the TMA
                    // engine has read it
                    for (int i = tid; i < S * T1 * T2 / 4; i += blockDim.x) smem_u4[i] = make_uint4(0u, 0u, 0u, 0u);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncthreads();
                    if (tid == 0) {
                        const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(smem_u4));
                        for (int r1 = 0; r1 < S; ++r1)
                            asm volatile(
                                "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&zmap),
                                "r"(d20), "r"(d10), "r"(sg2 << K), "r"((sg1 << K) + r1), "r"(inst), "r"(src)
                                : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    }
                    return;
                }
            }
            constexpr int EPV = 16 / (int)sizeof(Out);
            if (T2 % EPV == 0 && d20 + T2 <= p.out_width && (p.out_pitch * (int)sizeof(Out)) % 16 == 0 &&
                (d20 * (int)sizeof(Out)) % 16 == 0 && (p.out_plane * (long long)sizeof(Out)) % 16 == 0) {
                // 16-byte streaming stores; the plane pointer changes every T1 * T2 / EPV chunks
                constexpr int CPR = T2 / EPV, CPP = T1 * CPR;
                for (int i = tid; i < S * S * CPP; i += blockDim.x) {
                    const int pl = i / CPP, rem = i - pl * CPP, e1 = rem / CPR, q = rem - e1 * CPR;
                    if (d10 + e1 < p.out_width) {
                        Out *dst = out_plane_ptr(pl / S, pl % S) + (long long)(d10 + e1) * p.out_pitch + d20 + q * EPV;
                        if (FINAL) st_cs_v4(dst, 0u, 0u, 0u, 0u);
                        else *reinterpret_cast<uint4 *>(dst) = make_uint4(0u, 0u, 0u, 0u);
                    }
                }
                return;
            }
            for (int i = tid; i < S * S * T1 * T2; i += blockDim.x) {
                const int e2 = i % T2, rest = i / T2, e1 = rest % T1, pl = rest / T1;
                if (d10 + e1 < p.out_width && d20 + e2 < p.out_width)
                    out_plane_ptr(pl / S, pl % S)[(long long)(d10 + e1) * p.out_pitch + d20 + e2] = to_out<Out, Acc>(Acc(0));
            }
            return;
        }
    }

    // programmatic dependent launch (DESIGN.md §5 item 8): wait for the previous pass's grid only now
    if constexpr (!FIRST && D3_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    // ---- stage the 2^K input planes' windows
    auto put = [&](int w, int i1, int i2, uint32_t bits) { sm[(w * WR + i1) * PJ + i2] = bits; };
    if constexpr (FIRST) {
        const Orient o = p.ori[inst % p.ndod];
        const In *cube = reinterpret_cast<const In *>(p.in) + (long long)(inst / p.ndod) * N * N * N;
        const int y0 = D1abs - N, z0 = D2abs - N;     // stage 0: D1 = y' + N, D2 = z' + N
        const int xb = V << K;
        auto run = [&](long long b, long long stride, int start, bool valid) {
            RowSrc<In> r;
            if (stride > 0) { r.ptr = cube + b; r.st = start; r.dir = 1; }
            else { r.ptr = cube + b - (N - 1); r.st = N - 1 - start; r.dir = -1; }
            r.width = valid ? N : 0;
            return r;
        };
        if (!p.vec_ok) {
            for (int i = tid; i < S * WR * WC; i += blockDim.x) {
                const int i2 = i % WC, rest = i / WC, i1 = rest % WR, w = rest / WR;
                const int y = y0 + i1, z = z0 + i2;
                uint32_t bits = 0;
                if ((unsigned)y < (unsigned)N && (unsigned)z < (unsigned)N)
                    bits = Elem<In>::load_bits(cube + o.off0 + (xb + w) * o.sx + y * o.sy + z * o.sz);
                put(w, i1, i2, bits);
            }
        } else if (o.fast == 2) {           // z' (D2) contiguous
            stage_rows<In, 8>(S * WR, WC, [&](int r) {
                const int i1 = r % WR, w = r / WR, y = y0 + i1;
                return run(o.off0 + (long long)(xb + w) * o.sx + (long long)y * o.sy, o.sz, z0, (unsigned)y < (unsigned)N);
            }, [&](int r, int i2, uint32_t bits) { put(r / WR, r % WR, i2, bits); });
        } else if (o.fast == 1) {           // y' (D1) contiguous
            stage_rows<In, 8>(S * WC, WR, [&](int r) {
                const int i2 = r % WC, w = r / WC, z = z0 + i2;
                return run(o.off0 + (long long)(xb + w) * o.sx + (long long)z * o.sz, o.sy, y0, (unsigned)z < (unsigned)N);
            }, [&](int r, int i1, uint32_t bits) { put(r / WC, i1, r % WC, bits); });
        } else {                            // x' (driving axis) contiguous
            stage_rows<In, 8>(WR * WC, S, [&](int r) {
                const int i2 = r % WC, i1 = r / WC, y = y0 + i1, z = z0 + i2;
                return run(o.off0 + (long long)y * o.sy + (long long)z * o.sz, o.sx, xb,
                           (unsigned)y < (unsigned)N && (unsigned)z < (unsigned)N);
            }, [&](int r, int w, uint32_t bits) { put(w, r / WC, r % WC, bits); });
        }
    } else {
        const In *inb = reinterpret_cast<const In *>(p.in) + (long long)li * p.in_inst_stride;
        const int nc = p.n - c;
        const long long rbase = ((((long long)sg1 << c) + sg2) << nc) + ((long long)V << K);
        stage_rows<In, 8>(S * WR, WC, [&](int r) {
            const int i1 = r % WR, w = r / WR;
            const int a1 = D1abs + sg1 * w - p.in_base + i1;
            RowSrc<In> rr;
            rr.ptr = inb + (rbase + w) * p.in_plane + (long long)a1 * p.in_pitch;
            rr.st = D2abs + sg2 * w - p.in_base;
            rr.dir = 1;
            rr.width = ((unsigned)a1 < (unsigned)p.in_width) ? p.in_width : 0;
            return rr;
        }, [&](int r, int i2, uint32_t bits) { put(r / WR, r % WR, i2, bits); });
    }
    __syncthreads();

    // ---- direct sum: thread task (r1, d1, run) accumulates all S values of r2
    constexpr int NB = (R + S + 2) / 4;
    for (int task = tid; task < G::TASKS; task += blockDim.x) {
        const int d1 = task % T1, rest = task / T1, rr = rest % NR, r1 = rest / NR;
        const int c0 = rr * (R / 4);
        Acc acc[S][R];
        // l^K_{r1}(w) at run time (r1 is a per-thread value; only a row offset)
        auto l1_of = [&](int w) {
            int l1 = 0, s = r1, u = w;
#pragma unroll
            for (int k = K; k >= 1; --k) {
                l1 += ((u >> (k - 1)) & 1) * ((s + 1) >> 1);
                s >>= 1;
                u &= (1 << (k - 1)) - 1;
            }
            return l1;
        };
        auto load_plane = [&](int w, int nc, uint32_t *buf) {
            const uint32_t *row = sm + (w * WR + d1 + l1_of(w)) * PJ + c0 * 4;
#pragma unroll
            for (int i = 0; i < nc; ++i) {
                const uint4 v = *reinterpret_cast<const uint4 *>(row + 4 * i);
                buf[4 * i + 0] = v.x;
                buf[4 * i + 1] = v.y;
                buf[4 * i + 2] = v.z;
                buf[4 * i + 3] = v.w;
            }
        };
        if constexpr (S == 1) {
            uint32_t buf[NB * 4];
            load_plane(0, (R + 3) / 4, buf);
#pragma unroll
            for (int j = 0; j < R; ++j) acc[0][j] = Lane<Acc>::get(buf[j]);
        } else {
            // planes two at a time: integer sums become 3-input adds; the first pair initialises
            static_for<0, S / 2>([&](auto p_) {
                constexpr int w0 = 2 * decltype(p_)::value, w1 = w0 + 1;
                constexpr int NC0 = (R + w0 + 3) / 4, NC1 = (R + w1 + 3) / 4;
                uint32_t b0[NC0 * 4], b1[NC1 * 4];
                load_plane(w0, NC0, b0);
                load_plane(w1, NC1, b1);
                static_for<0, S>([&](auto r_) {
                    constexpr int r = decltype(r_)::value;
                    constexpr int o0 = lk(K, r, w0), o1 = lk(K, r, w1);
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        if constexpr (w0 == 0) acc[r][j] = Lane<Acc>::get(b0[j + o0]) + Lane<Acc>::get(b1[j + o1]);
                        else acc[r][j] = add2<Acc>(acc[r][j], b0[j + o0], b1[j + o1], 1u, false);
                    }
                });
            });
        }
        if constexpr (FINAL && sizeof(Out) == 4 && G::OUT_TMA) {
            if (p.zero_tma) {
                // this warp's tasks = one r1: its S x T1 x T2 outputs go to the warp's image, then one
                // TMA tensor store (zmap, box {T2, T1, S, 1, 1}); the image is reused next iteration
                // after lane 0 has waited for the TMA engine to read it
                unsigned char *img = reinterpret_cast<unsigned char *>(smem_u4) + G::SMEM_STAGE + (tid >> 5) * G::IMG;
#pragma unroll
                for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                    for (int q = 0; q < R / 4; ++q)
                        *reinterpret_cast<uint4 *>(img + ((r2 * T1 + d1) * T2 + rr * R + 4 * q) * 4) =
                            make_uint4(Lane<Acc>::bits(acc[r2][4 * q]), Lane<Acc>::bits(acc[r2][4 * q + 1]),
                                       Lane<Acc>::bits(acc[r2][4 * q + 2]), Lane<Acc>::bits(acc[r2][4 * q + 3]));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if ((tid & 31) == 0) {
                    const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(img));
                    asm volatile(
                        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&zmap),
                        "r"(d20), "r"(d10), "r"(sg2 << K), "r"((sg1 << K) + r1), "r"(inst), "r"(src)
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
                __syncwarp();
                continue;
            }
        }
        if constexpr (FINAL && sizeof(Out) == 4 && G::OUT_SMEM) {
            if (d10 + T1 <= p.out_width && d20 + T2 <= p.out_width && (p.out_pitch % 4) == 0 && (d20 % 4) == 0 &&
                (p.out_plane % 4) == 0) {
                // image rows (r2, d1) of 8 chunks; piece k = 2 rr + q of row d1 at chunk k ^ d1 (the 8
                // lanes of a quarter-warp -- 8 rows d1 of one piece, or 8 pieces of one row -- touch 8
                // distinct 16-byte bank groups both ways)
                uint4 *img = reinterpret_cast<uint4 *>(reinterpret_cast<unsigned char *>(smem_u4) + G::SMEM_STAGE +
                                                       (tid >> 5) * G::IMG);
                __syncwarp();                               // the previous iteration's reads are done
#pragma unroll
                for (int r2 = 0; r2 < S; ++r2)
#pragma unroll
                    for (int q = 0; q < 2; ++q)
                        img[(r2 * T1 + d1) * 8 + ((2 * rr + q) ^ d1)] =
                            make_uint4(Lane<Acc>::bits(acc[r2][4 * q]), Lane<Acc>::bits(acc[r2][4 * q + 1]),
                                       Lane<Acc>::bits(acc[r2][4 * q + 2]), Lane<Acc>::bits(acc[r2][4 * q + 3]));
                __syncwarp();
                const int lane = tid & 31, k = lane & 7;
#ifndef D3_DJT_IMG256
#define D3_DJT_IMG256 0
#endif
                if (D3_DJT_IMG256 && (p.out_pitch % 8) == 0 && (p.out_plane % 8) == 0 && (p.out_inst_stride % 8) == 0 &&
                    (reinterpret_cast<unsigned long long>(outp) & 31ull) == 0) {
                    // 32-byte stores: 4 lanes per 128-byte row segment, 8 whole lines per instruction
                    const int k2 = lane & 3;
#pragma unroll
                    for (int it = 0; it < S * T1 / 8; ++it) {
                        const int row = 8 * it + (lane >> 2), r2 = row / T1, e = row - r2 * T1;
                        const uint4 a = img[row * 8 + ((2 * k2) ^ e)], b = img[row * 8 + ((2 * k2 + 1) ^ e)];
                        Out *dst = out_plane_ptr(r1, r2) + (long long)(d10 + e) * p.out_pitch + d20 + 8 * k2;
                        const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                        st_cs_v8(dst, v);
                    }
                    continue;
                }
#pragma unroll
                for (int it = 0; it < S * T1 / 4; ++it) {
                    const int row = 4 * it + (lane >> 3), r2 = row / T1, e = row - r2 * T1;
                    const uint4 v = img[row * 8 + (k ^ e)];
                    Out *dst = out_plane_ptr(r1, r2) + (long long)(d10 + e) * p.out_pitch + d20 + 4 * k;
                    st_cs_v4(dst, v.x, v.y, v.z, v.w);
                }
                continue;
            }
        }
        // store S output planes (r1, r2), row d1, columns run rr
        const int e1 = d10 + d1, e2 = d20 + rr * R;
        if (e1 < p.out_width) {
            const bool vec_ok = (e2 + R <= p.out_width) && ((p.out_pitch * (int)sizeof(Out)) % 16 == 0) &&
                                ((e2 * (int)sizeof(Out)) % 16 == 0) && ((p.out_plane * (long long)sizeof(Out)) % 16 == 0);
            [[maybe_unused]] const bool vec32_ok =
                vec_ok && ((p.out_pitch * (int)sizeof(Out)) % 32 == 0) && ((e2 * (int)sizeof(Out)) % 32 == 0) &&
                ((p.out_plane * (long long)sizeof(Out)) % 32 == 0) && ((p.out_inst_stride * (long long)sizeof(Out)) % 32 == 0) &&
                ((reinterpret_cast<unsigned long long>(outp) & 31ull) == 0);
#pragma unroll
            for (int r2 = 0; r2 < S; ++r2) {
                Out *dst = out_plane_ptr(r1, r2) + (long long)e1 * p.out_pitch + e2;
                if (vec_ok) {
                    if constexpr (sizeof(Out) == 2) {
#pragma unroll
                        for (int q = 0; q < R / 8; ++q) {
                            uint32_t wv[4];
#pragma unroll
                            for (int h = 0; h < 4; ++h)
                                wv[h] = (uint32_t)to_out<Out, Acc>(acc[r2][8 * q + 2 * h]) |
                                        ((uint32_t)to_out<Out, Acc>(acc[r2][8 * q + 2 * h + 1]) << 16);
                            *reinterpret_cast<uint4 *>(dst + 8 * q) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                        }
                    } else {
                        if constexpr (FINAL && R == 8 && D3_DJT_ST256) {
                            if (vec32_ok) {
                                uint32_t v[8];
#pragma unroll
                                for (int j = 0; j < 8; ++j) v[j] = Lane<Acc>::bits(acc[r2][j]);
                                st_cs_v8(dst, v);
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
                        if (e2 + j < p.out_width) dst[j] = to_out<Out, Acc>(acc[r2][j]);
                }
            }
        }
    }
}

}  // namespace d3
