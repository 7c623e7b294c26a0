// launch.cuh -- kernel launch templates (tile shapes per radix) shared by
// the per-dtype translation units k_*.cu.
#pragma once
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>
#include "dispatch.h"
#include "drt_first_swar.cuh"

namespace d3 {

template <int A, int B, int C = 0> struct IntPair { static constexpr int first = A, second = B, third = C; };

// ---- DRT kernel selection
template <int K> struct DrtTile;
template <> struct DrtTile<1> { static constexpr int R = 8, T = 128; };
template <> struct DrtTile<2> { static constexpr int R = 8, T = 128; };
template <> struct DrtTile<3> { static constexpr int R = 8, T = 64; };
template <> struct DrtTile<4> { static constexpr int R = 8, T = 64; };

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// 4D map of the stacked DRT output out[inst][s1][s2][3N] (32-bit), box {T, S, S1, 1}
inline bool make_out_map(CUtensorMap *m, void *out, int N, int inst_total, int T, int S, int S1,
                         CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_UINT32) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    const cuuint64_t W = 3ull * N;
    cuuint64_t dims[4] = {W, (cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)inst_total};
    cuuint64_t str[3] = {W * 4, W * 4 * N, W * 4 * N * N};
    cuuint32_t box[4] = {(cuuint32_t)T, (cuuint32_t)S, (cuuint32_t)S1, 1}, es[4] = {1, 1, 1, 1};
    return enc(m, dt, 4, out, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

template <int K, class In, class Acc, class Out, bool FIRST, bool FINAL>
drt3d_status launch_drt_k(const DrtPass &prm_in, int ninst, cudaStream_t st) {
    DrtPass prm = prm_in;
    // u16-input final passes use a narrower tile (more resident CTAs per SM); non-final passes keep
    // T / R a power of two (their epilogue shuffles across the T / R runs of a row)
#ifndef D3_SINGLE_T
#define D3_SINGLE_T 64                  // the single-pass plan (N = 16, K = 4): D tile width
#endif
#ifndef D3_FINAL2_T
#define D3_FINAL2_T 96                  // K = 2 final passes: T = 3N at N = 32 (swept 48 / 64 / 96 / 128: cfg5 0.827 -> 0.741 ms)
#endif
#ifndef D3_FINAL16K3_T
#define D3_FINAL16K3_T 64               // u16-input K = 3 final passes (u8 voxels, N = 128)
#endif
    constexpr int R = DrtTile<K>::R,
                  T = (!FIRST && FINAL && sizeof(In) == 2 && K == 4) ? D3_FINAL16_T
                      : (!FIRST && FINAL && sizeof(In) == 2 && K == 3) ? D3_FINAL16K3_T
                      : (FIRST && FINAL && K == 4)                 ? D3_SINGLE_T
                      : (!FIRST && FINAL && K == 2)                ? D3_FINAL2_T
                                                                   : DrtTile<K>::T;
    if constexpr (FIRST && !FINAL && K >= 3 && std::is_same<In, uint8_t>::value && std::is_same<Out, uint16_t>::value) {
        // u8 voxels -> u16 stage-K rows: packed 16-bit lanes (drt_first_swar.cuh)
#ifndef SWAR_R
#define SWAR_R 8
#endif
        constexpr int RS = SWAR_R;
        // few tiles (under D3_SWAR_SMALL_CTAS CTAs at T = 64, about one per SM): half-width tiles
        // (T = 32, R = 4), twice the CTAs on the latency-bound per-tile chain.  Measured at N = 64:
        // one dodecant (32 CTAs) 0.0154 -> 0.0133 ms; 12 dodecants (384 CTAs) 0.0317 -> 0.0338 (kept
        // at T = 64 by the threshold)
#ifndef D3_SWAR_SMALL_CTAS
#define D3_SWAR_SMALL_CTAS 160
#endif
#ifndef D3_SWAR_TMA_MIN_N
#define D3_SWAR_TMA_MIN_N 128           // N = 64 measured: no gain (cfg2 0.0317 vs 0.0297 ms)
#endif
        const long long groups = 1LL << (2 * prm.m);
        const bool half = K == 4 && T == 64 && prm.zf_T == 0 &&
                          (long long)((prm.out_width + 8 + T - 1) / T) * groups * ninst < D3_SWAR_SMALL_CTAS;
        auto go = [&](auto geo) -> drt3d_status {
            constexpr int RR = decltype(geo)::first, TT = decltype(geo)::second, EE = decltype(geo)::third;
            using SG = SwarGeom<K, RR, TT, EE>;
            auto kern = drt_first_swar_kernel<K, RR, TT, EE>;
            static std::atomic<uint32_t> smem_done{0};
            if (!set_smem_once(kern, SG::SMEM + 16, smem_done)) return DRT3D_ERR_CUDA;      // + the staging mbarrier
            const int ntiles = (prm.out_width + 8 + TT - 1) / TT;
            dim3 grid(ntiles, (unsigned)groups, ninst);
            // the final pass's zero tiles (api.cu, DESIGN.md §5 item 6): map of the final output
            CUtensorMap zmap;
            std::memset(&zmap, 0, sizeof(zmap));
            DrtPass q = prm;
            if (q.zf_T > 0 && !(K == 4 && q.zf_T == D3_FINAL16_T && SG::SMEM >= (1 << (2 * K)) * D3_FINAL16_T * 4 &&
                                make_out_map(&zmap, q.zf_out, q.N, q.inst_total, q.zf_T, 1 << K, 1 << K)))
                return DRT3D_ERR_UNSUPPORTED;
            // cube brick maps for the TMA staging (drt_first_swar.cuh, SwarCubeMaps): cube[batch][x][y][z]
            // u8, box BW along original axis a and 16 along the other two; boxes must fit the cube
            SwarCubeMaps cm;
            std::memset(&cm, 0, sizeof(cm));
            int tma_in = 0;
            if (K == 4 && D3_SWAR_TMA_STAGE && q.N >= D3_SWAR_TMA_MIN_N && q.vec_ok) {
                auto enc = tmap_encoder();
                const cuuint64_t Nn = (cuuint64_t)q.N, nb = (cuuint64_t)((q.inst_total + q.ndod - 1) / q.ndod);
                cuuint64_t dims[4] = {Nn, Nn, Nn, nb};
                cuuint32_t es[4] = {1, 1, 1, 1};
                tma_in = enc != nullptr;
                for (int a = 0; a < 3 && tma_in; ++a) {
                    // a = 1: dimensions (z, x, y), so that the BW-long side is outermost
                    cuuint64_t str[3] = {a == 1 ? Nn * Nn : Nn, a == 1 ? Nn : Nn * Nn, Nn * Nn * Nn};
                    cuuint32_t box[4] = {16, 16, 16, 1};
                    box[a == 2 ? 0 : 2] = (cuuint32_t)(a == 2 ? SG::BWI : SG::BW);
                    tma_in = enc(&cm.m[a], CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(q.in), dims, str, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
                }
            }
            // stage-K rows as [inst][r1 r2][V1 V2][D] (u16): the copy-out's whole chunks of a tile's
            // 256 rows leave with one TMA store
            int tma_out = 0;
            if (K == 4 && D3_SWAR_TMA_OUT) {
                auto enc = tmap_encoder();
                const cuuint64_t pb = (cuuint64_t)q.out_pitch * 2;
                cuuint64_t dims[4] = {(cuuint64_t)q.out_width, (cuuint64_t)groups, 1ull << (2 * K), (cuuint64_t)ninst};
                cuuint64_t str[3] = {pb, pb * groups, (cuuint64_t)q.out_inst_stride * 2};
                cuuint32_t box[4] = {(cuuint32_t)(TT - 8), 1, 1u << (2 * K), 1}, es[4] = {1, 1, 1, 1};
                tma_out = enc != nullptr && (reinterpret_cast<uintptr_t>(q.out) & 15) == 0 && pb % 16 == 0 &&
                          (q.out_inst_stride * 2) % 16 == 0 &&
                          enc(&cm.st, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, q.out, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            }
            if (EE > 0 && !tma_in) return DRT3D_ERR_UNSUPPORTED;      // E > 0 needs the brick load: the caller falls back
            kern<<<grid, SG::THREADS, SG::SMEM + 16, st>>>(q, zmap, cm, tma_in, tma_out);
            return DRT3D_OK;
        };
        if constexpr (K == 4 && T == 64) {
            if (half) return go(IntPair<4, 32>{});
#ifndef D3_SWAR_E8
#define D3_SWAR_E8 0                    // measured (bit-exact): cfg3 first pass 0.3289 vs 0.3305 ms, N = 128 0.1341 vs 0.1321: neutral, off
#endif
            if constexpr (RS == 8 && D3_SWAR_E8 && D3_SWAR_TMA_STAGE) {
                // the TMA-staged kernel with whole stored chunks (SwarGeom, E = 8)
                if (prm.N >= D3_SWAR_TMA_MIN_N && prm.vec_ok) {
                    const drt3d_status r = go(IntPair<RS, T, 8>{});
                    if (r != DRT3D_ERR_UNSUPPORTED) return r;
                }
            }
        }
        return go(IntPair<RS, T>{});
    }
    using G = DrtGeom<K, R, T, !FIRST && sizeof(In) == 2>;
    auto kern = drt_pass_kernel<K, R, T, In, Acc, Out, FIRST, FINAL>;
    static std::atomic<uint32_t> smem_done{0};
    if (!set_smem_once(kern, G::SMEM, smem_done)) return DRT3D_ERR_CUDA;
    // intermediate outputs are stored pre-shifted by up to one chunk: cover one extra chunk
    const int ntiles = (prm.out_width + (FINAL ? 0 : 16 / (int)sizeof(Out)) + T - 1) / T;
    const long long groups = 1LL << (2 * (prm.c + prm.m));
    dim3 grid(ntiles, (unsigned)groups, ninst);
    CUtensorMap omap;
    std::memset(&omap, 0, sizeof(omap));
    prm.tma_store = 0;
#ifdef D3_NO_TMA_STORE
    constexpr bool no_tma = true;      // measurement builds: direct 16-byte stores
#else
    constexpr bool no_tma = false;
#endif
    if constexpr (FINAL && sizeof(Out) == 4) {
        constexpr int S = 1 << K;
        if (!no_tma && prm.layout == 0 && prm.m == 0 && prm.out_width % T == 0 && S * S * T * 4 <= G::SMEM &&
            make_out_map(&omap, prm.out, prm.N, prm.inst_total, T, S,
                         drt_warp_store<K, R, T, !FIRST && sizeof(In) == 2, FINAL>()    ? 4
                         : drt_hybrid_store<K, R, T, !FIRST && sizeof(In) == 2, FINAL>() ? S / 2
                                                                                        : S,
                         std::is_same<Out, float>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                         : CU_TENSOR_MAP_DATA_TYPE_UINT32))
            prm.tma_store = 1;
    }
    // the in-place residual (out <- out - A f) needs the fp32 CTA-wide TMA reduce path
    if ((prm.reduce_sub || prm.sq_part) && !(FINAL && std::is_same<Out, float>::value && prm.tma_store &&
                            !drt_warp_store<K, R, T, !FIRST && sizeof(In) == 2, FINAL>() &&
                            !drt_hybrid_store<K, R, T, !FIRST && sizeof(In) == 2, FINAL>()))
        return DRT3D_ERR_UNSUPPORTED;
    if constexpr (!FIRST && D3_PDL) {
        // programmatic dependent launch: scheduled while the previous kernel on the stream finishes
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(G::THREADS);
        cfg.dynamicSmemBytes = G::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, prm, omap) != cudaSuccess) return DRT3D_ERR_CUDA;
        return DRT3D_OK;
    }
    kern<<<grid, G::THREADS, G::SMEM, st>>>(prm, omap);
    return DRT3D_OK;
}

template <class In, class Acc, class Out, bool FIRST, bool FINAL>
drt3d_status launch_drt(int K, const DrtPass &prm, int ninst, cudaStream_t st) {
    switch (K) {
        case 1: return launch_drt_k<1, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
        case 2: return launch_drt_k<2, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
        case 3: return launch_drt_k<3, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
        case 4: return launch_drt_k<4, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
    }
    return DRT3D_ERR_UNSUPPORTED;
}

// ---- DJT kernel selection
template <int K> struct DjtTile;
template <> struct DjtTile<1> { static constexpr int R = 8, T1 = 8, T2 = 64; };
template <> struct DjtTile<2> { static constexpr int R = 8, T1 = 8, T2 = 64; };
#ifndef D3_DJT3_T1
#define D3_DJT3_T1 8
#endif
#ifndef D3_DJT3_T2
#define D3_DJT3_T2 32      // swept 16 / 32 / 64 / 128 (T1 = 4 / 8 / 16 / 32): T1 8 x T2 32 best on cfg4
#endif
#ifndef D3_DJT3_R
#define D3_DJT3_R 8
#endif
template <> struct DjtTile<3> { static constexpr int R = D3_DJT3_R, T1 = D3_DJT3_T1, T2 = D3_DJT3_T2; };
template <> struct DjtTile<4> { static constexpr int R = 8, T1 = 4, T2 = 64; };

template <int K, class In, class Acc, class Out, bool FIRST, bool FINAL>
drt3d_status launch_djt_k(DjtPass prm, int ninst, cudaStream_t st) {
#ifndef D3_DJT_FIRST_T1
#define D3_DJT_FIRST_T1 4      // first passes: 4-row tiles (twice the CTAs of 8 at N=64: cfg4 -2%)
#endif
    constexpr int R = DjtTile<K>::R, T2 = DjtTile<K>::T2;
    constexpr int T1 = (FIRST && D3_DJT_FIRST_T1 > 0) ? D3_DJT_FIRST_T1 : DjtTile<K>::T1;
    using G = DjtGeom<K, R, T1, T2>;
    auto kern = djt_pass_kernel<K, R, T1, T2, In, Acc, Out, FIRST, FINAL>;
    static std::atomic<uint32_t> smem_done{0};
    if (!set_smem_once(kern, G::SMEM, smem_done)) return DRT3D_ERR_CUDA;
    const int nt1 = (prm.out_width + T1 - 1) / T1, nt2 = (prm.out_width + T2 - 1) / T2;
    prm.nt2 = nt2;
    const long long groups = (1LL << (2 * prm.c)) << prm.m;
    dim3 grid(nt1 * nt2, (unsigned)groups, ninst);
    // final pass: a 5D map of the output [inst][s1][s2][D1][D2] for the zero tiles' TMA stores
    CUtensorMap zmap;
    std::memset(&zmap, 0, sizeof(zmap));
    prm.zero_tma = 0;
#ifndef D3_DJT_ZERO_TMA
#define D3_DJT_ZERO_TMA 1
#endif
    if constexpr (FINAL && sizeof(Out) == 4) {
        constexpr int S = 1 << K;
        if (D3_DJT_ZERO_TMA && prm.m == 0 && prm.out_width % T1 == 0 && prm.out_width % T2 == 0 &&
            S * T1 * T2 * 4 <= G::SMEM && prm.inst_total > 0) {
            auto enc = tmap_encoder();
            const cuuint64_t W = (cuuint64_t)prm.out_width, Nn = (cuuint64_t)prm.N;
            cuuint64_t dims[5] = {W, W, Nn, Nn, (cuuint64_t)prm.inst_total};
            cuuint64_t str[4] = {W * 4, W * W * 4, W * W * 4 * Nn, W * W * 4 * Nn * Nn};
            cuuint32_t box[5] = {(cuuint32_t)T2, (cuuint32_t)T1, (cuuint32_t)S, 1, 1}, es[5] = {1, 1, 1, 1, 1};
            if (enc && enc(&zmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, prm.out, dims, str, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                prm.zero_tma = 1;
        }
    }
    if constexpr (!FIRST && D3_PDL) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(G::THREADS);
        cfg.dynamicSmemBytes = G::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, prm, zmap) == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
    }
    kern<<<grid, G::THREADS, G::SMEM, st>>>(prm, zmap);
    return DRT3D_OK;
}

template <class In, class Acc, class Out, bool FIRST, bool FINAL>
drt3d_status launch_djt(int K, const DjtPass &prm, int ninst, cudaStream_t st) {
    switch (K) {
        case 1: return launch_djt_k<1, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
        case 2: return launch_djt_k<2, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
        case 3: return launch_djt_k<3, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
        case 4: return launch_djt_k<4, In, Acc, Out, FIRST, FINAL>(prm, ninst, st);
    }
    return DRT3D_ERR_UNSUPPORTED;
}


}  // namespace d3

#define D3_DRT_CASE(SI, SO, F, L, IT, AT, OT) \
    if (sin == SI && sout == SO && first == F && fin == L) return launch_drt<IT, AT, OT, F, L>(K, prm, ninst, st);
#define D3_DJT_CASE(SI, SO, F, L, IT, AT, OT) \
    if (sin == SI && sout == SO && first == F && fin == L) return launch_djt<IT, AT, OT, F, L>(K, prm, ninst, st);
