// apps.cu -- applications on top of the transforms.
//
//   * coefficient threshold (ray denoising, PAPER.md:448 and fig:output3DDJT: "a thresholding of
//     the highest amplitude coefficients, and subsequent backprojection"): keep c when
//     c * den >= num * max(c) (reading R19, exact in int64), else 0;
//   * coefficient selection: keep the flagged coefficients ("When those planes are backprojected,
//     they correspond to the walls": select, then drt3d_planes_adjoint);
//   * plane detection: the global argmax plane (R20: ties to the smallest
//     stacked index), then every coefficient above the R19 threshold that is a relative maximum
//     in its dodecant's (s1, s2, D) 26-neighbourhood (R21: >= all neighbours, > those with a
//     smaller index) and whose plane normal is orthogonal to the argmax plane's (R22: integer
//     normals (s1, s2, -(N-1)) mapped through the signed axis permutation of the orientation
//     table, |cos| <= onum/oden tested as (n.m)^2 oden^2 <= onum^2 |n|^2 |m|^2 in 128-bit integers).
//
// Reductions are two-pass with a fixed grid (deterministic).  All on the caller's stream.
#include "drt3d.h"

#include <cstdint>

#include <cuda_runtime.h>

namespace d3 {
namespace apps {

constexpr int kBlocks = 1184;                 // 8 x 148 SMs, fixed: the reduction order is fixed
constexpr int kThreads = 256;

struct VI {
    int v;
    long long i;
};

__device__ __forceinline__ VI better(VI a, VI b) {          // larger value, then smaller index
    return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}

__device__ VI block_best(VI x) {
    __shared__ int sv[kThreads / 32];
    __shared__ long long si[kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        VI y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o)};
        x = better(x, y);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sv[w] = x.v;
        si[w] = x.i;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        x = threadIdx.x < (int)(blockDim.x >> 5) ? VI{sv[threadIdx.x], si[threadIdx.x]} : VI{INT32_MIN, -1};
        if (x.i < 0) x.i = 0x7fffffffffffffffLL;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            VI y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o)};
            x = better(x, y);
        }
    }
    return x;                                              // valid in thread 0
}

// pass 1: per-block best (value, index); pass 2: one block over the partials.  16-byte loads,
// four in flight per thread (vector v covers elements 4v .. 4v+3); a thread visits increasing
// indices, so `>` keeps the first of equal values; the scalar tail follows.
__global__ void __launch_bounds__(kThreads) argmax_partial(const int32_t *__restrict__ c, size_t n, int *pv,
                                                             long long *pi) {
    VI b{INT32_MIN, 0x7fffffffffffffffLL};
    auto take = [&](int v, size_t i) {
        if (v > b.v || b.i == 0x7fffffffffffffffLL) b = VI{v, (long long)i};
    };
    const bool vec = (reinterpret_cast<uintptr_t>(c) & 15) == 0;
    const size_t nv = vec ? n / 4 : 0;
    const int4 *c4 = reinterpret_cast<const int4 *>(c);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t v0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v0 + 3 * stride < nv; v0 += 4 * stride) {
        int4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = __ldg(c4 + v0 + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const size_t e = 4 * (v0 + u * stride);
            take(q[u].x, e);
            take(q[u].y, e + 1);
            take(q[u].z, e + 2);
            take(q[u].w, e + 3);
        }
    }
    for (; v0 < nv; v0 += stride) {
        const int4 q = __ldg(c4 + v0);
        const size_t e = 4 * v0;
        take(q.x, e);
        take(q.y, e + 1);
        take(q.z, e + 2);
        take(q.w, e + 3);
    }
    for (size_t i = 4 * nv + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) take(c[i], i);
    b = block_best(b);
    if (threadIdx.x == 0) {
        pv[blockIdx.x] = b.v;
        pi[blockIdx.x] = b.i;
    }
}

__global__ void __launch_bounds__(kThreads) argmax_final(const int *pv, const long long *pi, int nb, int *max_out,
                                                           long long *idx_out, long long *user_idx) {
    VI b{INT32_MIN, 0x7fffffffffffffffLL};
    for (int i = threadIdx.x; i < nb; i += blockDim.x) b = better(b, VI{pv[i], pi[i]});
    b = block_best(b);
    if (threadIdx.x == 0) {
        *max_out = b.v;
        *idx_out = b.i;
        if (user_idx) *user_idx = b.i;
    }
}

__global__ void threshold_kernel(const int32_t *c, size_t n, int num, int den, const int *mx,
                                 int32_t *out) {              // out may alias c (same index)
    const long long lim = (long long)num * *mx;
    auto keep = [&](int v) { return (long long)v * den >= lim ? v : 0; };
    const bool vec = ((reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    const size_t nv = vec ? n / 4 : 0, stride = (size_t)gridDim.x * blockDim.x;
    for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
        const int4 q = reinterpret_cast<const int4 *>(c)[v];
        reinterpret_cast<int4 *>(out)[v] = make_int4(keep(q.x), keep(q.y), keep(q.z), keep(q.w));
    }
    for (size_t i = 4 * nv + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = keep(c[i]);
}

// out[i] = flags[i] ? c[i] : 0 (16-byte groups of four; the flags as one 32-bit word)
__global__ void select_kernel(const int32_t *__restrict__ c, const uint8_t *__restrict__ flags, size_t n,
                              int32_t *__restrict__ out) {
    const bool vec = ((reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(out)) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(flags) & 3) == 0;
    const size_t nv = vec ? n / 4 : 0, stride = (size_t)gridDim.x * blockDim.x;
    for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
        const int4 q = reinterpret_cast<const int4 *>(c)[v];
        const uint32_t f = reinterpret_cast<const uint32_t *>(flags)[v];
        reinterpret_cast<int4 *>(out)[v] = make_int4((f & 0xFFu) ? q.x : 0, (f & 0xFF00u) ? q.y : 0,
                                                     (f & 0xFF0000u) ? q.z : 0, (f & 0xFF000000u) ? q.w : 0);
    }
    for (size_t i = 4 * nv + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = flags[i] ? c[i] : 0;
}

struct DetectArgs {
    int N, K;
    int num, den, onum, oden;
    int8_t rows[12][3];          // orientation rows of the mask's dodecants, in stacked order
};

__device__ __forceinline__ void normal(const DetectArgs &a, int j, int s1, int s2, long long (&n)[3]) {
    const long long np[3] = {s1, s2, -(long long)(a.N - 1)};
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const int p = a.rows[j][t];
        n[(p < 0 ? -p : p) - 1] = p > 0 ? np[t] : -np[t];
    }
}

// flags[i] = 1 for the argmax and for the coefficients passing threshold, orthogonality and
// relative-maximum tests; 0 otherwise.  One thread per coefficient (grid-stride).
__global__ void __launch_bounds__(kThreads) detect_kernel(const int32_t *__restrict__ c, const DetectArgs a,
                                                          const int *mx, const long long *am, uint8_t *flags) {
    const int N = a.N, W = 3 * a.N;
    const size_t per = (size_t)N * N * W, n = per * a.K;
    const long long amax = *am;
    const long long lim = (long long)a.num * *mx;
    // the argmax plane's normal
    long long m[3];
    {
        const long long j0 = amax / per, r = amax % per;
        normal(a, (int)j0, (int)(r / ((long long)N * W)), (int)((r / W) % N), m);
    }
    const long long mm = m[0] * m[0] + m[1] * m[1] + m[2] * m[2];
    auto decide = [&](int v, size_t i) -> uint8_t {
        if ((long long)i == amax) return 1;
        if ((long long)v * a.den < lim) return 0;
        const int j = (int)(i / per);
        const size_t r = i - (size_t)j * per;
        const int s1 = (int)(r / ((size_t)N * W)), s2 = (int)((r / W) % N), D = (int)(r % W);
        long long nv[3];
        normal(a, j, s1, s2, nv);
        const long long dot = nv[0] * m[0] + nv[1] * m[1] + nv[2] * m[2];
        const long long nn = nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2];
        // |cos| <= onum / oden as (n.m)^2 oden^2 <= onum^2 |n|^2 |m|^2, exactly: each side is below
        // (3 N^2)^2 * 2^62 < 2^128 for N <= 1024 and 31-bit onum / oden
        using u128 = unsigned __int128;
        const u128 dd = (u128)(unsigned long long)(dot < 0 ? -dot : dot);
        const u128 lhs = dd * dd * (u128)(unsigned long long)a.oden * (u128)(unsigned long long)a.oden;
        const u128 rhs = (u128)(unsigned long long)a.onum * (u128)(unsigned long long)a.onum * (u128)(unsigned long long)nn *
                         (u128)(unsigned long long)mm;
        if (lhs > rhs) return 0;
        const int32_t *base = c + (size_t)j * per;
        for (int d1 = -1; d1 <= 1; ++d1)
            for (int d2 = -1; d2 <= 1; ++d2)
                for (int d3 = -1; d3 <= 1; ++d3) {
                    if (d1 == 0 && d2 == 0 && d3 == 0) continue;
                    const int t1 = s1 + d1, t2 = s2 + d2, t3 = D + d3;
                    if (t1 < 0 || t1 >= N || t2 < 0 || t2 >= N || t3 < 0 || t3 >= W) continue;
                    const int u = base[((size_t)t1 * N + t2) * W + t3];
                    const bool smaller = d1 < 0 || (d1 == 0 && (d2 < 0 || (d2 == 0 && d3 < 0)));
                    if (u > v || (smaller && u == v)) return 0;
                }
        return 1;
    };
    // W = 3N is a multiple of 4 for N >= 4, so 4-element groups never straddle rows; the flags go
    // out as one 32-bit word per group
    const bool vec = (N >= 4) && ((reinterpret_cast<uintptr_t>(c) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(flags) & 3) == 0);
    const size_t nv = vec ? n / 4 : 0, stride = (size_t)gridDim.x * blockDim.x;
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < nv; g += stride) {
        const int4 q = __ldg(reinterpret_cast<const int4 *>(c) + g);
        const size_t e = 4 * g;
        const int qv[4] = {q.x, q.y, q.z, q.w};
        uint32_t word = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const bool cand = (long long)qv[t] * a.den >= lim || (long long)(e + t) == amax;
            if (cand) word |= (uint32_t)decide(qv[t], e + t) << (8 * t);
        }
        reinterpret_cast<uint32_t *>(flags)[g] = word;
    }
    for (size_t i = 4 * nv + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        flags[i] = decide(c[i], i);
}

// workspace: partial values, partial indices, max, argmax
struct Ws {
    int *pv;
    long long *pi;
    int *mx;
    long long *am;
};
constexpr size_t kPiOff = (4 * kBlocks + 255) / 256 * 256;
constexpr size_t kMxOff = kPiOff + (8 * kBlocks + 255) / 256 * 256;
inline Ws carve(void *ws) {
    unsigned char *w = reinterpret_cast<unsigned char *>(ws);
    Ws s;
    s.pv = reinterpret_cast<int *>(w);
    s.pi = reinterpret_cast<long long *>(w + kPiOff);
    s.mx = reinterpret_cast<int *>(w + kMxOff);
    s.am = reinterpret_cast<long long *>(w + kMxOff + 256);
    return s;
}
constexpr size_t kWsBytes = kMxOff + 512;

inline void run_argmax(const int32_t *c, size_t n, const Ws &w, long long *user_idx, cudaStream_t st) {
    argmax_partial<<<kBlocks, kThreads, 0, st>>>(c, n, w.pv, w.pi);
    argmax_final<<<1, kThreads, 0, st>>>(w.pv, w.pi, kBlocks, w.mx, w.am, user_idx);
}

}  // namespace apps
}  // namespace d3

using namespace d3::apps;

extern "C" size_t drt3d_apps_workspace_size(void) { return kWsBytes; }

extern "C" drt3d_status drt3d_coef_argmax(const int32_t *coef, size_t n, long long *index, void *ws, size_t ws_bytes,
                                          void *stream) {
    if (!coef || !index || n == 0) return DRT3D_ERR_INVALID_ARG;
    if (!ws || ws_bytes < kWsBytes || (reinterpret_cast<uintptr_t>(ws) & 255)) return DRT3D_ERR_WORKSPACE;
    run_argmax(coef, n, carve(ws), index, reinterpret_cast<cudaStream_t>(stream));
    return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
}

extern "C" drt3d_status drt3d_coef_threshold(const int32_t *coef, size_t n, int num, int den, int32_t *out, void *ws,
                                             size_t ws_bytes, void *stream) {
    if (!coef || !out || n == 0 || num < 0 || den <= 0) return DRT3D_ERR_INVALID_ARG;
    if (!ws || ws_bytes < kWsBytes || (reinterpret_cast<uintptr_t>(ws) & 255)) return DRT3D_ERR_WORKSPACE;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Ws w = carve(ws);
    run_argmax(coef, n, w, nullptr, st);
    threshold_kernel<<<kBlocks, kThreads, 0, st>>>(coef, n, num, den, w.mx, out);
    return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
}

extern "C" drt3d_status drt3d_coef_select(const int32_t *coef, const uint8_t *flags, size_t n, int32_t *out,
                                          void *stream) {
    if (!coef || !flags || !out || n == 0) return DRT3D_ERR_INVALID_ARG;
    select_kernel<<<kBlocks, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(coef, flags, n, out);
    return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
}

extern "C" drt3d_status drt3d_detect_planes(const int32_t *coef, int N, uint32_t mask, int num, int den, int onum,
                                            int oden, const drt3d_opts *opts, uint8_t *flags, long long *argmax,
                                            void *ws, size_t ws_bytes, void *stream) {
    if (!coef || !flags || N < 2 || N > 1024 || (N & (N - 1)) || mask == 0 || mask >= (1u << 12))
        return DRT3D_ERR_INVALID_ARG;
    if (num < 0 || den <= 0 || onum < 0 || oden <= 0) return DRT3D_ERR_INVALID_ARG;
    if (!ws || ws_bytes < kWsBytes || (reinterpret_cast<uintptr_t>(ws) & 255)) return DRT3D_ERR_WORKSPACE;
    const int table = opts ? opts->table : DRT3D_TABLE_HEMISPHERE;
    int8_t rows[36];
    drt3d_status s = drt3d_orientation_table(table, 0, rows);
    if (s != DRT3D_OK) return s;
    DetectArgs a{};
    a.N = N;
    a.num = num;
    a.den = den;
    a.onum = onum;
    a.oden = oden;
    for (int k = 0; k < 12; ++k)
        if ((mask >> k) & 1) {
            for (int t = 0; t < 3; ++t) a.rows[a.K][t] = rows[3 * k + t];
            ++a.K;
        }
    const size_t n = (size_t)a.K * N * N * 3 * N;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Ws w = carve(ws);
    run_argmax(coef, n, w, argmax, st);
    detect_kernel<<<4 * kBlocks, kThreads, 0, st>>>(coef, a, w.mx, w.am, flags);
    return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
}
