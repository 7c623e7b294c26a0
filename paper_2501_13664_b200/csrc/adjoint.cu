// adjoint.cu -- backprojection (adjoint) of the 3D DRT of planes and of the 3D DJT of lines
// (SURVEY §8(f) F-1): the gather maps eq:invmap3Dsummation and
// eq:invmap3DJsummation run "in reversal of the order of the m loop"
// (PAPER.md:560), one kernel per stage, followed by the transpose of the seeding step and of
// the dodecant orientation (a scatter back into the original cube, accumulated over dodecants
// in a fixed order, so results are deterministic).
//
// First version: one thread per output cell and stage, gathers straight from HBM/L2 (no
// shared-memory blocking).  Integer lanes wrap mod 2^32 like the forward transform; float lanes
// accumulate in fp32 in the oracle's order (b1 outer, b2 inner).
#include "drt3d.h"

#include <cstdint>

#include "adjoint.h"

namespace d3 {

template <class T> __device__ __forceinline__ T zero_v() { return T(0); }

// ---- DRT stage m (b^{m+1} -> b^m), rows ii = sg1 + 2^m v1m + 2^(m+1) v1 (same for jj), D in [0, 3N):
//   b^m(ii, jj, d) = sum_{b1, b2} b^{m+1}(b1 + 2 sg1 + 2^(m+1) v1, b2 + 2 sg2 + 2^(m+1) v2,
//                                      d - v1m (b1 + sg1) - v2m (b2 + sg2)),  reads below 0 are 0.
template <class T>
__global__ void drt_adj_stage(const T *__restrict__ in, T *__restrict__ out, int N, int m, long long ncell) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ncell) return;
    const int W = 3 * N;
    const int d = (int)(idx % W);
    const long long row = idx / W;
    const int jj = (int)(row % N), ii = (int)(row / N);
    const int msk = (1 << m) - 1;
    const int sg1 = ii & msk, v1m = (ii >> m) & 1, v1 = ii >> (m + 1);
    const int sg2 = jj & msk, v2m = (jj >> m) & 1, v2 = jj >> (m + 1);
    T acc = zero_v<T>();
#pragma unroll
    for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
            const int dd = d - v1m * (b1 + sg1) - v2m * (b2 + sg2);
            if (dd < 0) continue;
            const int oi = b1 + (sg1 << 1) + (v1 << (m + 1)), oj = b2 + (sg2 << 1) + (v2 << (m + 1));
            acc = acc + in[((long long)oi * N + oj) * W + dd];
        }
    out[idx] = acc;
}

// ---- seeding transpose + orientation transpose: cube[c] (+)= b^0(x', y', 2N + z') with
// oriented x'_j = c_{|p_j|} or N - 1 - c_{|p_j|} (reading A)
template <class T>
__global__ void drt_adj_scatter(const T *__restrict__ b0, T *__restrict__ cube, int N, int p0, int p1, int p2,
                                bool first) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n3 = (long long)N * N * N;
    if (idx >= n3) return;
    const int c[3] = {(int)(idx / ((long long)N * N)), (int)((idx / N) % N), (int)(idx % N)};
    auto o = [&](int p) { const int a = (p < 0 ? -p : p) - 1; return p > 0 ? c[a] : N - 1 - c[a]; };
    const int x = o(p0), y = o(p1), z = o(p2);
    const T v = b0[((long long)x * N + y) * (3 * N) + 2 * N + z];
    cube[idx] = first ? v : cube[idx] + v;
}

// ---- DJT stage m: rows i = vm + 2 v + 2^(n-m) sg1 + 2^n sg2, (D1, D2) in [0, 2N)^2:
//   b^m(i, d1, d2) = sum_{b1,b2} b^{m+1}(v + 2^(n-m-1) b1 + 2^(n-m) sg1 + 2^n b2 + 2^(n+1) sg2,
//                                        d1 - vm (b1 + sg1), d2 - vm (b2 + sg2)).
// Stage n-1 reads the caller's [s1][s2][D1][D2] layout (inverse of separateS1S2: row s1 + N s2).
// Only the first 2^(n+m) rows of a stage-m buffer exist (m slope bits per axis), so a stage
// computes exactly those.
template <class T>
__global__ void djt_adj_stage(const T *__restrict__ in, T *__restrict__ out, int N, int n, int m, bool from_coef,
                              long long ncell) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ncell) return;
    const int W = 2 * N;
    const int d2 = (int)(idx % W);
    const int d1 = (int)((idx / W) % W);
    const int i = (int)(idx / ((long long)W * W));
    const int vm = i & 1, v = (i >> 1) & ((1 << (n - m - 1)) - 1);
    const int sg1 = (i >> (n - m)) & ((1 << m) - 1), sg2 = i >> n;
    T acc = zero_v<T>();
#pragma unroll
    for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
            const int e1 = d1 - vm * (b1 + sg1), e2 = d2 - vm * (b2 + sg2);
            if (e1 < 0 || e2 < 0) continue;
            int o = v + (b1 << (n - m - 1)) + (sg1 << (n - m)) + (b2 << n) + (sg2 << (n + 1));
            if (from_coef) o = (o % N) * N + o / N;          // packed s1 + N s2 -> caller row s1 N + s2
            acc = acc + in[((long long)o * W + e1) * W + e2];
        }
    out[idx] = acc;
}

template <class T>
__global__ void djt_adj_scatter(const T *__restrict__ b0, T *__restrict__ cube, int N, int p0, int p1, int p2,
                                bool first) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n3 = (long long)N * N * N;
    if (idx >= n3) return;
    const int c[3] = {(int)(idx / ((long long)N * N)), (int)((idx / N) % N), (int)(idx % N)};
    auto o = [&](int p) { const int a = (p < 0 ? -p : p) - 1; return p > 0 ? c[a] : N - 1 - c[a]; };
    const int x = o(p0), y = o(p1), z = o(p2);
    const int W = 2 * N;
    const T v = b0[((long long)x * W + N + y) * W + N + z];
    cube[idx] = first ? v : cube[idx] + v;
}

namespace {
constexpr int kThreads = 256;
inline unsigned nblk(long long n) { return (unsigned)((n + kThreads - 1) / kThreads); }
}  // namespace

template <class T>
static drt3d_status run_adj(int transform, const void *coef, int N, int n, const int8_t (*rows)[3], uint32_t mask,
                            int batch, void *cube, void *ws, cudaStream_t st, int *launches) {
    const long long W = transform == 0 ? 3LL * N : 2LL * N;
    const long long cells = transform == 0 ? (long long)N * N * W : (long long)N * N * W * W;
    const int K = __builtin_popcount(mask & 0xFFFu);
    T *buf[2] = {reinterpret_cast<T *>(ws), reinterpret_cast<T *>(ws) + cells};
    const T *cf = reinterpret_cast<const T *>(coef);
    T *cb = reinterpret_cast<T *>(cube);
    const long long n3 = (long long)N * N * N;
    int nl = 0;
    for (int b = 0; b < batch; ++b) {
        int j = 0;
        for (int k = 0; k < 12; ++k) {
            if (!((mask >> k) & 1)) continue;
            const T *src = cf + ((long long)b * K + j) * cells;
            int cur = 0;
            for (int m = n - 1; m >= 0; --m) {
                const T *in = (m == n - 1) ? src : buf[cur ^ 1];
                if (transform == 0) drt_adj_stage<T><<<nblk(cells), kThreads, 0, st>>>(in, buf[cur], N, m, cells);
                else {
                    const long long rows_m = 1LL << (n + m), ncell = rows_m * W * W;
                    djt_adj_stage<T><<<nblk(ncell), kThreads, 0, st>>>(in, buf[cur], N, n, m, m == n - 1, ncell);
                }
                ++nl;
                cur ^= 1;
            }
            const T *b0 = buf[cur ^ 1];
            if (transform == 0)
                drt_adj_scatter<T><<<nblk(n3), kThreads, 0, st>>>(b0, cb + (long long)b * n3, N, rows[k][0], rows[k][1],
                                                                  rows[k][2], j == 0);
            else
                djt_adj_scatter<T><<<nblk(n3), kThreads, 0, st>>>(b0, cb + (long long)b * n3, N, rows[k][0], rows[k][1],
                                                                  rows[k][2], j == 0);
            ++nl;
            ++j;
        }
    }
    if (launches) *launches = nl;
    return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
}

size_t adjoint_workspace_bytes(int transform, int N) {
    const long long W = transform == 0 ? 3LL * N : 2LL * N;
    const long long cells = transform == 0 ? (long long)N * N * W : (long long)N * N * W * W;
    return (size_t)(2 * cells * 4 + 255) / 256 * 256;
}

drt3d_status run_adjoint(int transform, const void *coef, int N, int n, const int8_t (*rows)[3], uint32_t mask,
                         int batch, int dtype, void *cube, void *ws, cudaStream_t st, int *launches) {
    if (dtype == DRT3D_F32) return run_adj<float>(transform, coef, N, n, rows, mask, batch, cube, ws, st, launches);
    return run_adj<uint32_t>(transform, coef, N, n, rows, mask, batch, cube, ws, st, launches);
}

}  // namespace d3
