// adjoint.cu -- backprojection (adjoint) of the 3D DRT of planes and of the 3D DJT of lines
// (SURVEY §8(f) F-1): the gather maps eq:invmap3Dsummation and
// eq:invmap3DJsummation run "in reversal of the order of the m loop"
// (PAPER.md:560), one kernel per stage, followed by the transpose of the seeding step and of
// the dodecant orientation (a scatter back into the original cube, accumulated over dodecants
// in a fixed order, so results are deterministic).
//
// One thread per output cell; a launch applies L consecutive gather stages at once (their
// composition: 4^L reads per cell for both transforms), straight from
// HBM/L2 with no shared-memory blocking.  Integer lanes wrap mod 2^32 like the forward transform;
// float lanes accumulate in fp32.
#include "drt3d.h"

#include <cstdint>
#include <cstdlib>

#include "adjoint.h"
#include "adjoint_pass.cuh"

namespace d3 {

template <class T> __device__ __forceinline__ T zero_v() { return T(0); }

// ---- DRT: L consecutive stages m_lo..m_lo+L-1 in one launch (b^{m_lo+L} -> b^{m_lo}).
// Stage m (b^{m+1} -> b^m), rows ii = sg1 + 2^m v1m + 2^(m+1) v1 (same for jj), D in [0, 3N):
//   b^m(ii, jj, d) = sum_{b1, b2} b^{m+1}(b1 + 2 sg1 + 2^(m+1) v1, b2 + 2 sg2 + 2^(m+1) v2,
//                                      d - v1m (b1 + sg1) - v2m (b2 + sg2)),  reads below 0 are 0.
// The maps act on the two row axes separately and all shifts are >= 0, so L stages compose into
// 2^L (row, shift) pairs per axis; a composite term whose final index is >= 0 had every
// intermediate index >= 0 too, hence the composition is exact (only the fp32 summation order
// differs from the stage-by-stage oracle).
template <int L>
__device__ __forceinline__ void drt_axis_terms(int ii, int m_lo, int (&row)[1 << L], int (&sh)[1 << L]) {
    row[0] = ii;
    sh[0] = 0;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const int m = m_lo + l, cnt = 1 << l;
#pragma unroll
        for (int t = cnt - 1; t >= 0; --t) {
            const int r = row[t], s = sh[t];
            const int sg = r & ((1 << m) - 1), vm = (r >> m) & 1, v = r >> (m + 1);
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                row[2 * t + b] = b + (sg << 1) + (v << (m + 1));
                sh[2 * t + b] = s + vm * (b + sg);
            }
        }
    }
}

// grid: x = output row ii * N + jj; the block's threads stride along D, so the row's terms are
// set up once per thread rather than once per cell
template <class T, int L>
__global__ void drt_adj_stage(const T *__restrict__ in, T *__restrict__ out, int N, int m_lo) {
    const int W = 3 * N;
    const int ii = blockIdx.x / N, jj = blockIdx.x - ii * N;
    int r1[1 << L], s1[1 << L], r2[1 << L], s2[1 << L];
    drt_axis_terms<L>(ii, m_lo, r1, s1);
    drt_axis_terms<L>(jj, m_lo, r2, s2);
    constexpr int NT = 1 << (2 * L);
    // per-term base pointers pre-offset by the term's shift: term t of cell d reads p[t][d]
    // when d >= sh[t] (never dereferenced otherwise)
    const T *p[NT];
    int sh[NT];
#pragma unroll
    for (int a = 0; a < (1 << L); ++a)
#pragma unroll
        for (int b = 0; b < (1 << L); ++b) {
            const int t = a * (1 << L) + b;
            sh[t] = s1[a] + s2[b];
            p[t] = in + ((long long)(r1[a] * N + r2[b]) * W - sh[t]);
        }
    // walk the term pointers along D (kept in registers: the empty asm stops the compiler from
    // rebuilding each address from the kernel parameter per load)
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        p[t] += threadIdx.x;
        asm volatile("" : "+l"(p[t]));
    }
    T *dst = out + (size_t)blockIdx.x * W + threadIdx.x;
    for (int d = threadIdx.x; d < W; d += blockDim.x) {
        T acc = zero_v<T>();
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (d >= sh[t]) acc = acc + __ldg(p[t]);
            p[t] += blockDim.x;
        }
        *dst = acc;
        dst += blockDim.x;
    }
}

// ---- DRT, shared-memory butterfly: the stage map sends the two output rows sg + 2^m vm + 2^(m+1) v
// (vm = 0, 1) to the same two input rows 2 sg + b + 2^(m+1) v (b = 0, 1), per axis.  Groups of
// 2^L rows per axis are therefore closed under L consecutive stages: a block loads its 4^L input
// rows (level m_lo + L) into shared memory once, runs the L gather stages there (double-buffered,
// whole rows of W = 3N cells, so every shifted read is in the buffer), and writes its 4^L output
// rows (level m_lo).  HBM traffic per L stages: one read and one write of the stage buffer.
// Tables (built by two threads per block): per level and axis the rows each slot holds, and per
// stage, output row q and term k = 2 b1 + b2, the buffer offset (slot row * W - shift) and shift.
template <int L>
struct BflyTab {
    int row[L + 1][2][1 << L];
    int off[L][1 << (2 * L)][4];
    int sh[L][1 << (2 * L)][4];
};

template <int L>
__device__ void bfly_tables(BflyTab<L> &tab, int N, int W, int m_lo) {
    constexpr int S = 1 << L;
    __shared__ int src[L][2][S][2], shx[L][2][S][2];
    if (threadIdx.x < 2) {
        // group id per axis: the bits of the level-m_lo row other than m_lo .. m_lo+L-1
        const int ng = N >> L, ax = threadIdx.x;
        const int g = ax == 0 ? (int)blockIdx.x / ng : (int)blockIdx.x % ng;
        const int lowm = (1 << m_lo) - 1;
        for (int u = 0; u < S; ++u) tab.row[0][ax][u] = (g & lowm) | (u << m_lo) | ((g >> m_lo) << (m_lo + L));
        for (int l = 0; l < L; ++l) {
            const int m = m_lo + l;
            int cnt = 0;
            for (int u = 0; u < S; ++u) {
                const int r = tab.row[l][ax][u];
                const int sg = r & ((1 << m) - 1), vm = (r >> m) & 1, v = r >> (m + 1);
                for (int b = 0; b < 2; ++b) {
                    const int x = b + (sg << 1) + (v << (m + 1));
                    int k = 0;
                    while (k < cnt && tab.row[l + 1][ax][k] != x) ++k;
                    if (k == cnt) tab.row[l + 1][ax][cnt++] = x;     // closure: cnt ends at exactly S
                    src[l][ax][u][b] = k;
                    shx[l][ax][u][b] = vm * (b + sg);
                }
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < L * S * S * 4; e += blockDim.x) {
        const int k = e & 3, q = (e >> 2) % (S * S), l = (e >> 2) / (S * S);
        const int u1 = q / S, u2 = q % S, b1 = k >> 1, b2 = k & 1;
        const int sh = shx[l][0][u1][b1] + shx[l][1][u2][b2];
        tab.sh[l][q][k] = sh;
        tab.off[l][q][k] = (src[l][0][u1][b1] * S + src[l][1][u2][b2]) * W - sh;
    }
    __syncthreads();
}

// One buffer of 4^L whole rows; a stage computes every output this thread owns (rows q, columns
// d = tid + 256 c, c < NC) into registers, then all threads write back after a barrier.
template <class T, int L, int NC>
__global__ void __launch_bounds__(256) drt_adj_bfly(const T *__restrict__ in, T *__restrict__ out, int N, int m_lo) {
    extern __shared__ __align__(16) unsigned char adj_smem[];
    constexpr int S = 1 << L, R = S * S;
    const int W = 3 * N;
    T *buf = reinterpret_cast<T *>(adj_smem);
    __shared__ BflyTab<L> tab;
    bfly_tables<L>(tab, N, W, m_lo);
    const int tid = threadIdx.x;
    // load the level-(m_lo + L) rows: 16-byte cp.async when rows are 16-byte multiples
    const bool vec = (W % 4) == 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const T *g = in + ((size_t)tab.row[L][0][q / S] * N + tab.row[L][1][q % S]) * W;
        T *dst = buf + q * W;
        if (vec) {
            for (int d = tid * 4; d < W; d += 1024) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + d);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g + d) : "memory");
            }
        } else {
            for (int d = tid; d < W; d += 256) dst[d] = __ldg(g + d);
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    // stages m_lo + L - 1 .. m_lo (the adjoint runs them in decreasing m)
    for (int l = L - 1; l >= 0; --l) {
        T acc[R][NC];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            int off[4], sh[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                off[k] = tab.off[l][q][k];
                sh[k] = tab.sh[l][q][k];
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int d = tid + 256 * c;
                T a = zero_v<T>();
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (d < W && d >= sh[k]) a = a + buf[off[k] + d];
                acc[q][c] = a;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int d = tid + 256 * c;
                if (d < W) buf[q * W + d] = acc[q][c];
            }
        __syncthreads();
    }
    // store the level-m_lo rows
#pragma unroll
    for (int q = 0; q < R; ++q) {
        T *g = out + ((size_t)tab.row[0][0][q / S] * N + tab.row[0][1][q % S]) * W;
        const T *src = buf + q * W;
        if (vec) {
            for (int d = tid * 4; d < W; d += 1024)
                *reinterpret_cast<uint4 *>(g + d) = *reinterpret_cast<const uint4 *>(src + d);
        } else {
            for (int d = tid; d < W; d += 256) g[d] = src[d];
        }
    }
}

// ---- seeding transpose + orientation transpose: cube[c] (+)= b^0(x', y', 2N + z') with
// oriented x'_j = c_{|p_j|} or N - 1 - c_{|p_j|} (reading A).
// grid: x = c0 * N + c1, threads along c2.
__device__ __forceinline__ int orient(const int (&c)[3], int p, int N) {
    const int a = (p < 0 ? -p : p) - 1;
    const int v = a == 0 ? c[0] : (a == 1 ? c[1] : c[2]);
    return p > 0 ? v : N - 1 - v;
}

// b0: level-0 rows (x', y') with pitch `pitch`, z' at element off + z'
template <class T>
__global__ void drt_adj_scatter(const T *__restrict__ b0, T *__restrict__ cube, int N, int p0, int p1, int p2,
                                bool first, int pitch, int off) {
    const int c2 = blockIdx.y * blockDim.x + threadIdx.x;
    if (c2 >= N) return;
    const int c0 = blockIdx.x / N;
    const int c[3] = {c0, (int)blockIdx.x - c0 * N, c2};
    const int x = orient(c, p0, N), y = orient(c, p1, N), z = orient(c, p2, N);
    const T v = b0[((size_t)x * N + y) * pitch + off + z];
    const size_t idx = (size_t)blockIdx.x * N + c2;
    cube[idx] = first ? v : cube[idx] + v;
}

// Transposing variant for orientations whose z' is not the cube's fast axis c2: a 32 x 32 tile of
// the (c_az, c2) plane (c_az = the cube axis carrying z') goes through shared memory so that the
// b0 reads run along z' and the cube read-modify-writes along c2.  grid (N/32 c2 tiles,
// N/32 c_az tiles, N values of the third axis), block 32 x 8.
template <class T>
__global__ void drt_adj_scatter_t(const T *__restrict__ b0, T *__restrict__ cube, int N, int p0, int p1, int p2,
                                  bool first, int pitch, int off) {
    __shared__ T tile[32][33];
    const int az = (p2 < 0 ? -p2 : p2) - 1;                         // 0 or 1 here
    const int ao = 1 - az;                                           // the remaining axis
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c2b = blockIdx.x * 32, czb = blockIdx.y * 32, co = blockIdx.z;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int c[3];
        c[2] = c2b + ty + 8 * i;
        c[az] = czb + tx;
        c[ao] = co;
        const int x = orient(c, p0, N), y = orient(c, p1, N), z = orient(c, p2, N);
        tile[ty + 8 * i][tx] = b0[((size_t)x * N + y) * pitch + off + z];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int c[3];
        c[2] = c2b + tx;
        c[az] = czb + ty + 8 * i;
        c[ao] = co;
        const size_t idx = ((size_t)c[0] * N + c[1]) * N + c[2];
        const T v = tile[tx][ty + 8 * i];
        cube[idx] = first ? v : cube[idx] + v;
    }
}

template <class T>
void drt_scatter(const T *b0, T *cube, int N, const int8_t *row, bool first, int pitch, int off, cudaStream_t st) {
    const int p2 = row[2];
    if ((p2 == 3 || p2 == -3) || N < 32) {
        const unsigned t = N >= 256 ? 256u : (unsigned)((N + 31) / 32 * 32);
        drt_adj_scatter<T><<<dim3((unsigned)(N * N), (unsigned)((N + t - 1) / t)), t, 0, st>>>(b0, cube, N, row[0], row[1],
                                                                                              p2, first, pitch, off);
    } else {
        drt_adj_scatter_t<T><<<dim3((unsigned)(N / 32), (unsigned)(N / 32), (unsigned)N), dim3(32, 8), 0, st>>>(
            b0, cube, N, row[0], row[1], p2, first, pitch, off);
    }
}

// All dodecants of a chunk at once: cube[c] (=|+=) sum_j l0_j[orient_j(c)] in the fixed order j
// (deterministic).  A CTA owns an 8 (c0) x 8 (c1) x 32 (c2) tile; for every dodecant the matching
// box of its level-0 rows is read along z' (runs of 8 or 32 elements: whole 32-byte sectors) into
// shared memory in cube order, then added to the CTA's registers; one coalesced write at the end.
constexpr int kGatherMax = 12;
struct GatherArgs {
    int D;                               // dodecants in this chunk
    int8_t rows[kGatherMax][3];
};
template <class T>
__global__ void __launch_bounds__(256) drt_adj_gather(const T *__restrict__ l0, long long l0_stride, int pitch, int N,
                                                      const GatherArgs g, T *__restrict__ cube, bool first) {
    __shared__ T sm[8 * 8 * 33];                                      // [c0 8][c1 8][c2 32 + 1 pad]
    const int tid = threadIdx.x;
    const int T0 = (int)blockIdx.z * 8, T1 = (int)blockIdx.y * 8, T2 = (int)blockIdx.x * 32;
    // per cube axis a: tile origin, extent (log2) and shared-memory stride; scalar selects only
    // (runtime-indexed arrays would go to local memory)
    auto org = [&](int a) { return a == 0 ? T0 : (a == 1 ? T1 : T2); };
    auto lex = [&](int a) { return a == 2 ? 5 : 3; };
    auto str = [&](int a) { return a == 0 ? 8 * 33 : (a == 1 ? 33 : 1); };
    T acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = T(0);
    for (int j = 0; j < g.D; ++j) {
        const int p0 = g.rows[j][0], p1 = g.rows[j][1], p2 = g.rows[j][2];
        const int a0 = (p0 < 0 ? -p0 : p0) - 1, a1 = (p1 < 0 ? -p1 : p1) - 1, a2 = (p2 < 0 ? -p2 : p2) - 1;
        const int l0e = lex(a0), l1e = lex(a1), l2e = lex(a2);
        // lowest oriented coordinate of the box along x', y', z'
        const int o0 = p0 > 0 ? org(a0) : N - org(a0) - (1 << l0e);
        const int o1 = p1 > 0 ? org(a1) : N - org(a1) - (1 << l1e);
        const int o2 = p2 > 0 ? org(a2) : N - org(a2) - (1 << l2e);
        // shared index of oriented offset (xo, yo, zo): base + xo m0 + yo m1 + zo m2
        const int m0 = p0 > 0 ? str(a0) : -str(a0), m1 = p1 > 0 ? str(a1) : -str(a1), m2 = p2 > 0 ? str(a2) : -str(a2);
        const int base = (p0 > 0 ? 0 : ((1 << l0e) - 1) * str(a0)) + (p1 > 0 ? 0 : ((1 << l1e) - 1) * str(a1)) +
                         (p2 > 0 ? 0 : ((1 << l2e) - 1) * str(a2));
        const T *src = l0 + (long long)j * l0_stride + ((size_t)o0 * N + o1) * pitch + o2;
        // 16-byte loads along z' (the box extent along z' is 8 or 32, origins are multiples of 8,
        // the pitch a multiple of 4): item = 4 consecutive z', 2 items per thread
        const int lq = l2e - 2;
        uint4 v[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int e = tid + 256 * i;
            const int zq = e & ((1 << lq) - 1), yo = (e >> lq) & ((1 << l1e) - 1), xo = e >> (lq + l1e);
            v[i] = __ldg(reinterpret_cast<const uint4 *>(src + ((size_t)xo * N + yo) * pitch + 4 * zq));
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int e = tid + 256 * i;
            const int zq = e & ((1 << lq) - 1), yo = (e >> lq) & ((1 << l1e) - 1), xo = e >> (lq + l1e);
            const int b = base + xo * m0 + yo * m1 + 4 * zq * m2;
            const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) sm[b + k * m2] = Lane<T>::get(w[k]);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = acc[i] + sm[(i * 8 + (tid >> 5)) * 33 + (tid & 31)];
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const size_t idx = ((size_t)(T0 + i) * N + T1 + (tid >> 5)) * N + T2 + (tid & 31);
        cube[idx] = first ? acc[i] : cube[idx] + acc[i];
    }
}

// ---- DJT stage m: rows i = vm + 2 v + 2^(n-m) sg1 + 2^n sg2, (D1, D2) in [0, 2N)^2:
//   b^m(i, d1, d2) = sum_{b1,b2} b^{m+1}(v + 2^(n-m-1) b1 + 2^(n-m) sg1 + 2^n b2 + 2^(n+1) sg2,
//                                        d1 - vm (b1 + sg1), d2 - vm (b2 + sg2)).
// Stage n-1 reads the caller's [s1][s2][D1][D2] layout (inverse of separateS1S2: row s1 + N s2).
// Only the first 2^(n+m) rows of a stage-m buffer exist (m slope bits per axis), so a stage
// computes exactly those.  L stages compose into 4^L (row, shift1, shift2) terms, exact for the
// same reason as the DRT's.
// grid: x = (output row i, block of kD1 consecutive d1); threads stride along d2.
constexpr int kD1 = 8;
template <class T, int L>
__global__ void djt_adj_stage(const T *__restrict__ in, T *__restrict__ out, int N, int n, int m_lo,
                              bool from_coef) {
    const int W = 2 * N;
    const int nb = (W + kD1 - 1) / kD1;
    const int i = blockIdx.x / nb, d1_0 = (blockIdx.x - i * nb) * kD1;
    constexpr int NT = 1 << (2 * L);
    int row[NT], e1[NT], e2[NT];
    row[0] = i;
    e1[0] = 0;
    e2[0] = 0;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const int m = m_lo + l, cnt = 1 << (2 * l);
#pragma unroll
        for (int t = cnt - 1; t >= 0; --t) {
            const int r = row[t], a1 = e1[t], a2 = e2[t];
            const int vm = r & 1, v = (r >> 1) & ((1 << (n - m - 1)) - 1);
            const int sg1 = (r >> (n - m)) & ((1 << m) - 1), sg2 = r >> n;
#pragma unroll
            for (int b1 = 0; b1 < 2; ++b1)
#pragma unroll
                for (int b2 = 0; b2 < 2; ++b2) {
                    const int k = 4 * t + 2 * b1 + b2;
                    row[k] = v + (b1 << (n - m - 1)) + (sg1 << (n - m)) + (b2 << n) + (sg2 << (n + 1));
                    e1[k] = a1 + vm * (b1 + sg1);
                    e2[k] = a2 + vm * (b2 + sg2);
                }
        }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t)
        if (from_coef) row[t] = (row[t] % N) * N + row[t] / N;   // packed s1 + N s2 -> caller row s1 N + s2
    for (int d2 = threadIdx.x; d2 < W; d2 += blockDim.x) {
        // per-term pointers to (row_t, d1_0 - e1_t, d2 - e2_t), walked down the d1 rows (kept in
        // registers; dereferenced only where both indices are >= 0)
        const T *pt[NT];
        bool ok2[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            pt[t] = in + (((long long)row[t] * W + (d1_0 - e1[t])) * W + (d2 - e2[t]));
            asm volatile("" : "+l"(pt[t]));
            ok2[t] = d2 >= e2[t];
        }
        T *dst = out + ((size_t)i * W + d1_0) * W + d2;
        for (int d1 = d1_0; d1 < d1_0 + kD1 && d1 < W; ++d1) {
            T acc = zero_v<T>();
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (ok2[t] && d1 >= e1[t]) acc = acc + __ldg(pt[t]);
                pt[t] += W;
            }
            *dst = acc;
            dst += W;
        }
    }
}

template <class T>
__global__ void djt_adj_scatter(const T *__restrict__ b0, T *__restrict__ cube, int N, int p0, int p1, int p2,
                                bool first) {
    const int c2 = blockIdx.y * blockDim.x + threadIdx.x;
    if (c2 >= N) return;
    const int c0 = blockIdx.x / N;
    const int c[3] = {c0, (int)blockIdx.x - c0 * N, c2};
    const int x = orient(c, p0, N), y = orient(c, p1, N), z = orient(c, p2, N);
    const int W = 2 * N;
    const T v = b0[((size_t)x * W + N + y) * W + N + z];
    const size_t idx = (size_t)blockIdx.x * N + c2;
    cube[idx] = first ? v : cube[idx] + v;
}

namespace {
// threads per block along the fast (D or z) axis: a multiple of 32, at most 256
inline unsigned tpb(int w) { return (unsigned)(w >= 256 ? 256 : ((w + 31) / 32) * 32); }
inline unsigned chunks(int w) { return (unsigned)((w + tpb(w) - 1) / tpb(w)); }
// threads per DRT stage row: about 8 cells per thread (per-thread term setup is ~130 instructions)
#ifndef D3_ADJ_EPT
#define D3_ADJ_EPT 8
#endif
inline unsigned row_threads(int w) {
    const int ept = D3_ADJ_EPT;
    const int t = ((w + ept - 1) / ept + 31) / 32 * 32;
    return (unsigned)(t < 32 ? 32 : (t > 1024 ? 1024 : t));
}

// stages fused per launch (default 1; -DD3_ADJ_L=2/3 for measurement builds: 2 and 3 were slower)
#ifndef D3_ADJ_L
#define D3_ADJ_L 1
#endif
int adj_fuse() { return D3_ADJ_L < 1 ? 1 : (D3_ADJ_L > 3 ? 3 : D3_ADJ_L); }

// butterfly launch: 4^L rows per block in one shared-memory buffer, NC columns per thread
template <class T, int L, int NC>
void drt_bfly_nc(const T *in, T *out, int N, int m_lo, cudaStream_t st) {
    const size_t smem = (size_t)(1 << (2 * L)) * 3 * N * sizeof(T);
    static std::atomic<uint32_t> smem_done{0};
    set_smem_once(drt_adj_bfly<T, L, NC>, 200 * 1024, smem_done);
    drt_adj_bfly<T, L, NC><<<(unsigned)((N >> L) * (N >> L)), 256, smem, st>>>(in, out, N, m_lo);
}

template <class T, int L>
void drt_bfly(const T *in, T *out, int N, int m_lo, cudaStream_t st) {
    const int nc = (3 * N + 255) / 256;
    if (nc <= 1) drt_bfly_nc<T, L, 1>(in, out, N, m_lo, st);
    else if (nc <= 3) drt_bfly_nc<T, L, 3>(in, out, N, m_lo, st);
    else if (nc <= 6) drt_bfly_nc<T, L, 6>(in, out, N, m_lo, st);
    else drt_bfly_nc<T, 1, 12>(in, out, N, m_lo, st);              // N = 1024: radix 2 only
}

// butterfly radix per launch: 2 (16 rows) up to N = 512, else 1 (-DD3_ADJ_BFLY=0 selects the
// plain gather kernels, for measurement builds)
#ifndef D3_ADJ_BFLY
#define D3_ADJ_BFLY 2
#endif
inline int bfly_max(int N) {
    const int cap = D3_ADJ_BFLY;
    return cap <= 0 ? 0 : (cap == 1 || N > 512 ? 1 : 2);
}

template <class T>
void drt_stage(int L, const T *in, T *out, int N, int m_lo, cudaStream_t st) {
    const dim3 g((unsigned)(N * N)), b(row_threads(3 * N));
    if (L == 1) drt_adj_stage<T, 1><<<g, b, 0, st>>>(in, out, N, m_lo);
    else if (L == 2) drt_adj_stage<T, 2><<<g, b, 0, st>>>(in, out, N, m_lo);
    else drt_adj_stage<T, 3><<<g, b, 0, st>>>(in, out, N, m_lo);
}

template <class T>
void djt_stage(int L, const T *in, T *out, int N, int n, int m_lo, bool from_coef, cudaStream_t st) {
    const long long rows = 1LL << (n + m_lo);                      // live rows of b^{m_lo}
    const dim3 g((unsigned)(rows * ((2 * N + kD1 - 1) / kD1))), b(tpb(2 * N));
    if (L == 1) djt_adj_stage<T, 1><<<g, b, 0, st>>>(in, out, N, n, m_lo, from_coef);
    else if (L == 2) djt_adj_stage<T, 2><<<g, b, 0, st>>>(in, out, N, n, m_lo, from_coef);
    else djt_adj_stage<T, 3><<<g, b, 0, st>>>(in, out, N, n, m_lo, from_coef);
}
}  // namespace

// ---- DRT backprojection by radix-2^K pass kernels (adjoint_pass.cuh): the forward's pass plan
// run backwards, levels n -> ... -> 0, then the seeding / orientation transpose.
namespace {
struct Level {
    int base, pitch;
};
// Level c storage: E = base + p.  For an intermediate level the base is chosen below lo_c so that
// the tile grid of the pass that READS it (its first tile at e = `ebase_reader`, staged from
// e - 2H) starts on a 4-element chunk: no tile is spent on a few misaligned columns.
inline Level level_layout(int N, int n, int c, int ebase_reader = 0, int h_reader = 0) {
    if (c == n) return {0, 3 * N};                                   // the caller's coefficients
    if (c == 0) return {2 * N, (N + 3) / 4 * 4};                     // z' = E - 2N
    const int lo = 2 * N - 2 * ((1 << c) - 1);
    int base = lo;
    base -= (((ebase_reader - 2 * h_reader - base) % 4) + 4) % 4;
    return {base, (3 * N - base + 15) / 16 * 16};
}
// lowest needed E of level c, and the first tile's e for the pass that writes level c with radix K
inline int level_lo(int N, int c) { return c == 0 ? 2 * N : 2 * N - 2 * ((1 << c) - 1); }
inline int pass_ebase(int N, int c, int K) { return level_lo(N, c) - 2 * ((1 << K) - 1) * ((1 << c) - 1); }
inline int pass_plan(int n, int (&ks)[4]) {                          // forward order, first pass first
    const int np = (n + 3) / 4;
    for (int i = 0; i < np; ++i) ks[i] = n / np + (i < n % np ? 1 : 0);
    return np;
}

#ifndef D3_ADJ_T
#define D3_ADJ_T 64        // swept 32 / 64 / 128: 2.52 / 2.02 / 2.19 ms (DRT N=256 x12)
#endif
constexpr int kAdjT = D3_ADJ_T, kAdjR = 8;

template <int K, class T>
void launch_adj_pass(const AdjPass &a, int ntiles, int groups, int D, cudaStream_t st) {
    using G = DrtGeom<K, kAdjR, kAdjT, false>;
    static std::atomic<uint32_t> smem_done{0};
    set_smem_once(drt_adj_pass_kernel<K, kAdjR, kAdjT, T>, G::SMEM, smem_done);
    drt_adj_pass_kernel<K, kAdjR, kAdjT, T><<<dim3((unsigned)ntiles, (unsigned)groups, (unsigned)D), G::THREADS, G::SMEM,
                                               st>>>(a);
}

// Pass-path workspace for a chunk of D dodecants: level-0 rows (D x N^2 x P0) and two
// intermediate regions (D x N^2 x the widest intermediate pitch); chunks are sized so the
// workspace stays within kAdjBudget (all 12 dodecants up to N = 256).
constexpr size_t kAdjBudget = 4ull << 30;
struct AdjWs {
    long long l0_stride, mid_stride;     // elements per dodecant
    int D;                               // dodecants per chunk
    size_t bytes;
};
inline AdjWs adj_ws(int N, int n, int K) {
    int ks[4];
    const int np = pass_plan(n, ks);
    int maxp = 0, c = 0;
    for (int i = 0; i < np - 1; ++i) {                               // intermediate levels c = ks[0], ks[0]+ks[1], ..
        c += ks[i];
        const Level l = level_layout(N, n, c, 0, 0);
        maxp = l.pitch + 16 > maxp ? l.pitch + 16 : maxp;            // + slack for the reader-aligned base
    }
    AdjWs w;
    w.l0_stride = (long long)N * N * ((N + 3) / 4 * 4);
    w.mid_stride = (long long)N * N * maxp;
    const size_t per = (size_t)(w.l0_stride + (np > 2 ? 2 : 1) * w.mid_stride) * 4;
    const size_t fit = kAdjBudget / (per ? per : 1);
    w.D = K < (int)(fit ? fit : 1) ? K : (int)(fit ? fit : 1);
    if (w.D > kGatherMax) w.D = kGatherMax;
    w.bytes = (per * (size_t)w.D + 255) / 256 * 256;
    return w;
}

// -DD3_ADJ_STAGES (measurement builds): the stage kernels for every N instead of the passes
bool adj_use_passes(int N) {
#ifdef D3_ADJ_STAGES
    return false && N >= 4;
#else
    return N >= 4;
#endif
}

// one instance: coefficients `src` (level n) -> level-0 rows in `l0`; returns launches
template <class T>
int drt_adj_passes(const T *src, int N, int n, int D, const AdjWs &w, T *tmp0, T *tmp1, T *l0, cudaStream_t st) {
    int ks[4];
    const int np = pass_plan(n, ks);
    int c_hi = n, nl = 0;
    const T *in = src;
    T *bufs[2] = {tmp0, tmp1};
    for (int i = np - 1; i >= 0; --i) {
        const int K = ks[i], c = c_hi - K;
        const int eb = pass_ebase(N, c, K), H = (1 << K) - 1;
        // this pass reads level c_hi (written by the previous pass with this pass's tile grid) and
        // writes level c (read by the next pass, radix ks[i - 1])
        const Level li = level_layout(N, n, c_hi, eb, H);
        const Level lo = c > 0 ? level_layout(N, n, c, pass_ebase(N, c - ks[i - 1], ks[i - 1]), (1 << ks[i - 1]) - 1)
                               : level_layout(N, n, 0);
        T *out = c == 0 ? l0 : bufs[i & 1];
        AdjPass a{};
        a.in = in;
        a.out = out;
        a.N = N;
        a.n = n;
        a.c = c;
        a.m = n - c - K;
        a.in_pitch = li.pitch;
        a.in_base = li.base;
        a.in_width = li.pitch;
        a.in_inst_stride = c_hi == n ? (long long)N * N * 3 * N : w.mid_stride;
        a.out_inst_stride = c == 0 ? w.l0_stride : w.mid_stride;
        a.out_pitch = lo.pitch;
        a.out_base = lo.base;
        a.out_width = lo.pitch;
        a.lo = level_lo(N, c);
        a.ebase = eb;
        if ((((eb - 2 * H - li.base) % 4) + 4) % 4 != 0) a.ebase -= (((eb - 2 * H - li.base) % 4) + 4) % 4;   // coefficients: base 0
        a.one = 1u;
        const int ntiles = (3 * N - a.ebase + kAdjT - 1) / kAdjT;
        const int groups = 1 << (2 * (n - K));
        switch (K) {
            case 1: launch_adj_pass<1, T>(a, ntiles, groups, D, st); break;
            case 2: launch_adj_pass<2, T>(a, ntiles, groups, D, st); break;
            case 3: launch_adj_pass<3, T>(a, ntiles, groups, D, st); break;
            default: launch_adj_pass<4, T>(a, ntiles, groups, D, st); break;
        }
        ++nl;
        in = out;
        c_hi = c;
    }
    return nl;
}
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
    const int Lb = transform == 0 ? bfly_max(N) : 0;
    const int Lmax = Lb > 0 ? Lb : adj_fuse();
    const dim3 sg((unsigned)(N * N), chunks(N)), sb(tpb(N));
    int nl = 0;
    if (transform == 0 && adj_use_passes(N)) {
        // pass kernels over chunks of D dodecants, then one gather into the cube per chunk
        const AdjWs w = adj_ws(N, n, K);
        int ks[4];
        const int np = pass_plan(n, ks);
        T *l0 = reinterpret_cast<T *>(ws);
        T *mid0 = l0 + (long long)w.D * w.l0_stride;
        T *mid1 = np > 2 ? mid0 + (long long)w.D * w.mid_stride : mid0;
        int kl[12], nk = 0;
        for (int k = 0; k < 12; ++k)
            if ((mask >> k) & 1) kl[nk++] = k;
        const int P0 = (N + 3) / 4 * 4;
        for (int b = 0; b < batch; ++b) {
            T *cube_b = cb + (long long)b * n3;
            for (int j0 = 0; j0 < K; j0 += w.D) {
                const int d = K - j0 < w.D ? K - j0 : w.D;
                nl += drt_adj_passes<T>(cf + ((long long)b * K + j0) * cells, N, n, d, w, mid0, mid1, l0, st);
                if (N >= 32) {
                    GatherArgs g{};
                    g.D = d;
                    for (int jj = 0; jj < d; ++jj)
                        for (int t = 0; t < 3; ++t) g.rows[jj][t] = rows[kl[j0 + jj]][t];
                    drt_adj_gather<T><<<dim3((unsigned)(N / 32), (unsigned)(N / 8), (unsigned)(N / 8)), 256, 0, st>>>(
                        l0, w.l0_stride, P0, N, g, cube_b, j0 == 0);
                    ++nl;
                } else {
                    for (int jj = 0; jj < d; ++jj) {
                        drt_scatter<T>(l0 + (long long)jj * w.l0_stride, cube_b, N, rows[kl[j0 + jj]], j0 + jj == 0, P0, 0,
                                       st);
                        ++nl;
                    }
                }
            }
        }
        if (launches) *launches = nl;
        return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
    }
    for (int b = 0; b < batch; ++b) {
        int j = 0;
        for (int k = 0; k < 12; ++k) {
            if (!((mask >> k) & 1)) continue;
            const T *src = cf + ((long long)b * K + j) * cells;
            int cur = 0;
            for (int m_hi = n - 1; m_hi >= 0;) {
                const int L = m_hi + 1 < Lmax ? m_hi + 1 : Lmax, m_lo = m_hi - L + 1;
                const T *in = (m_hi == n - 1) ? src : buf[cur ^ 1];
                if (transform == 0 && Lb > 0) {
                    if (L == 2) drt_bfly<T, 2>(in, buf[cur], N, m_lo, st);
                    else drt_bfly<T, 1>(in, buf[cur], N, m_lo, st);
                } else if (transform == 0) drt_stage<T>(L, in, buf[cur], N, m_lo, st);
                else djt_stage<T>(L, in, buf[cur], N, n, m_lo, m_hi == n - 1, st);
                ++nl;
                cur ^= 1;
                m_hi = m_lo - 1;
            }
            const T *b0 = buf[cur ^ 1];
            if (transform == 0)
                drt_adj_scatter<T><<<sg, sb, 0, st>>>(b0, cb + (long long)b * n3, N, rows[k][0], rows[k][1],
                                                      rows[k][2], j == 0, 3 * N, 2 * N);
            else
                djt_adj_scatter<T><<<sg, sb, 0, st>>>(b0, cb + (long long)b * n3, N, rows[k][0], rows[k][1],
                                                      rows[k][2], j == 0);
            ++nl;
            ++j;
        }
    }
    if (launches) *launches = nl;
    return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
}

size_t adjoint_workspace_bytes(int transform, int N, uint32_t mask) {
    const long long W = transform == 0 ? 3LL * N : 2LL * N;
    const long long cells = transform == 0 ? (long long)N * N * W : (long long)N * N * W * W;
    size_t b = (size_t)(2 * cells * 4 + 255) / 256 * 256;            // the stage kernels' two buffers
    if (transform == 0 && N >= 4) {                                  // the pass path (default)
        int n = 0;
        while ((1 << n) < N) ++n;
        const size_t pb = adj_ws(N, n, __builtin_popcount(mask & 0xFFFu)).bytes;
        b = pb > b ? pb : b;
    }
    return b;
}

drt3d_status run_adjoint(int transform, const void *coef, int N, int n, const int8_t (*rows)[3], uint32_t mask,
                         int batch, int dtype, void *cube, void *ws, cudaStream_t st, int *launches) {
    if (dtype == DRT3D_F32) return run_adj<float>(transform, coef, N, n, rows, mask, batch, cube, ws, st, launches);
    return run_adj<uint32_t>(transform, coef, N, n, rows, mask, batch, cube, ws, st, launches);
}

}  // namespace d3
