// invert.cu -- iterative inverse of the 3D DRT of planes.
//
// the adjoint is used "as an approximate inverse operator of the DRT in the
// theory of iterative improvement of a solution to linear equations" (Press, Numerical Recipes
// §2.5), x <- x + B (b - A x), with the 3D high-pass filter h of PAPER.md:576-591 and the
// prolongation P / restriction S multigrid of PAPER.md:592-601.  Readings (R15-R18):
// the filtered-backprojection step is alpha h*(A^T r) with alpha = <r, A p> / <A p, A p>,
// p = h*(A^T r) (residual-minimising); h with zero padding; B (mg_apply) = restrict the residual,
// recurse to N/2, prolongate, then one filtered-backprojection step on what remains; the
// coarsest size n_min takes the step alone (n_min = N: single-grid iteration).
//
// Iteration 1 is enqueued directly; the others replay one captured iteration (a CUDA graph, cached
// per buffers and shapes; ~100 launches per iteration at N = 64 become one).
// Every iteration is enqueued on the caller's stream with no host synchronisation: A^T is the
// library's backprojection, A its forward transform (fp32 in / fp32 out), and alpha is computed
// on the device by a fixed-order two-pass fp64 reduction (deterministic) and read by the update
// kernels from device memory.
#include "drt3d.h"

#include <cstdint>
#include <mutex>

#include <cuda_runtime.h>

namespace d3 {
// api.cu: r <- r - A f (fp32, stacked) with the residual folded into the forward's final pass
drt3d_status planes_residual(const void *cube, int N, uint32_t mask, float *r, const drt3d_opts *opts,
                             void *workspace, size_t workspace_bytes, void *stream);
// api.cu: out = A f (fp32, stacked) with per-CTA sums of out^2 fused into the final pass
size_t planes_sumsq_parts(int N, int instances);
drt3d_status planes_sumsq(const void *cube, int N, uint32_t mask, float *out, const drt3d_opts *opts,
                          void *workspace, size_t workspace_bytes, void *stream, double *sq_part, int *sq_count);
namespace inv {

constexpr int kRedBlocks = 1184;     // 8 x 148 SMs, fixed so the reduction order is fixed
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;                                   // valid in thread 0
}

// part[2 blk] = sum r*q, part[2 blk + 1] = sum q*q over this block's grid-stride share.
// Element counts of the coefficient and cube arrays are multiples of 4 (N >= 2) and every
// buffer is 256-byte aligned: the streaming kernels use 16-byte accesses.
__global__ void __launch_bounds__(kRedThreads) dot_rq_qq(const float *__restrict__ r, const float *__restrict__ q,
                                                          size_t n, double *__restrict__ part) {
    __shared__ double sh[2][kRedThreads / 32];
    double rq = 0.0, qq = 0.0;
    const float4 *r4 = reinterpret_cast<const float4 *>(r), *q4 = reinterpret_cast<const float4 *>(q);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 a = r4[i], b = q4[i];
        rq += (double)a.x * b.x + (double)a.y * b.y + (double)a.z * b.z + (double)a.w * b.w;
        qq += (double)b.x * b.x + (double)b.y * b.y + (double)b.z * b.z + (double)b.w * b.w;
    }
    const double s0 = block_sum(rq, sh[0]);
    const double s1 = block_sum(qq, sh[1]);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = s0;
        part[2 * blockIdx.x + 1] = s1;
    }
}

__global__ void finalize_alpha(const double *__restrict__ part, int nb, double *__restrict__ alpha) {
    __shared__ double sh[2][kRedThreads / 32];
    double rq = 0.0, qq = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        rq += part[2 * i];
        qq += part[2 * i + 1];
    }
    const double s0 = block_sum(rq, sh[0]);
    const double s1 = block_sum(qq, sh[1]);
    if (threadIdx.x == 0) *alpha = s1 > 0.0 ? s0 / s1 : 0.0;
}

// alpha = <g, p> / <q, q>: <g, p> = sum part[2i] (dot_rq_qq(g, p) partials; <r, A p> = <A^T r, p>
// with g = A^T r), <q, q> = sum qq[0 .. *count) (the forward's per-CTA sums), both in a fixed order
__global__ void finalize_alpha_gp(const double *__restrict__ part, int nb, const double *__restrict__ qq,
                                  const int *__restrict__ count, double *__restrict__ alpha) {
    __shared__ double sh[2][kRedThreads / 32];
    double gp = 0.0, q2 = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) gp += part[2 * i];
    const int n = *count;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q2 += qq[i];
    const double s0 = block_sum(gp, sh[0]);
    const double s1 = block_sum(q2, sh[1]);
    if (threadIdx.x == 0) *alpha = s1 > 0.0 ? s0 / s1 : 0.0;
}

// dst <- src - alpha q (fp32; dst may be src), part[blk] = sum dst^2
__global__ void __launch_bounds__(kRedThreads) update_r(const float *src, const float *__restrict__ q, float *dst,
                                                         size_t n, const double *__restrict__ alpha,
                                                         double *__restrict__ part) {
    __shared__ double sh[kRedThreads / 32];
    const float a = (float)*alpha;
    double rr = 0.0;
    const float4 *s4 = reinterpret_cast<const float4 *>(src), *q4 = reinterpret_cast<const float4 *>(q);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 u = s4[i], w = q4[i];
        const float4 v = make_float4(u.x - a * w.x, u.y - a * w.y, u.z - a * w.z, u.w - a * w.w);
        d4[i] = v;
        rr += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
    const double s = block_sum(rr, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// part[blk] = sum r^2 (initial residual norm)
__global__ void __launch_bounds__(kRedThreads) sum_sq(const float *__restrict__ r, size_t n, double *__restrict__ part) {
    __shared__ double sh[kRedThreads / 32];
    double rr = 0.0;
    const float4 *r4 = reinterpret_cast<const float4 *>(r);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = r4[i];
        rr += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
    const double s = block_sum(rr, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// out[*ctr] = sqrt(sum part), then ++*ctr: the residual-norm slot of an iteration comes from
// device memory, so one captured iteration (a CUDA graph) serves every iteration
__global__ void finalize_norm_ctr(const double *__restrict__ part, int nb, double *__restrict__ out, int *ctr) {
    __shared__ double sh[kRedThreads / 32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0) {
        if (out) out[*ctr] = sqrt(t);
        *ctr += 1;
    }
}

__global__ void set_int(int *p, int v) { *p = v; }

__global__ void finalize_norm(const double *__restrict__ part, int nb, double *__restrict__ out) {
    __shared__ double sh[kRedThreads / 32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
    const double t = block_sum(s, sh);
    if (threadIdx.x == 0 && out) *out = sqrt(t);
}

// x <- x + alpha p
__global__ void update_x(float *__restrict__ x, const float *__restrict__ p, size_t n,
                         const double *__restrict__ alpha) {
    const float a = (float)*alpha;
    float4 *x4 = reinterpret_cast<float4 *>(x);
    const float4 *p4 = reinterpret_cast<const float4 *>(p);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 u = x4[i], v = p4[i];
        x4[i] = make_float4(u.x + a * v.x, u.y + a * v.y, u.z + a * v.z, u.w + a * v.w);
    }
}

// p = h * g, h of PAPER.md:576-591 (centre 7/8, faces -1/16, edges -1/32, corners -1/64), zero
// outside the cube.  grid.x = x * N + y, threads along z.
__global__ void highpass(const float *__restrict__ g, float *__restrict__ p, int N) {
    const int x = blockIdx.x / N, y = blockIdx.x - x * N;
    const float w[4] = {7.f / 8.f, -1.f / 16.f, -1.f / 32.f, -1.f / 64.f};
    for (int z = threadIdx.x; z < N; z += blockDim.x) {
        float acc = 0.f;
#pragma unroll
        for (int a = -1; a <= 1; ++a) {
            if (x + a < 0 || x + a >= N) continue;
#pragma unroll
            for (int b = -1; b <= 1; ++b) {
                if (y + b < 0 || y + b >= N) continue;
                const float *row = g + ((size_t)(x + a) * N + (y + b)) * N;
#pragma unroll
                for (int c = -1; c <= 1; ++c) {
                    if (z + c < 0 || z + c >= N) continue;
                    acc += w[(a != 0) + (b != 0) + (c != 0)] * __ldg(row + z + c);
                }
            }
        }
        p[((size_t)x * N + y) * N + z] = acc;
    }
}

// S: rc[k][s1][s2][d] = (r[k][2 s1][2 s2][2 d] + r[k][2 s1][2 s2][2 d + 1]) / 8,
// coarse size nc (fine 2 nc).  grid.x = k * nc * nc + s1 * nc + s2, threads along d.
__global__ void restrict_coef(const float *__restrict__ r, float *__restrict__ rc, int nc) {
    const int Wc = 3 * nc, W = 6 * nc, n = 2 * nc;
    const int row = blockIdx.x, k = row / (nc * nc), s1 = (row / nc) % nc, s2 = row % nc;
    const float *src = r + (((size_t)k * n + 2 * s1) * n + 2 * s2) * W;
    float *dst = rc + (size_t)row * Wc;
    for (int d = threadIdx.x; d < Wc; d += blockDim.x) dst[d] = 0.125f * (src[2 * d] + src[2 * d + 1]);
}

// P: e[x][y][z] = ec[x/2][y/2][z/2].  grid.x = x * n + y, threads along z.
__global__ void prolong_cube(const float *__restrict__ ec, float *__restrict__ e, int n) {
    const int x = blockIdx.x / n, y = blockIdx.x % n, nc = n / 2;
    const float *src = ec + ((size_t)(x / 2) * nc + y / 2) * nc;
    float *dst = e + (size_t)blockIdx.x * n;
    for (int z = threadIdx.x; z < n; z += blockDim.x) dst[z] = src[z / 2];
}

// out = a - b
__global__ void diff(const float *__restrict__ a, const float *__restrict__ b, float *__restrict__ out, size_t n) {
    const float4 *a4 = reinterpret_cast<const float4 *>(a), *b4 = reinterpret_cast<const float4 *>(b);
    float4 *o4 = reinterpret_cast<float4 *>(out);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 u = a4[i], v = b4[i];
        o4[i] = make_float4(u.x - v.x, u.y - v.y, u.z - v.z, u.w - v.w);
    }
}

inline size_t align256(size_t b) { return (b + 255) / 256 * 256; }

constexpr int kMaxLevels = 11;

// Per grid level (0 = the caller's size N, level l has size N >> l): residual r (its remainder
// r - A e replaces it in place), and A e / A p sharing one buffer (coefficient-sized); e, A^T r, p
// (cube-sized).  Level 0's r is the outer residual.
struct Level {
    int n;
    size_t ncoef, ncube;
    size_t r, ae, q, e, g, p;
};

struct Layout {
    int nlev;
    Level lv[kMaxLevels];
    size_t part, scal, tws, total, tws_bytes, qq, qq_cap;
};

inline drt3d_opts f32_opts(int table) {
    drt3d_opts o = {};
    o.batch = 1;
    o.in_dtype = DRT3D_F32;
    o.out_dtype = DRT3D_F32;
    o.layout = DRT3D_LAYOUT_STACKED;
    o.table = table;
    return o;
}

inline drt3d_status layout(int N, int n_min, uint32_t mask, int table, Layout &L) {
    const int K = __builtin_popcount(mask & 0xFFFu);
    drt3d_opts o = f32_opts(table);
    size_t fw = 0, aw = 0;
    drt3d_status s = drt3d_planes_workspace_size(N, mask, &o, &fw);       // the largest level's
    if (s != DRT3D_OK) return s;
    s = drt3d_planes_adjoint_workspace_size(N, mask, &o, &aw);
    if (s != DRT3D_OK) return s;
    L.tws_bytes = align256(fw > aw ? fw : aw);          // forward and adjoint run one after the other
    size_t off = 0;
    L.nlev = 0;
    for (int n = N; n >= n_min && L.nlev < kMaxLevels; n >>= 1) {
        Level &v = L.lv[L.nlev++];
        v.n = n;
        v.ncoef = (size_t)K * n * n * 3 * n;
        v.ncube = (size_t)n * n * n;
        v.r = off; off += align256(v.ncoef * 4);
        v.q = off; off += align256(v.ncoef * 4);
        v.ae = v.q;                                     // A e is dead once r' = r - A e is formed
        v.e = off; off += align256(v.ncube * 4);
        v.g = off; off += align256(v.ncube * 4);
        v.p = off; off += align256(v.ncube * 4);
    }
    L.part = off; off += align256(2 * kRedBlocks * sizeof(double));
    L.qq_cap = planes_sumsq_parts(N, K);                // per-CTA sums of (A p)^2 of the largest level
    L.qq = off; off += align256(L.qq_cap * sizeof(double) + 256);
    L.scal = off; off += 256;                           // [0] = 1.0, [1 + l] = alpha of level l, int at +128
    static_assert(8 * (1 + kMaxLevels) <= 128, "scalar slots");
    L.tws = off; off += L.tws_bytes;
    L.total = off;
    return DRT3D_OK;
}

}  // namespace inv
}  // namespace d3

using namespace d3::inv;

static drt3d_status invert_check(int N, int n_min, uint32_t mask, const drt3d_opts *opts, int &table) {
    if (N < 2 || N > 1024 || (N & (N - 1)) || mask == 0 || mask >= (1u << 12)) return DRT3D_ERR_INVALID_ARG;
    if (n_min < 2 || n_min > N || (n_min & (n_min - 1))) return DRT3D_ERR_INVALID_ARG;
    table = DRT3D_TABLE_HEMISPHERE;
    if (opts) {
        if (opts->batch != 1 || opts->out_dtype != DRT3D_F32 || opts->layout != DRT3D_LAYOUT_STACKED)
            return DRT3D_ERR_INVALID_ARG;
        if (opts->table < 0 || opts->table > 2) return DRT3D_ERR_INVALID_ARG;
        table = opts->table;
    }
    return DRT3D_OK;
}

extern "C" drt3d_status drt3d_planes_invert_workspace_size(int N, int n_min, uint32_t mask, const drt3d_opts *opts,
                                                           size_t *bytes) {
    int table;
    if (!bytes) return DRT3D_ERR_INVALID_ARG;
    drt3d_status s = invert_check(N, n_min, mask, opts, table);
    if (s != DRT3D_OK) return s;
    Layout L;
    s = layout(N, n_min, mask, table, L);
    if (s != DRT3D_OK) return s;
    *bytes = L.total;
    return DRT3D_OK;
}

namespace {

struct Ctx {
    const Layout *L;
    unsigned char *w;
    uint32_t mask;
    cudaStream_t st;
    void *stream;
    drt3d_opts o;
    int nl;
    double *rnorm;
    float *f(size_t off) const { return reinterpret_cast<float *>(w + off); }
    double *part() const { return reinterpret_cast<double *>(w + L->part); }
    double *qq() const { return reinterpret_cast<double *>(w + L->qq); }
    int *qq_count() const { return reinterpret_cast<int *>(w + L->qq + L->qq_cap * sizeof(double)); }
    double *one() const { return reinterpret_cast<double *>(w + L->scal); }
    double *alpha(int l) const { return reinterpret_cast<double *>(w + L->scal) + 1 + l; }
    int *ctr() const { return reinterpret_cast<int *>(w + L->scal + 128); }
    void *tws() const { return w + L->tws; }
};

inline unsigned row_threads(int len) { return len >= 128 ? 128u : (unsigned)((len + 31) / 32 * 32); }

// R16 step on residual `res` at level l: p = h*(A^T res), q = A p, alpha_l = <res,q>/<q,q>.
drt3d_status step(Ctx &c, int l, const float *res) {
    const Level &v = c.L->lv[l];
    int l1 = 0, l2 = 0;
    c.o.launches = &l1;
    drt3d_status s = drt3d_planes_adjoint(res, v.n, c.mask, c.f(v.g), &c.o, c.tws(), c.L->tws_bytes, c.stream);
    if (s != DRT3D_OK) return s;
    highpass<<<(unsigned)(v.n * v.n), row_threads(v.n), 0, c.st>>>(c.f(v.g), c.f(v.p), v.n);
    c.o.launches = &l2;
    // q = A p with <q, q> summed in the forward's final pass, <res, q> = <A^T res, p> = <g, p> over the
    // cube: no pass over the coefficients (N >= 64); smaller levels take the coefficient-sized dot
    s = d3::planes_sumsq(c.f(v.p), v.n, c.mask, c.f(v.q), &c.o, c.tws(), c.L->tws_bytes, c.stream, c.qq(), c.qq_count());
    if (s == DRT3D_OK) {
        dot_rq_qq<<<kRedBlocks, kRedThreads, 0, c.st>>>(c.f(v.g), c.f(v.p), v.ncube, c.part());
        finalize_alpha_gp<<<1, kRedThreads, 0, c.st>>>(c.part(), kRedBlocks, c.qq(), c.qq_count(), c.alpha(l));
        c.nl += l1 + l2 + 3;
        return DRT3D_OK;
    }
    if (s != DRT3D_ERR_UNSUPPORTED) return s;
    l2 = 0;
    s = drt3d_planes(c.f(v.p), v.n, c.mask, c.f(v.q), &c.o, c.tws(), c.L->tws_bytes, c.stream);
    if (s != DRT3D_OK) return s;
    dot_rq_qq<<<kRedBlocks, kRedThreads, 0, c.st>>>(res, c.f(v.q), v.ncoef, c.part());
    finalize_alpha<<<1, kRedThreads, 0, c.st>>>(c.part(), kRedBlocks, c.alpha(l));
    c.nl += l1 + l2 + 3;
    return DRT3D_OK;
}

// Multigrid approximate inverse (R18) of the residual in level l's `r` buffer: leaves e_l = B r_l
// in `e`.  A parent uses only its child's e (it applies A to the prolongated e itself), so A e_l
// is never formed below the top; at the top (l = 0) the outer residual is updated in place,
// r <- r' - alpha q with r' = r - A P e_c the remainder the last step minimised (r' = r on a
// single grid), which equals r - A e_0.
drt3d_status mg_apply(Ctx &c, int l) {
    const Level &v = c.L->lv[l];
    const unsigned nb = kRedBlocks;
    const float *rem = c.f(v.r);                                                // what the step sees
    if (l < c.L->nlev - 1) {
        const Level &u = c.L->lv[l + 1];
        const int K = (int)(v.ncoef / ((size_t)v.n * v.n * 3 * v.n));
        restrict_coef<<<(unsigned)(K * u.n * u.n), row_threads(3 * u.n), 0, c.st>>>(c.f(v.r), c.f(u.r), u.n);  // S r
        c.nl += 1;
        drt3d_status s = mg_apply(c, l + 1);                                                                  // B_{n/2}
        if (s != DRT3D_OK) return s;
        prolong_cube<<<(unsigned)(v.n * v.n), row_threads(v.n), 0, c.st>>>(c.f(u.e), c.f(v.e), v.n);        // e = P e_c
        int l1 = 0;
        c.o.launches = &l1;
        // r' = r - A e, in place in r (r is not used again at this level): the forward's final pass
        // adds -A e into r; small levels take A e and an elementwise difference
        s = d3::planes_residual(c.f(v.e), v.n, c.mask, c.f(v.r), &c.o, c.tws(), c.L->tws_bytes, c.stream);
        if (s == DRT3D_OK) {
            c.nl += l1 + 1;
            rem = c.f(v.r);
        } else if (s == DRT3D_ERR_UNSUPPORTED) {
            l1 = 0;
            s = drt3d_planes(c.f(v.e), v.n, c.mask, c.f(v.ae), &c.o, c.tws(), c.L->tws_bytes, c.stream);   // A e
            if (s != DRT3D_OK) return s;
            diff<<<nb, kRedThreads, 0, c.st>>>(c.f(v.r), c.f(v.ae), c.f(v.r), v.ncoef);                     // r' = r - A e
            c.nl += l1 + 2;
            rem = c.f(v.r);
        } else {
            return s;
        }
    } else {
        if (cudaMemsetAsync(c.f(v.e), 0, v.ncube * 4, c.st) != cudaSuccess) return DRT3D_ERR_CUDA;
    }
    drt3d_status s = step(c, l, rem);                                                      // alpha, p, q = A p
    if (s != DRT3D_OK) return s;
    update_x<<<nb, kRedThreads, 0, c.st>>>(c.f(v.e), c.f(v.p), v.ncube, c.alpha(l));                         // e += a p
    c.nl += 1;
    if (l == 0) {
        update_r<<<nb, kRedThreads, 0, c.st>>>(rem, c.f(v.q), c.f(v.r), v.ncoef, c.alpha(l), c.part());      // r = r' - a q
        c.nl += 1;
    }
    return DRT3D_OK;
}

// one outer iteration: e = B r, r <- r - A e (in mg_apply), x += e, ||r|| into rnorm[ctr++]
drt3d_status iteration(Ctx &c, float *x) {
    const Level &top = c.L->lv[0];
    drt3d_status s = mg_apply(c, 0);
    if (s != DRT3D_OK) return s;
    update_x<<<kRedBlocks, kRedThreads, 0, c.st>>>(x, c.f(top.e), top.ncube, c.one());
    finalize_norm_ctr<<<1, kRedThreads, 0, c.st>>>(c.part(), kRedBlocks, c.rnorm, c.ctr());
    c.nl += 2;
    return DRT3D_OK;
}

// Instantiated one-iteration graphs, keyed by everything they bake in.  Kept for the life of the
// process (a graph may still be executing when the call returns, so none is destroyed); at most
// kGraphCache entries, beyond which calls fall back to eager enqueue.
struct GraphKey {
    int dev, N, n_min, mask, table;
    const void *x, *rnorm, *ws;
    bool operator==(const GraphKey &o) const {
        return dev == o.dev && N == o.N && n_min == o.n_min && mask == o.mask && table == o.table && x == o.x &&
               rnorm == o.rnorm && ws == o.ws;
    }
};
constexpr int kGraphCache = 16;

cudaGraphExec_t graph_for(GraphKey key, Ctx &c, float *x) {
    static std::mutex mu;
    static GraphKey keys[kGraphCache];
    static cudaGraphExec_t execs[kGraphCache];
    static int count = 0;
    static cudaStream_t capture_stream[32] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    key.dev = dev;
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < count; ++i)
        if (keys[i] == key) return execs[i];
    if (count == kGraphCache || dev >= 32) return nullptr;
    // capture on an internal stream (capture is illegal on the legacy default stream, which the
    // caller may use); nothing executes during capture
    if (!capture_stream[dev] && cudaStreamCreateWithFlags(&capture_stream[dev], cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    Ctx cc = c;
    cc.st = capture_stream[dev];
    cc.stream = capture_stream[dev];
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    if (cudaStreamBeginCapture(cc.st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    const drt3d_status s = iteration(cc, x);
    const cudaError_t e = cudaStreamEndCapture(cc.st, &graph);
    if (s != DRT3D_OK || e != cudaSuccess || !graph || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return nullptr;
    }
    cudaGraphDestroy(graph);                                  // the executable keeps its own copy
    keys[count] = key;
    execs[count] = exec;
    ++count;
    return exec;
}

}  // namespace

extern "C" drt3d_status drt3d_planes_invert(const void *coef, int N, int n_min, uint32_t mask, int iters, void *cube,
                                            double *rnorm, const drt3d_opts *opts, void *ws, size_t ws_bytes,
                                            void *stream) {
    int table;
    drt3d_status s = invert_check(N, n_min, mask, opts, table);
    if (s != DRT3D_OK) return s;
    if (!coef || !cube || iters < 0) return DRT3D_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(coef) | reinterpret_cast<uintptr_t>(cube)) & 15) return DRT3D_ERR_INVALID_ARG;
    Layout L;
    s = layout(N, n_min, mask, table, L);
    if (s != DRT3D_OK) return s;
    if (!ws || ws_bytes < L.total || (reinterpret_cast<uintptr_t>(ws) & 255)) return DRT3D_ERR_WORKSPACE;
    Ctx c{&L, reinterpret_cast<unsigned char *>(ws), mask, reinterpret_cast<cudaStream_t>(stream), stream,
          f32_opts(table), 0, nullptr};
    const Level &top = L.lv[0];
    float *x = reinterpret_cast<float *>(cube), *r = c.f(top.r);
    static const double kOne = 1.0;
    if (cudaMemcpyAsync(c.one(), &kOne, sizeof(double), cudaMemcpyHostToDevice, c.st) != cudaSuccess)
        return DRT3D_ERR_CUDA;
    // x0 = 0, r0 = b
    if (cudaMemsetAsync(x, 0, top.ncube * 4, c.st) != cudaSuccess) return DRT3D_ERR_CUDA;
    if (cudaMemcpyAsync(r, coef, top.ncoef * 4, cudaMemcpyDeviceToDevice, c.st) != cudaSuccess) return DRT3D_ERR_CUDA;
    c.rnorm = rnorm;
    if (rnorm) {
        sum_sq<<<kRedBlocks, kRedThreads, 0, c.st>>>(r, top.ncoef, c.part());
        finalize_norm<<<1, kRedThreads, 0, c.st>>>(c.part(), kRedBlocks, rnorm);
        c.nl += 2;
    }
    set_int<<<1, 1, 0, c.st>>>(c.ctr(), 1);
    c.nl += 1;
    if (iters == 0) {
        if (opts && opts->launches) *opts->launches = c.nl;
        return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
    }
    // iteration 1 eagerly (it also sets every kernel attribute), the others by replaying one
    // captured iteration
    s = iteration(c, x);
    if (s != DRT3D_OK) return s;
    if (iters > 1) {
        const GraphKey key{0, N, n_min, (int)mask, table, x, rnorm, ws};
        cudaGraphExec_t exec = graph_for(key, c, x);
        for (int k = 1; k < iters; ++k) {
            if (exec) {
                if (cudaGraphLaunch(exec, c.st) != cudaSuccess) return DRT3D_ERR_CUDA;
                c.nl += 1;
            } else {
                s = iteration(c, x);
                if (s != DRT3D_OK) return s;
            }
        }
    }
    if (opts && opts->launches) *opts->launches = c.nl;
    return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
}
