/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for arXiv 2501.13664
 * ("Multiscale 3D DRT of planes and DJT of lines", Marichal-Hernandez et al.).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or helper with the CUDA path in
 * paper_2501_13664_b200/csrc, and neither includes the other.
 *
 * Every routine is a direct transcription of a passage of /root/reference/PAPER.md
 * (cited as PAPER.md:line + equation label / algorithm), single-threaded, with
 * int64 accumulation for integer data and fp64 for floating point.  No blocking,
 * fusion or reordering beyond what the cited definition or algorithm states.
 *
 * Index conventions:
 *   cube g[x][y][z], C order, z fastest, N = 2^n.
 *   DRT dodecant out[s1][s2][D], D in [0,3N): z = l_{s1}(x) + l_{s2}(y) + D - 2N
 *       (Alg. 1 literal; seeding at 2N..3N-1).
 *   DJT dodecant out[s1][s2][D1][D2], Di in [0,2N): y = l_{s1}(u)+D1-N,
 *       z = l_{s2}(u)+D2-N (Alg. 3 literal).
 *
 * Pins (tests/test_oracle_*.py): closed form == recursion for the line,
 * brute force == recursion for both transforms, separable sum == recursion,
 * adjoint identity, CG round trip, mass conservation, hand-derived goldens.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static int ilog2_exact(int64_t N) {
    int n = 0;
    while (((int64_t)1 << n) < N) n++;
    return (((int64_t)1 << n) == N) ? n : -1;
}

/* ------------------------------------------------------------------ L0 --
 * eq:digitalLine, recursive form (normative):
 *   l^n_s(u_0..u_{n-1}) = l^{n-1}_{floor(s/2)}(u_0..u_{n-2}) + u_{n-1} * floor((s+1)/2),
 * with u = lambda(u_0..u_{n-1}) = sum u_i 2^i and l^0 = 0.
 */
int64_t oracle_line(int n, int64_t s, int64_t u) {
    if (n == 0) return 0;
    int64_t u_top = (u >> (n - 1)) & 1;              /* u_{n-1}            */
    int64_t u_rest = u & (((int64_t)1 << (n - 1)) - 1); /* (u_0..u_{n-2})  */
    return oracle_line(n - 1, s / 2, u_rest) + u_top * ((s + 1) / 2);
}

/* Closed form of eq:digitalLine:
 *   sum_{i=0}^{n-1} u_{n-1-i} * floor((s/2^i + 1)/2).
 * real_division != 0 reads s/2^i as a real quotient, else as integer division
 * (the two readings SPEC.md:61 asks about). */
int64_t oracle_line_closed(int n, int64_t s, int64_t u, int real_division) {
    int64_t acc = 0;
    for (int i = 0; i < n; i++) {
        int64_t bit = (u >> (n - 1 - i)) & 1;
        int64_t c;
        if (real_division) c = (int64_t)floor(((double)s / (double)((int64_t)1 << i) + 1.0) / 2.0);
        else c = ((s >> i) + 1) / 2;
        acc += bit * c;
    }
    return acc;
}

/* table L[s*N + u] = l^n_s(u) for s,u in [0,N) */
static int64_t *line_table(int n) {
    int64_t N = (int64_t)1 << n;
    int64_t *L = (int64_t *)malloc(sizeof(int64_t) * N * N);
    for (int64_t s = 0; s < N; s++)
        for (int64_t u = 0; u < N; u++) L[s * N + u] = oracle_line(n, s, u);
    return L;
}

/* ----------------------------------------------------------- L2 planes --
 * eq:3DfDRT, brute force:
 *   out(s1,s2,D) = sum_{x,y} g(x, y, l_{s1}(x) + l_{s2}(y) + D - 2N),
 * only terms with 0 <= z < N.  O(N^5).  Output N*N*3N (fp64). */
int oracle_drt_brute_f64(const double *g, int64_t N, double *out) {
    int n = ilog2_exact(N);
    if (n < 0) return -1;
    int64_t *L = line_table(n);
    int64_t W = 3 * N;
    for (int64_t s1 = 0; s1 < N; s1++)
        for (int64_t s2 = 0; s2 < N; s2++)
            for (int64_t D = 0; D < W; D++) {
                double acc = 0.0;
                for (int64_t x = 0; x < N; x++)
                    for (int64_t y = 0; y < N; y++) {
                        int64_t z = L[s1 * N + x] + L[s2 * N + y] + D - 2 * N;
                        if (z >= 0 && z < N) acc += g[(x * N + y) * N + z];
                    }
                out[(s1 * N + s2) * W + D] = acc;
            }
    free(L);
    return 0;
}

/* One output of eq:3DfDRT by direct summation, O(N^2): used for sampled
 * parity checks at BASELINE sizes.  long double accumulation (exact for the
 * integer configs, >= fp64 for the float config). */
double oracle_drt_point_f64(const double *g, int64_t N, int64_t s1, int64_t s2, int64_t D) {
    int n = ilog2_exact(N);
    long double acc = 0.0L;
    for (int64_t x = 0; x < N; x++) {
        int64_t lx = oracle_line(n, s1, x);
        for (int64_t y = 0; y < N; y++) {
            int64_t z = lx + oracle_line(n, s2, y) + D - 2 * N;
            if (z >= 0 && z < N) acc += g[(x * N + y) * N + z];
        }
    }
    return (double)acc;
}

/* Same as above, sum of |g| (the F6 / C-amb-14 tolerance scale). */
double oracle_drt_point_abs_f64(const double *g, int64_t N, int64_t s1, int64_t s2, int64_t D) {
    int n = ilog2_exact(N);
    long double acc = 0.0L;
    for (int64_t x = 0; x < N; x++) {
        int64_t lx = oracle_line(n, s1, x);
        for (int64_t y = 0; y < N; y++) {
            int64_t z = lx + oracle_line(n, s2, y) + D - 2 * N;
            if (z >= 0 && z < N) acc += fabs(g[(x * N + y) * N + z]);
        }
    }
    return (double)acc;
}

/* Separable direct sum (Wu & Brady): two 2D DRT
 * definitions (eq:GotzfDRT) in sequence:
 *   G_{s1}(y, w) = sum_x g(x, y, l_{s1}(x) + w - 2N),   w in [0, 3N)
 *   out(s1,s2,D) = sum_y G_{s1}(y, l_{s2}(y) + D).
 * O(5 N^4); an independent route to eq:3DfDRT usable at N = 32..64. */
int oracle_drt_separable_f64(const double *g, int64_t N, double *out) {
    int n = ilog2_exact(N);
    if (n < 0) return -1;
    int64_t *L = line_table(n);
    int64_t W = 3 * N;
    double *G = (double *)calloc((size_t)(N * W), sizeof(double));
    for (int64_t s1 = 0; s1 < N; s1++) {
        for (int64_t y = 0; y < N; y++)
            for (int64_t w = 0; w < W; w++) {
                double acc = 0.0;
                for (int64_t x = 0; x < N; x++) {
                    int64_t z = L[s1 * N + x] + w - 2 * N;
                    if (z >= 0 && z < N) acc += g[(x * N + y) * N + z];
                }
                G[y * W + w] = acc;
            }
        for (int64_t s2 = 0; s2 < N; s2++)
            for (int64_t D = 0; D < W; D++) {
                double acc = 0.0;
                for (int64_t y = 0; y < N; y++) {
                    int64_t w = L[s2 * N + y] + D;
                    if (w < W) acc += G[y * W + w];
                }
                out[(s1 * N + s2) * W + D] = acc;
            }
    }
    free(G);
    free(L);
    return 0;
}

/* Algorithm 1 basicDRT3D, transcribed loop for loop.
 * Reading C-amb-2: the write index "sigma, v" of PAPER.md:262 is sigma1, v1.
 * Reads at d + offset >= 3N return 0 ("should be 0 ... if overflow 3rd
 * dimension").  Two element types: int64 and fp64.  The
 * fp64 version sums f00+f10+f01+f11 left to right as written. */
#define ALG1_BODY(T)                                                                    \
    int n = ilog2_exact(N);                                                             \
    if (n < 0) return -1;                                                               \
    int64_t W = 3 * N;                                                                  \
    size_t cells = (size_t)(N * N * W);                                                 \
    T *fm = (T *)calloc(cells, sizeof(T));                 /* f^m <- zeros(N,N,3N)  */  \
    T *fm1 = (T *)calloc(cells, sizeof(T));                /* f^{m+1}               */  \
    for (int64_t x = 0; x < N; x++)                        /* f^m(:,:,2N:3N-1) <- f */  \
        for (int64_t y = 0; y < N; y++)                                                 \
            for (int64_t z = 0; z < N; z++) fm[(x * N + y) * W + 2 * N + z] = (T)g[(x * N + y) * N + z]; \
    for (int m = 0; m < n; m++) {                                                       \
        int64_t nv = ((int64_t)1 << (n - m - 1)), ns = ((int64_t)1 << m);                \
        for (int64_t d = 0; d < W; d++)                                                 \
            for (int64_t v1 = 0; v1 < nv; v1++)                                         \
                for (int64_t sg1 = 0; sg1 < ns; sg1++)                                  \
                    for (int64_t v2 = 0; v2 < nv; v2++)                                 \
                        for (int64_t sg2 = 0; sg2 < ns; sg2++)                          \
                            for (int64_t b1 = 0; b1 < 2; b1++)                          \
                                for (int64_t b2 = 0; b2 < 2; b2++) {                    \
                                    int64_t i0 = sg1 + (v1 << (m + 1));                  \
                                    int64_t i1 = sg1 + ns + (v1 << (m + 1));             \
                                    int64_t j0 = sg2 + (v2 << (m + 1));                  \
                                    int64_t j1 = sg2 + ns + (v2 << (m + 1));             \
                                    int64_t d10 = d + sg1 + b1;                          \
                                    int64_t d01 = d + sg2 + b2;                          \
                                    int64_t d11 = d + sg1 + sg2 + b1 + b2;               \
                                    T f00 = fm[(i0 * N + j0) * W + d];                   \
                                    T f10 = d10 < W ? fm[(i1 * N + j0) * W + d10] : (T)0; \
                                    T f01 = d01 < W ? fm[(i0 * N + j1) * W + d01] : (T)0; \
                                    T f11 = d11 < W ? fm[(i1 * N + j1) * W + d11] : (T)0; \
                                    int64_t oi = b1 + (sg1 << 1) + (v1 << (m + 1));      \
                                    int64_t oj = b2 + (sg2 << 1) + (v2 << (m + 1));      \
                                    fm1[(oi * N + oj) * W + d] = f00 + f10 + f01 + f11;  \
                                }                                                       \
        T *t = fm; fm = fm1; fm1 = t;                      /* swap buffers          */  \
    }                                                                                   \
    memcpy(out, fm, cells * sizeof(T));                                                 \
    free(fm); free(fm1);                                                                \
    return 0;

int oracle_drt_alg1_i64(const int64_t *g, int64_t N, int64_t *out) { ALG1_BODY(int64_t) }
int oracle_drt_alg1_f64(const double *g, int64_t N, double *out) { ALG1_BODY(double) }

/* Adjoint of Alg. 1 by eq:invmap3Dsummation, run as the
 * "reversal in the order of the m loop":
 *   b^m(sigma1|v1m,v1|sigma2|v2m,v2|d) = sum_{b1,b2} b^{m+1}(b1,sigma1|v1|b2,sigma2|v2|
 *                                  d - v1m (b1 + sigma1) - v2m (b2 + sigma2)),
 * reads below index 0 are 0.  Input: N*N*3N coefficients; output: the N^3
 * cube read from b^0(:,:,2N:3N-1) (the adjoint of the seeding step). */
int oracle_drt_adjoint_f64(const double *coef, int64_t N, double *g) {
    int n = ilog2_exact(N);
    if (n < 0) return -1;
    int64_t W = 3 * N;
    size_t cells = (size_t)(N * N * W);
    double *bm1 = (double *)malloc(cells * sizeof(double)); /* b^{m+1} */
    double *bm = (double *)malloc(cells * sizeof(double));  /* b^m     */
    memcpy(bm1, coef, cells * sizeof(double));
    for (int m = n - 1; m >= 0; m--) {
        int64_t nv = ((int64_t)1 << (n - m - 1)), ns = ((int64_t)1 << m);
        for (int64_t d = 0; d < W; d++)
            for (int64_t v1 = 0; v1 < nv; v1++)
                for (int64_t sg1 = 0; sg1 < ns; sg1++)
                    for (int64_t v1m = 0; v1m < 2; v1m++)
                        for (int64_t v2 = 0; v2 < nv; v2++)
                            for (int64_t sg2 = 0; sg2 < ns; sg2++)
                                for (int64_t v2m = 0; v2m < 2; v2m++) {
                                    double acc = 0.0;
                                    for (int64_t b1 = 0; b1 < 2; b1++)
                                        for (int64_t b2 = 0; b2 < 2; b2++) {
                                            int64_t dd = d - v1m * (b1 + sg1) - v2m * (b2 + sg2);
                                            if (dd < 0) continue;
                                            int64_t oi = b1 + (sg1 << 1) + (v1 << (m + 1));
                                            int64_t oj = b2 + (sg2 << 1) + (v2 << (m + 1));
                                            acc += bm1[(oi * N + oj) * W + dd];
                                        }
                                    int64_t ii = sg1 + (v1m << m) + (v1 << (m + 1));
                                    int64_t jj = sg2 + (v2m << m) + (v2 << (m + 1));
                                    bm[(ii * N + jj) * W + d] = acc;
                                }
        double *t = bm; bm = bm1; bm1 = t;
    }
    for (int64_t x = 0; x < N; x++)
        for (int64_t y = 0; y < N; y++)
            for (int64_t z = 0; z < N; z++) g[(x * N + y) * N + z] = bm1[(x * N + y) * W + 2 * N + z];
    free(bm); free(bm1);
    return 0;
}

/* ------------------------------------------------------------ L2 lines --
 * eq:3DfDJT, brute force:
 *   out(s1,s2,D1,D2) = sum_u g(u, l_{s1}(u) + D1 - N, l_{s2}(u) + D2 - N),
 * in-range terms only.  Output N*N*2N*2N. */
int oracle_djt_brute_f64(const double *g, int64_t N, double *out) {
    int n = ilog2_exact(N);
    if (n < 0) return -1;
    int64_t *L = line_table(n);
    int64_t W = 2 * N;
    for (int64_t s1 = 0; s1 < N; s1++)
        for (int64_t s2 = 0; s2 < N; s2++)
            for (int64_t D1 = 0; D1 < W; D1++)
                for (int64_t D2 = 0; D2 < W; D2++) {
                    double acc = 0.0;
                    for (int64_t u = 0; u < N; u++) {
                        int64_t y = L[s1 * N + u] + D1 - N, z = L[s2 * N + u] + D2 - N;
                        if (y >= 0 && y < N && z >= 0 && z < N) acc += g[(u * N + y) * N + z];
                    }
                    out[((s1 * N + s2) * W + D1) * W + D2] = acc;
                }
    free(L);
    return 0;
}

double oracle_djt_point_f64(const double *g, int64_t N, int64_t s1, int64_t s2, int64_t D1, int64_t D2) {
    int n = ilog2_exact(N);
    long double acc = 0.0L;
    for (int64_t u = 0; u < N; u++) {
        int64_t y = oracle_line(n, s1, u) + D1 - N, z = oracle_line(n, s2, u) + D2 - N;
        if (y >= 0 && y < N && z >= 0 && z < N) acc += g[(u * N + y) * N + z];
    }
    return (double)acc;
}

/* Algorithm 3 basicDJT3D, loop for loop.  Stage buffer
 * N^2 x 2N x 2N with packed first index (v: n-m bits | s1: m bits | s2: m bits),
 * "greater significance to the right".  Reads beyond 2N-1
 * are 0.  separateS1S2: packed index
 * s1 + N*s2 -> out[s1][s2]. */
#define ALG3_BODY(T)                                                                    \
    int n = ilog2_exact(N);                                                             \
    if (n < 0) return -1;                                                               \
    int64_t W = 2 * N;                                                                  \
    size_t cells = (size_t)(N * N * W * W);                                             \
    T *fm = (T *)calloc(cells, sizeof(T));                                              \
    T *fm1 = (T *)calloc(cells, sizeof(T));                                             \
    for (int64_t x = 0; x < N; x++)                       /* f^m(0:N-1,N:2N-1,N:2N-1) */\
        for (int64_t y = 0; y < N; y++)                                                 \
            for (int64_t z = 0; z < N; z++) fm[(x * W + N + y) * W + N + z] = (T)g[(x * N + y) * N + z]; \
    for (int m = 0; m < n; m++) {                                                       \
        int64_t nv = ((int64_t)1 << (n - m - 1)), ns = ((int64_t)1 << m);                \
        for (int64_t d2 = 0; d2 < W; d2++)                                              \
            for (int64_t d1 = 0; d1 < W; d1++)                                          \
                for (int64_t sg2 = 0; sg2 < ns; sg2++)                                  \
                    for (int64_t b2 = 0; b2 < 2; b2++)                                  \
                        for (int64_t sg1 = 0; sg1 < ns; sg1++)                          \
                            for (int64_t b1 = 0; b1 < 2; b1++)                          \
                                for (int64_t v = 0; v < nv; v++) {                      \
                                    int64_t i0 = (v << 1) + (sg1 << (n - m)) + (sg2 << n); \
                                    int64_t i1 = 1 + i0;                                 \
                                    int64_t e1 = d1 + sg1 + b1, e2 = d2 + sg2 + b2;      \
                                    T f0 = fm[(i0 * W + d1) * W + d2];                   \
                                    T f1 = (e1 < W && e2 < W) ? fm[(i1 * W + e1) * W + e2] : (T)0; \
                                    int64_t o = v + (b1 << (n - m - 1)) + (sg1 << (n - m)) + (b2 << n) + (sg2 << (n + 1)); \
                                    fm1[(o * W + d1) * W + d2] = f0 + f1;                \
                                }                                                       \
        T *t = fm; fm = fm1; fm1 = t;                                                   \
    }                                                                                   \
    for (int64_t s1 = 0; s1 < N; s1++)                        /* separateS1S2 */         \
        for (int64_t s2 = 0; s2 < N; s2++)                                              \
            memcpy(out + ((s1 * N + s2) * W) * W, fm + ((s1 + N * s2) * W) * W, sizeof(T) * W * W); \
    free(fm); free(fm1);                                                                \
    return 0;

int oracle_djt_alg3_i64(const int64_t *g, int64_t N, int64_t *out) { ALG3_BODY(int64_t) }
int oracle_djt_alg3_f64(const double *g, int64_t N, double *out) { ALG3_BODY(double) }

/* Adjoint of Alg. 3 by eq:invmap3DJsummation:
 *   b^m(v_m, v | sigma1 | sigma2 | d1 | d2) = sum_{b1,b2} b^{m+1}(v | b1,sigma1 | b2,sigma2 |
 *                         d1 - v_m (b1 + sigma1) | d2 - v_m (b2 + sigma2)),
 * reads below 0 are 0.  Input out[s1][s2][D1][D2]; output cube from
 * b^0(x, N+y, N+z). */
int oracle_djt_adjoint_f64(const double *coef, int64_t N, double *g) {
    int n = ilog2_exact(N);
    if (n < 0) return -1;
    int64_t W = 2 * N;
    size_t cells = (size_t)(N * N * W * W);
    double *bm1 = (double *)malloc(cells * sizeof(double));
    double *bm = (double *)malloc(cells * sizeof(double));
    for (int64_t s1 = 0; s1 < N; s1++)                       /* inverse of separateS1S2 */
        for (int64_t s2 = 0; s2 < N; s2++)
            memcpy(bm1 + ((s1 + N * s2) * W) * W, coef + ((s1 * N + s2) * W) * W, sizeof(double) * W * W);
    for (int m = n - 1; m >= 0; m--) {
        int64_t nv = ((int64_t)1 << (n - m - 1)), ns = ((int64_t)1 << m);
        for (int64_t d2 = 0; d2 < W; d2++)
            for (int64_t d1 = 0; d1 < W; d1++)
                for (int64_t sg2 = 0; sg2 < ns; sg2++)
                    for (int64_t sg1 = 0; sg1 < ns; sg1++)
                        for (int64_t v = 0; v < nv; v++)
                            for (int64_t vm = 0; vm < 2; vm++) {
                                double acc = 0.0;
                                for (int64_t b1 = 0; b1 < 2; b1++)
                                    for (int64_t b2 = 0; b2 < 2; b2++) {
                                        int64_t e1 = d1 - vm * (b1 + sg1), e2 = d2 - vm * (b2 + sg2);
                                        if (e1 < 0 || e2 < 0) continue;
                                        int64_t o = v + (b1 << (n - m - 1)) + (sg1 << (n - m)) + (b2 << n) + (sg2 << (n + 1));
                                        acc += bm1[(o * W + e1) * W + e2];
                                    }
                                int64_t i = vm + (v << 1) + (sg1 << (n - m)) + (sg2 << n);
                                bm[(i * W + d1) * W + d2] = acc;
                            }
        double *t = bm; bm = bm1; bm1 = t;
    }
    for (int64_t x = 0; x < N; x++)
        for (int64_t y = 0; y < N; y++)
            for (int64_t z = 0; z < N; z++) g[(x * N + y) * N + z] = bm1[(x * W + N + y) * W + N + z];
    free(bm); free(bm1);
    return 0;
}
