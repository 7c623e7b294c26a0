// api.cu -- C ABI (include/drt3d.h): validation, pass planning, workspace
// sizing and kernel launches for the 3D DRT of planes and 3D DJT of lines.
#include "drt3d.h"

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "dispatch.h"
#include "adjoint.h"

using namespace d3;


namespace {

// Zero the 4 unused N x N blocks of the Alg. 2 mosaic.
__global__ void mosaic_fill_kernel(void *out, int N, int batch, int elt_bytes, int i0, int j0) {
    const long long row = blockIdx.x;                 // 0 .. batch*N*N-1
    const int b = (int)(row / ((long long)N * N));
    const int rr = (int)(row % ((long long)N * N));
    const int i = rr / N, j = rr % N;
    const long long W = 3LL * N - 2;
    const long long base = (long long)b * 16 * N * N * W + ((long long)(i0 * N + i) * 4 * N + (j0 * N + j)) * W;
    char *o = reinterpret_cast<char *>(out) + base * elt_bytes;
    for (long long e = threadIdx.x; e < W * elt_bytes; e += blockDim.x) o[e] = 0;
}



// ------------------------------------------------------------ tables --------
// The library's own copy of the orientation tables (R6-R8).
// Alg. 2 InOrder, printed.
const int8_t kDrtPrinted[12][3] = {{1, 2, 3},   {-2, 1, 3},   {-1, -2, 3},  {2, -1, 3},
                                   {-1, -3, -2}, {-3, -1, 2},  {3, -1, -2},  {1, 3, -2},
                                   {-3, -2, -1}, {-2, -3, 1},  {-2, 3, -1},  {3, 2, -1}};
// Repaired plane table: rows 5 and 9 complete the y- and x-normal sets (R7).
const int8_t kDrtHemisphere[12][3] = {{1, 2, 3},   {-2, 1, 3},  {-1, -2, 3},  {2, -1, 3},
                                      {-1, -3, -2}, {-3, 1, -2}, {3, -1, -2},  {1, 3, -2},
                                      {-3, -2, -1}, {2, -3, -1}, {-2, 3, -1},  {3, 2, -1}};
// Complete, identity-anchored line table (R8): x-, z-, y-driven sets.
const int8_t kDjtHemisphere[12][3] = {{1, 2, 3},   {1, -3, 2},   {1, -2, -3},  {1, 3, -2},
                                      {-3, -2, -1}, {-3, -1, 2},  {-3, 1, -2},  {-3, 2, 1},
                                      {-2, -1, -3}, {-2, 3, -1},  {-2, -3, 1},  {-2, 1, 3}};
// One table complete for planes and lines (R8, alternative).
const int8_t kShared[12][3] = {{1, 2, 3},  {-2, 1, 3}, {-1, -2, 3}, {2, -1, 3},  {3, 1, 2},   {-1, 3, 2},
                               {3, -1, -2}, {1, 3, -2}, {2, 3, 1},   {3, -2, 1},  {-2, 3, -1}, {3, 2, -1}};
// Alg. 2 OutOrder as the mosaic applies it, and DodecantCoords.
// Rows 4-11 are printed verbatim; rows 0-3 (the z-set) are the repaired rows of reading R13
// (DESIGN.md): fig:shapeOutput has the dodecants "fit accurately", i.e. the
// boundary planes two dodecants share lie on facing block edges, and these are the unique rows
// that do so (the printed z-set rows act as if s1 and s2 were exchanged).
const int8_t kOutOrder[12][3] = {{-1, -2, 3}, {-2, 1, 3}, {1, 2, 3},  {2, -1, 3}, {2, 1, 3},  {1, -2, 3},
                                 {-1, 2, 3},  {-2, -1, 3}, {2, 1, 3}, {-1, 2, 3}, {1, -2, 3}, {-2, -1, 3}};
const int8_t kCoords[12][2] = {{1, 1}, {1, 2}, {2, 2}, {2, 1}, {0, 2}, {0, 1},
                               {3, 2}, {3, 1}, {2, 0}, {1, 0}, {2, 3}, {1, 3}};

const int8_t (*table_rows(int table, int transform))[3] {
    if (table == DRT3D_TABLE_HEMISPHERE) return transform == 0 ? kDrtHemisphere : kDjtHemisphere;
    if (table == DRT3D_TABLE_PRINTED) return kDrtPrinted;
    if (table == DRT3D_TABLE_SHARED) return kShared;
    return nullptr;
}

// reading A: oriented axis j = original axis |p_j| (1=x, 2=y, 3=z),
// reversed when p_j < 0.  Original strides: x N^2, y N, z 1.
Orient make_orient(const int8_t row[3], int N, int dod) {
    Orient o{};
    long long stride[3] = {(long long)N * N, (long long)N, 1};
    long long s[3];
    o.off0 = 0;
    o.fast = 0;
    for (int j = 0; j < 3; ++j) {
        const int a = (row[j] < 0 ? -row[j] : row[j]) - 1;
        if (row[j] > 0) s[j] = stride[a];
        else { s[j] = -stride[a]; o.off0 += (long long)(N - 1) * stride[a]; }
        if (a == 2) o.fast = j;
    }
    o.sx = s[0];
    o.sy = s[1];
    o.sz = s[2];
    o.dod = dod;
    return o;
}

// ------------------------------------------------------------ planning ------
int stor_bytes(int s) { return s == ST_U8 ? 1 : s == ST_U16 ? 2 : 4; }
int round_up(int a, int b) { return (a + b - 1) / b * b; }

struct Plan {
    int transform;          // 0 DRT, 1 DJT
    int N, n, batch, ndod, inst;
    int npass;
    int ks[4];              // radix bits of each pass
    int cs[5];              // bits done before pass p (cs[npass] = n)
    int stor[5];            // storage type of stage cs[p] (stor[0] = input dtype)
    int base[5], width[5], pitch[5];
    long long plane[5];     // DJT: elements per plane
    long long inst_elems[5];// elements per instance of stage buffers
    int chunk;              // instances per chunk
    size_t buf_bytes;       // one intermediate buffer (chunk instances)
    int nbuf;
    int nset;               // 2: consecutive chunks use alternate buffer sets (cross-stream overlap)
    size_t ws_bytes;
    int nlaunch;
    int small;              // 2: the separable on-chip
                            // N = 32 kernel (k_sep32.cu), 3: the one-CTA N = 16 kernel (k_sep16.cu);
                            // one launch, no workspace
};

#ifndef D3_CHUNK_MB
#define D3_CHUNK_MB 512
#endif
// Intermediates per chunk.  Large chunks win (measured): one first-pass launch over
// many dodecants re-reads the cube from L2 and neither launch has a partial last wave; the stage
// buffers then live in HBM (they do not stay in L2 under the output stream anyway).
const size_t kChunkBudget = (size_t)D3_CHUNK_MB << 20;
// DRT pipeline (run_drt): instances of a chunk are split into up to D3_OVERLAP_GROUPS groups whose
// first pass overlaps the previous group's later passes; D3_FINAL_PRIORITY = 1 gives the later
// passes' stream the higher scheduling priority.
#ifndef D3_OVERLAP_GROUPS
#define D3_OVERLAP_GROUPS 1
#endif
#ifndef D3_FINAL_PRIORITY
#define D3_FINAL_PRIORITY 0
#endif
#ifndef D3_ZERO_BY_FIRST
#define D3_ZERO_BY_FIRST 0          // measured: 1.2213 ms per cfg3 step vs 1.1488 with the final pass's own TMA zero tiles
#endif
#ifndef D3_OVERLAP_MIN_N
#define D3_OVERLAP_MIN_N 128
#endif

int ilog2_exact(int N) {
    if (N < 2 || N > 1024) return -1;
    int n = 0;
    while ((1 << n) < N) ++n;
    return (1 << n) == N ? n : -1;
}

drt3d_opts default_opts() {
    drt3d_opts o{};
    o.batch = 1;
    o.in_dtype = DRT3D_U8;
    o.out_dtype = DRT3D_I32;
    o.layout = DRT3D_LAYOUT_STACKED;
    o.table = DRT3D_TABLE_HEMISPHERE;
    return o;
}

int popcount12(uint32_t m) {
    int c = 0;
    for (int k = 0; k < 12; ++k) c += (m >> k) & 1;
    return c;
}

drt3d_status make_plan(int transform, int N, uint32_t mask, const drt3d_opts &o, Plan &P) {
    std::memset(&P, 0, sizeof(P));
    const int n = ilog2_exact(N);
    if (n < 0) return DRT3D_ERR_INVALID_ARG;
    if (mask == 0 || mask >= (1u << 12)) return DRT3D_ERR_INVALID_ARG;
    if (o.batch < 1) return DRT3D_ERR_INVALID_ARG;
    const bool dt_ok = (o.in_dtype == DRT3D_U8 && o.out_dtype == DRT3D_I32) ||
                       (o.in_dtype == DRT3D_I32 && o.out_dtype == DRT3D_I32) ||
                       (o.in_dtype == DRT3D_F32 && o.out_dtype == DRT3D_F32);
    if (!dt_ok) return DRT3D_ERR_INVALID_ARG;
    if (o.table < 0 || o.table > 2) return DRT3D_ERR_INVALID_ARG;
    if (o.layout != DRT3D_LAYOUT_STACKED && o.layout != DRT3D_LAYOUT_MOSAIC) return DRT3D_ERR_INVALID_ARG;
    if (o.layout == DRT3D_LAYOUT_MOSAIC && (transform != 0 || mask != 0xFFFu)) return DRT3D_ERR_INVALID_ARG;

    P.transform = transform;
    P.N = N;
    P.n = n;
    P.batch = o.batch;
    P.ndod = popcount12(mask);
    P.inst = P.batch * P.ndod;
    // pass radices: <= 4 stages per pass, the first pass takes the larger half
#ifndef D3_N16_TWO_PASS_MAX_INST
#define D3_N16_TWO_PASS_MAX_INST 24
#endif
    // N = 16 with few instances (one cube, up to 2 x 12 dodecants): two radix-4 passes instead of one
    // radix-16 pass -- a few large CTAs of the radix-16 kernel are latency-bound (cfg1: 0.0195 ->
    // 0.0132 ms, one cube x 12 dodecants 0.0174 -> 0.0133 ms); large batches keep the single pass
    // (no intermediate: 64 fp32 cubes x 12 0.046 vs 0.064 ms)
    if (transform == 0 && n == 4 && P.inst <= D3_N16_TWO_PASS_MAX_INST) { P.npass = 2; P.ks[0] = 2; P.ks[1] = 2; }
    else if (n <= 4) { P.npass = 1; P.ks[0] = n; }
    else if (n <= 8) {
        P.npass = 2;
        P.ks[0] = (n + 1) / 2;
        P.ks[1] = n / 2;
#ifndef D3_DJT_K1
#define D3_DJT_K1 0
#endif
        if (transform == 1 && D3_DJT_K1 > 0 && D3_DJT_K1 < n && D3_DJT_K1 <= 4 && n - D3_DJT_K1 <= 4) {
            P.ks[0] = D3_DJT_K1;
            P.ks[1] = n - D3_DJT_K1;
        }
#ifndef D3_DRT6_K1_U8
#define D3_DRT6_K1_U8 4
#endif
        // u8 voxels at N = 64: the SWAR radix-16 first pass (two 16-bit lanes per add) does more of
        // the work, 4 | 2 instead of 3 | 3 (cfg2 0.0461 -> 0.0358 ms; 2 | 4: 0.042); fp32 / int32
        // keep 3 | 3 (8 fp32 cubes x 12: 0.198 ms vs 0.259 at 4 | 2)
#ifndef D3_PLAN_K1
#define D3_PLAN_K1 0                    // measurement builds: first-pass radix of every 2-pass plan
#endif
        if (D3_PLAN_K1 > 0 && D3_PLAN_K1 < n && D3_PLAN_K1 <= 4 && n - D3_PLAN_K1 <= 4) {
            P.ks[0] = D3_PLAN_K1;
            P.ks[1] = n - D3_PLAN_K1;
        } else if (transform == 0 && n == 6 && o.in_dtype == DRT3D_U8 && D3_DRT6_K1_U8 > 0 && D3_DRT6_K1_U8 <= 4 &&
            n - D3_DRT6_K1_U8 <= 4) {
            P.ks[0] = D3_DRT6_K1_U8;
            P.ks[1] = n - D3_DRT6_K1_U8;
        }
    }
    else { P.npass = 3; P.ks[0] = 4; P.ks[1] = (n - 3) / 2; P.ks[2] = n - 4 - P.ks[1]; }
    P.cs[0] = 0;
    for (int p = 0; p < P.npass; ++p) P.cs[p + 1] = P.cs[p] + P.ks[p];

    P.stor[0] = o.in_dtype == DRT3D_U8 ? ST_U8 : o.in_dtype == DRT3D_I32 ? ST_U32 : ST_F32;
    for (int p = 1; p <= P.npass; ++p) {
        const int c = P.cs[p];
        if (o.in_dtype == DRT3D_F32) P.stor[p] = ST_F32;
        else if (o.in_dtype == DRT3D_I32) P.stor[p] = ST_U32;
        else {
            // u8 voxels: a stage-c partial sum adds 4^c (planes) or 2^c (lines)
            // voxels <= 255, which fits 16 bits while 255 * count < 2^16.
            const long long cnt = transform == 0 ? (1LL << (2 * c)) : (1LL << c);
            P.stor[p] = (p < P.npass && 255LL * cnt < 65536LL) ? ST_U16 : ST_U32;
        }
        if (transform == 0) {
            if (p == P.npass) { P.base[p] = 0; P.width[p] = 3 * N; P.pitch[p] = 3 * N; }
            else {
                // stage-c support starts at D = 2N - 2(2^c - 1) (eq:3Dfm).  Rows are
                // stored pre-shifted left by rho < EPC elements (DESIGN.md "Aligned stage buffers",
                // EPC = elements per 16-byte chunk), so the stored origin sits at least EPC - 1 below
                // the support, rounded down to a chunk so that every reader window starts on one;
                // the pitch is a whole number of chunks and rows are computed (zero-padded) up to
                // it, so any chunk inside a row is valid data.
                // Origin granularity: a pass stages its input from chunk (D_tile - base_in) / EPC_in
                // with D_tile = base_out + a multiple of its tile width, so base_out - base_in must
                // be a multiple of the INPUT's chunk (8 for u16, 4 for 32-bit), and the final
                // origin is 0.  All origins are multiples of 16 when a u16 level is involved (this
                // level or the one before it: u8 three-pass plans, N >= 512, where a 32-bit level
                // after a u16 one must not round to 4) -- the first pass's vector cube loads also
                // want z' = D - 2N on 16 bytes; all-32-bit plans keep 4 (narrower rows at small N).
                const int epc = 16 / stor_bytes(P.stor[p]);
                const bool u16_near = P.stor[p] == ST_U16 || (p >= 2 && P.stor[p - 1] == ST_U16);
                const int gb = u16_near ? 16 : epc;
                P.base[p] = (2 * N - 2 * ((1 << c) - 1) - (epc - 1)) / gb * gb;
                P.pitch[p] = round_up(3 * N - P.base[p], epc);
                P.width[p] = P.pitch[p];
            }
            P.inst_elems[p] = (long long)N * N * P.pitch[p];
        } else {
            if (p == P.npass) { P.base[p] = 0; P.width[p] = 2 * N; P.pitch[p] = 2 * N; }
            else {
                P.base[p] = N - ((1 << c) - 1);
                P.width[p] = N + (1 << c) - 1;
                P.pitch[p] = round_up(P.width[p], 8);
            }
            P.plane[p] = (long long)P.width[p] * P.pitch[p];
            P.inst_elems[p] = (long long)N * (1LL << c) * P.plane[p];
        }
    }
    P.base[0] = transform == 0 ? 2 * N : N;
#ifndef D3_SEP16
#define D3_SEP16 1
#endif
    // N = 16: every stage of an instance in one CTA (k_sep16.cu), one launch, no stage buffer;
    // -DD3_SEP16=0 keeps the pass kernels (measurement builds)
    if (transform == 0 && N == 16 && o.layout == DRT3D_LAYOUT_STACKED && D3_SEP16) {
        P.small = 3;
        P.chunk = P.inst;
        P.nset = 1;
        P.ws_bytes = 0;
        P.nlaunch = 1;
        return DRT3D_OK;
    }
#ifndef D3_SEP32
#define D3_SEP32 1
#endif
    // N = 32: the separable on-chip kernel (k_sep32.cu), one 4-CTA cluster per instance, no stage
    // buffer; default for every dtype (256 cubes x 12 dodecants: u8 0.642 ms, i32 0.686, f32 0.713,
    // against 0.990 / 0.731 / 0.739 for round 1's kernels).  -DD3_SEP32=0 keeps the
    // pass kernels (measurement builds)
    if (transform == 0 && N == 32 && o.layout == DRT3D_LAYOUT_STACKED && D3_SEP32) {
        P.small = 2;
        P.chunk = P.inst;
        P.nset = 1;
        P.ws_bytes = 0;
        P.nlaunch = 1;
        return DRT3D_OK;
    }
    P.width[0] = N;
    size_t per_inst = 0;
    for (int p = 1; p < P.npass; ++p) {
        const size_t b = (size_t)P.inst_elems[p] * stor_bytes(P.stor[p]);
        if (b > per_inst) per_inst = b;
    }
    if (P.npass == 1) { P.chunk = P.inst; P.nbuf = 0; P.buf_bytes = 0; }
    else {
        long long ch = (long long)(kChunkBudget / (per_inst ? per_inst : 1));
        if (ch < 1) ch = 1;
        if (ch > P.inst) ch = P.inst;
        if (ch > 65535) ch = 65535;
        P.chunk = (int)ch;
        P.nbuf = P.npass >= 3 ? 2 : 1;
        P.buf_bytes = ((per_inst * (size_t)P.chunk + 255) / 256) * 256;
    }
    const int nchunks = (P.inst + P.chunk - 1) / P.chunk;
    P.nset = (transform == 0 && P.npass > 1 && nchunks > 1) ? 2 : 1;
    P.ws_bytes = P.buf_bytes * P.nbuf * P.nset;
    P.nlaunch = nchunks * P.npass + ((o.layout == DRT3D_LAYOUT_MOSAIC) ? 4 : 0);
    return DRT3D_OK;
}

// ------------------------------------------------------------ launching -----
struct Launcher {
    cudaStream_t stream;
    const drt3d_opts *o;
    int count = 0;
    template <class F>
    drt3d_status run(int kind, F &&launch) { return run_on(stream, kind, launch); }
    template <class F>
    drt3d_status run_on(cudaStream_t stream, int kind, F &&launch) {
        cudaEvent_t *ev = o && o->events ? reinterpret_cast<cudaEvent_t *>(o->events) : nullptr;
        const bool rec = ev && count < o->max_events;
        if (rec) cudaEventRecord(ev[2 * count], stream);
        launch();
        if (rec) cudaEventRecord(ev[2 * count + 1], stream);
        if (o && o->launch_kind && count < o->max_events) o->launch_kind[count] = kind;
        ++count;
        return cudaGetLastError() == cudaSuccess ? DRT3D_OK : DRT3D_ERR_CUDA;
    }
};

drt3d_status dispatch_drt(int in_dtype, int K, int sin, int sout, bool first, bool fin, const DrtPass &prm, int ninst,
                          cudaStream_t st) {
    if (in_dtype == DRT3D_U8) return dispatch_drt_u8(K, sin, sout, first, fin, prm, ninst, st);
    if (in_dtype == DRT3D_I32) return dispatch_drt_i32(K, sin, sout, first, fin, prm, ninst, st);
    return dispatch_drt_f32(K, sin, sout, first, fin, prm, ninst, st);
}
drt3d_status dispatch_djt(int in_dtype, int K, int sin, int sout, bool first, bool fin, const DjtPass &prm, int ninst,
                          cudaStream_t st) {
    if (in_dtype == DRT3D_U8) return dispatch_djt_u8(K, sin, sout, first, fin, prm, ninst, st);
    if (in_dtype == DRT3D_I32) return dispatch_djt_i32(K, sin, sout, first, fin, prm, ninst, st);
    return dispatch_djt_f32(K, sin, sout, first, fin, prm, ninst, st);
}

size_t out_elems(int transform, const Plan &P, const drt3d_opts &o) {
    const size_t N = (size_t)P.N;
    if (transform == 0) {
        if (o.layout == DRT3D_LAYOUT_MOSAIC) return (size_t)P.batch * 16 * N * N * (3 * N - 2);
        return (size_t)P.inst * N * N * 3 * N;
    }
    return (size_t)P.inst * N * N * 4 * N * N;
}

int in_bytes(int dt) { return dt == DRT3D_U8 ? 1 : 4; }

drt3d_status check_ptrs(const void *cube, void *out, void *ws, size_t ws_bytes, const Plan &P, const drt3d_opts &o,
                        int transform) {
    if (!cube || !out) return DRT3D_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return DRT3D_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(cube) & 15) != 0) return DRT3D_ERR_INVALID_ARG;
    const size_t cb = (size_t)P.batch * P.N * P.N * P.N * in_bytes(o.in_dtype);
    const size_t ob = out_elems(transform, P, o) * 4;
    const uintptr_t c0 = reinterpret_cast<uintptr_t>(cube), o0 = reinterpret_cast<uintptr_t>(out);
    if (c0 < o0 + ob && o0 < c0 + cb) return DRT3D_ERR_INVALID_ARG;   // overlap
    if (P.ws_bytes > 0) {
        if (!ws || ws_bytes < P.ws_bytes) return DRT3D_ERR_WORKSPACE;
        if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return DRT3D_ERR_INVALID_ARG;
    }
    return DRT3D_OK;
}

// Auxiliary streams and events (DESIGN.md §5 "Overlap"): a pool per process, one entry per
// concurrently running call on a device, created on first use and reused by every later call on
// any host thread (never destroyed: the count is bounded by the number of concurrent callers, so
// nothing leaks per thread).  A call leases an entry for its duration; work it left on the entry's
// streams is joined into the caller's stream before the call returns (JoinGuard, every exit path),
// so a later lessee's work may queue behind it but is never unordered with it.
constexpr int kHostGroups = 4;
struct Aux {
    int dev = -1;
    bool busy = false;
    cudaStream_t a = nullptr;                    // later passes of the DRT pipeline
    cudaEvent_t start = nullptr, fdone = nullptr, join = nullptr, cdone[2] = {nullptr, nullptr};
    // host-buffer calls: device-to-host copies of finished dodecant groups
    cudaStream_t cp = nullptr;
    cudaEvent_t gdone[kHostGroups] = {}, cpdone = nullptr;
};
std::mutex g_aux_mu;
std::vector<Aux *> g_aux;

bool aux_create(Aux &x) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    bool e = cudaStreamCreateWithPriority(&x.a, cudaStreamNonBlocking, D3_FINAL_PRIORITY ? hi : lo) == cudaSuccess;
    e = e && cudaStreamCreateWithFlags(&x.cp, cudaStreamNonBlocking) == cudaSuccess;
    for (cudaEvent_t *ev : {&x.start, &x.fdone, &x.join, &x.cdone[0], &x.cdone[1], &x.cpdone})
        e = e && cudaEventCreateWithFlags(ev, cudaEventDisableTiming) == cudaSuccess;
    for (int g = 0; g < kHostGroups; ++g)
        e = e && cudaEventCreateWithFlags(&x.gdone[g], cudaEventDisableTiming) == cudaSuccess;
    return e;
}

void aux_destroy(Aux &x) {
    for (cudaStream_t sh : {x.a, x.cp})
        if (sh) cudaStreamDestroy(sh);
    for (cudaEvent_t ev : {x.start, x.fdone, x.join, x.cdone[0], x.cdone[1], x.cpdone})
        if (ev) cudaEventDestroy(ev);
    for (int g = 0; g < kHostGroups; ++g)
        if (x.gdone[g]) cudaEventDestroy(x.gdone[g]);
}

class AuxLease {
    Aux *x_ = nullptr;
public:
    explicit AuxLease(bool want) {
        if (!want) return;
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return;
        std::lock_guard<std::mutex> lk(g_aux_mu);
        for (Aux *c : g_aux)
            if (c->dev == dev && !c->busy) { x_ = c; break; }
        if (!x_) {
            Aux *c = new Aux();
            c->dev = dev;
            if (!aux_create(*c)) {                          // release what was created, run without
                aux_destroy(*c);
                delete c;
                return;
            }
            g_aux.push_back(c);
            x_ = c;
        }
        x_->busy = true;
    }
    ~AuxLease() {
        if (!x_) return;
        std::lock_guard<std::mutex> lk(g_aux_mu);
        x_->busy = false;
    }
    AuxLease(const AuxLease &) = delete;
    AuxLease &operator=(const AuxLease &) = delete;
    Aux *get() const { return x_; }
};

// Joins an auxiliary stream into the caller's stream when it goes out of scope (also on the
// error returns), so the caller's stream always orders after everything the call enqueued.
struct JoinGuard {
    cudaStream_t st, from;
    cudaEvent_t ev;
    ~JoinGuard() {
        if (from && cudaEventRecord(ev, from) == cudaSuccess) cudaStreamWaitEvent(st, ev, 0);
    }
};

// DRT pipeline over groups of instances (DESIGN.md §5 "Overlap"): the first pass of group g+1
// (latency-bound: SMEM and integer issue) runs on the caller's stream while the later passes of
// group g (HBM-write-bound) run on the auxiliary stream, so the two kinds of work share the SMs.
// Each instance has its own stage buffer slice inside the chunk, so groups never wait on each
// other's buffers; consecutive chunks of large batches alternate between two buffer sets.
drt3d_status run_drt(const void *cube, uint32_t mask, void *out, const drt3d_opts &o, const Plan &P, void *ws,
                     cudaStream_t st, bool reduce_sub = false, double *sq_part = nullptr, int *sq_count = nullptr) {
    if ((reduce_sub || sq_part) && (P.small || o.layout != DRT3D_LAYOUT_STACKED || o.out_dtype != DRT3D_F32))
        return DRT3D_ERR_UNSUPPORTED;
    const int8_t(*rows)[3] = table_rows(o.table, 0);
    DrtPass base{};
    base.N = P.N;
    base.n = P.n;
    base.ndod = P.ndod;
    base.layout = o.layout;
    base.vec_ok = (P.N >= 16) ? 1 : 0;
    base.one = 1;
    base.inst_total = P.inst;
    int j = 0;
    for (int k = 0; k < 12; ++k)
        if ((mask >> k) & 1) {
            base.ori[j] = make_orient(rows[k], P.N, k);
            base.out_order[j][0] = kOutOrder[k][0];
            base.out_order[j][1] = kOutOrder[k][1];
            base.coords[j][0] = kCoords[k][0];
            base.coords[j][1] = kCoords[k][1];
            ++j;
        }
    Launcher L{st, &o};
    if (P.small) {
        base.inst0 = 0;
        base.in = cube;
        base.out = out;
        drt3d_status s = DRT3D_OK;
        drt3d_status ls = L.run(2, [&] {
            s = P.small == 3 ? dispatch_drt_sep16(o.in_dtype, base, P.inst, st)
                             : dispatch_drt_sep32(o.in_dtype, base, P.inst, st);
        });
        if (s != DRT3D_OK) return s;
        if (o.launches) *o.launches = L.count;
        return ls;
    }
    const int ngroups_max =
        (P.npass > 1 && P.N >= D3_OVERLAP_MIN_N) ? (P.inst < D3_OVERLAP_GROUPS ? P.inst : D3_OVERLAP_GROUPS) : 1;
    AuxLease lease(P.npass > 1 && (ngroups_max > 1 || P.nset == 2));
    Aux *ax = lease.get();
    if (ax && (cudaEventRecord(ax->start, st) != cudaSuccess || cudaStreamWaitEvent(ax->a, ax->start, 0) != cudaSuccess))
        return DRT3D_ERR_CUDA;
    JoinGuard join{st, ax ? ax->a : nullptr, ax ? ax->join : nullptr};
    // -DD3_ZERO_BY_FIRST=1 (measurement builds): for u8 voxels, plan 4 | 4 (N = 256), stacked, the
    // final pass's all-zero tiles are written by the first pass (one TMA store of a zeroed
    // shared-memory tile each, DESIGN.md §5 item 6), and the final pass skips them
    const bool zfirst = D3_ZERO_BY_FIRST && o.in_dtype == DRT3D_U8 && o.layout == DRT3D_LAYOUT_STACKED &&
                        P.npass == 2 && P.ks[0] == 4 && P.ks[1] == 4 && (3 * P.N) % D3_FINAL16_T == 0;
    const long long final_inst = (o.layout == DRT3D_LAYOUT_MOSAIC) ? 0 : (long long)P.N * P.N * 3 * P.N;
    int chunk_idx = 0;
    for (int i0 = 0; i0 < P.inst; i0 += P.chunk, ++chunk_idx) {
        const int ninst = (P.inst - i0) < P.chunk ? (P.inst - i0) : P.chunk;
        const int set = (ax && P.nset == 2) ? (chunk_idx & 1) : 0;
        char *sb = reinterpret_cast<char *>(ws) + (size_t)set * P.buf_bytes * P.nbuf;
        if (ax && P.nset == 2 && chunk_idx >= 2) cudaStreamWaitEvent(st, ax->cdone[set], 0);   // buffer set free again
        const int ng = ax ? (ninst < ngroups_max ? ninst : ngroups_max) : 1;
        for (int g = 0, gi0 = 0; g < ng; ++g) {
            const int gn = ninst / ng + (g < ninst % ng ? 1 : 0);
            for (int p = 0; p < P.npass; ++p) {
                const bool first = p == 0, fin = p == P.npass - 1;
                cudaStream_t ps = (ax && !first) ? ax->a : st;
                if (ax && p == 1) {
                    if (cudaEventRecord(ax->fdone, st) != cudaSuccess || cudaStreamWaitEvent(ax->a, ax->fdone, 0) != cudaSuccess)
                        return DRT3D_ERR_CUDA;
                }
                // this group's slices of the chunk's stage buffers
                char *bin = sb + (size_t)((p - 1) & 1) * P.buf_bytes;
                char *bout = sb + (size_t)(p & 1) * P.buf_bytes;
                DrtPass prm = base;
                prm.c = P.cs[p];
                prm.m = P.n - P.cs[p + 1];
                prm.inst0 = i0 + gi0;
                prm.in = first ? cube : bin + (size_t)gi0 * P.inst_elems[p] * stor_bytes(P.stor[p]);
                prm.in_inst_stride = first ? 0 : P.inst_elems[p];
                prm.in_pitch = P.pitch[p];
                prm.in_base = P.base[p];
                prm.in_width = P.width[p];
                prm.out = fin ? out : bout + (size_t)gi0 * P.inst_elems[p + 1] * stor_bytes(P.stor[p + 1]);
                prm.out_inst_stride = fin ? final_inst : P.inst_elems[p + 1];
                prm.out_pitch = P.pitch[p + 1];
                prm.out_base = P.base[p + 1];
                prm.out_width = P.width[p + 1];
                prm.next_k = fin ? 0 : P.ks[p + 1];
                if (zfirst && first) {
                    prm.zf_T = D3_FINAL16_T;
                    prm.zf_out = out;
                    prm.zf_inst_stride = final_inst;
                }
                if (zfirst && fin) prm.zeros_by_first = 1;
                prm.reduce_sub = (reduce_sub && fin) ? 1 : 0;
                prm.sq_part = fin ? sq_part : nullptr;
                prm.sq_count = fin ? sq_count : nullptr;
                drt3d_status s = DRT3D_OK;
                drt3d_status ls = L.run_on(ps, first ? 0 : (fin ? 2 : 1), [&] {
                    s = dispatch_drt(o.in_dtype, P.ks[p], P.stor[p], P.stor[p + 1], first, fin, prm, gn, ps);
                });
                if (s != DRT3D_OK) return s;
                if (ls != DRT3D_OK) return ls;
            }
            gi0 += gn;
        }
        if (ax && P.nset == 2) cudaEventRecord(ax->cdone[set], ax->a);
    }
    if (o.layout == DRT3D_LAYOUT_MOSAIC) {
        // the 4 blocks of the 4x4 grid no dodecant occupies
        for (int bi = 0; bi < 4; ++bi)
            for (int bj = 0; bj < 4; ++bj) {
                bool used = false;
                for (int k = 0; k < 12; ++k) used |= (kCoords[k][0] == bi && kCoords[k][1] == bj);
                if (used) continue;
                drt3d_status ls = L.run(3, [&] {
                    mosaic_fill_kernel<<<P.batch * P.N * P.N, 128, 0, st>>>(out, P.N, P.batch, 4, bi, bj);
                });
                if (ls != DRT3D_OK) return ls;
            }
    }
    if (o.launches) *o.launches = L.count;
    return DRT3D_OK;
}

drt3d_status run_djt(const void *cube, uint32_t mask, void *out, const drt3d_opts &o, const Plan &P, void *ws,
                     cudaStream_t st) {
    const int8_t(*rows)[3] = table_rows(o.table, 1);
    DjtPass base{};
    base.N = P.N;
    base.n = P.n;
    base.ndod = P.ndod;
    base.vec_ok = (P.N >= 16) ? 1 : 0;
    base.inst_total = P.inst;
    int j = 0;
    for (int k = 0; k < 12; ++k)
        if ((mask >> k) & 1) base.ori[j++] = make_orient(rows[k], P.N, k);
    Launcher L{st, &o};
    char *buf[2] = {reinterpret_cast<char *>(ws), reinterpret_cast<char *>(ws) + P.buf_bytes};
    for (int i0 = 0; i0 < P.inst; i0 += P.chunk) {
        const int ninst = (P.inst - i0) < P.chunk ? (P.inst - i0) : P.chunk;
        for (int p = 0; p < P.npass; ++p) {
            const bool first = p == 0, fin = p == P.npass - 1;
            DjtPass prm = base;
            prm.c = P.cs[p];
            prm.m = P.n - P.cs[p + 1];
            prm.inst0 = i0;
            prm.in = first ? cube : buf[(p - 1) & 1];
            prm.in_inst_stride = first ? 0 : P.inst_elems[p];
            prm.in_plane = first ? 0 : P.plane[p];
            prm.in_pitch = P.pitch[p];
            prm.in_base = P.base[p];
            prm.in_width = P.width[p];
            prm.out = fin ? out : buf[p & 1];
            prm.out_inst_stride = P.inst_elems[p + 1];
            prm.out_plane = P.plane[p + 1];
            prm.out_pitch = P.pitch[p + 1];
            prm.out_base = P.base[p + 1];
            prm.out_width = P.width[p + 1];
            drt3d_status s = DRT3D_OK;
            drt3d_status ls = L.run(first ? 0 : (fin ? 2 : 1), [&] {
                s = dispatch_djt(o.in_dtype, P.ks[p], P.stor[p], P.stor[p + 1], first, fin, prm, ninst, st);
            });
            if (s != DRT3D_OK) return s;
            if (ls != DRT3D_OK) return ls;
        }
    }
    if (o.launches) *o.launches = L.count;
    return DRT3D_OK;
}

const drt3d_opts &opts_or_default(const drt3d_opts *o, drt3d_opts &tmp) {
    if (o) return *o;
    tmp = default_opts();
    return tmp;
}

}  // namespace

// ============================================================== C ABI =======
extern "C" {

const char *drt3d_status_string(drt3d_status s) {
    switch (s) {
        case DRT3D_OK: return "DRT3D_OK";
        case DRT3D_ERR_INVALID_ARG: return "DRT3D_ERR_INVALID_ARG";
        case DRT3D_ERR_UNSUPPORTED: return "DRT3D_ERR_UNSUPPORTED";
        case DRT3D_ERR_WORKSPACE: return "DRT3D_ERR_WORKSPACE";
        case DRT3D_ERR_CUDA: return "DRT3D_ERR_CUDA";
    }
    return "DRT3D_ERR_UNKNOWN";
}

drt3d_status drt3d_orientation_table(int table, int transform, int8_t rows[36]) {
    if (!rows || transform < 0 || transform > 1) return DRT3D_ERR_INVALID_ARG;
    const int8_t(*t)[3] = table_rows(table, transform);
    if (!t) return DRT3D_ERR_INVALID_ARG;
    for (int k = 0; k < 12; ++k)
        for (int j = 0; j < 3; ++j) rows[3 * k + j] = t[k][j];
    return DRT3D_OK;
}

size_t drt3d_planes_out_elems(int N, uint32_t mask, const drt3d_opts *opts) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    Plan P;
    if (make_plan(0, N, mask, o, P) != DRT3D_OK) return 0;
    return out_elems(0, P, o);
}

drt3d_status drt3d_planes_workspace_size(int N, uint32_t mask, const drt3d_opts *opts, size_t *bytes) {
    if (!bytes) return DRT3D_ERR_INVALID_ARG;
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    Plan P;
    drt3d_status s = make_plan(0, N, mask, o, P);
    if (s != DRT3D_OK) return s;
    *bytes = P.ws_bytes;
    return DRT3D_OK;
}

drt3d_status drt3d_planes(const void *cube, int N, uint32_t mask, void *out, const drt3d_opts *opts,
                          void *workspace, size_t workspace_bytes, void *stream) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    Plan P;
    drt3d_status s = make_plan(0, N, mask, o, P);
    if (s != DRT3D_OK) return s;
    s = check_ptrs(cube, out, workspace, workspace_bytes, P, o, 0);
    if (s != DRT3D_OK) return s;
    return run_drt(cube, mask, out, o, P, workspace, reinterpret_cast<cudaStream_t>(stream));
}

size_t djt3d_lines_out_elems(int N, uint32_t mask, const drt3d_opts *opts) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    Plan P;
    if (make_plan(1, N, mask, o, P) != DRT3D_OK) return 0;
    return out_elems(1, P, o);
}

drt3d_status djt3d_lines_workspace_size(int N, uint32_t mask, const drt3d_opts *opts, size_t *bytes) {
    if (!bytes) return DRT3D_ERR_INVALID_ARG;
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    Plan P;
    drt3d_status s = make_plan(1, N, mask, o, P);
    if (s != DRT3D_OK) return s;
    *bytes = P.ws_bytes;
    return DRT3D_OK;
}

drt3d_status djt3d_lines(const void *cube, int N, uint32_t mask, void *out, const drt3d_opts *opts, void *workspace,
                         size_t workspace_bytes, void *stream) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    Plan P;
    drt3d_status s = make_plan(1, N, mask, o, P);
    if (s != DRT3D_OK) return s;
    s = check_ptrs(cube, out, workspace, workspace_bytes, P, o, 1);
    if (s != DRT3D_OK) return s;
    return run_djt(cube, mask, out, o, P, workspace, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- adjoints
static drt3d_status adjoint_check(int transform, int N, uint32_t mask, const drt3d_opts &o, int &n) {
    n = ilog2_exact(N);
    if (n < 0 || mask == 0 || mask >= (1u << 12) || o.batch < 1) return DRT3D_ERR_INVALID_ARG;
    if (o.out_dtype != DRT3D_I32 && o.out_dtype != DRT3D_F32) return DRT3D_ERR_INVALID_ARG;
    if (o.table < 0 || o.table > 2 || o.layout != DRT3D_LAYOUT_STACKED) return DRT3D_ERR_INVALID_ARG;
    (void)transform;
    return DRT3D_OK;
}

static drt3d_status adjoint_ws(int transform, int N, uint32_t mask, const drt3d_opts *opts, size_t *bytes) {
    if (!bytes) return DRT3D_ERR_INVALID_ARG;
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    int n;
    drt3d_status s = adjoint_check(transform, N, mask, o, n);
    if (s != DRT3D_OK) return s;
    *bytes = d3::adjoint_workspace_bytes(transform, N, mask);
    return DRT3D_OK;
}

static drt3d_status adjoint_run(int transform, const void *coef, int N, uint32_t mask, void *cube,
                                const drt3d_opts *opts, void *ws, size_t ws_bytes, void *stream) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    int n;
    drt3d_status s = adjoint_check(transform, N, mask, o, n);
    if (s != DRT3D_OK) return s;
    if (!coef || !cube) return DRT3D_ERR_INVALID_ARG;
    // 16-byte staging copies / vector stores, like the forward transform
    if ((reinterpret_cast<uintptr_t>(coef) | reinterpret_cast<uintptr_t>(cube)) & 15) return DRT3D_ERR_INVALID_ARG;
    if (!ws || ws_bytes < d3::adjoint_workspace_bytes(transform, N, mask)) return DRT3D_ERR_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(ws) & 255) return DRT3D_ERR_WORKSPACE;
    const int K = popcount12(mask);
    const size_t cb = (size_t)o.batch * N * N * N * 4;
    const size_t ob = (size_t)o.batch * K * N * N * (transform == 0 ? 3 * N : 4 * N * N) * 4;
    const uintptr_t c0 = reinterpret_cast<uintptr_t>(cube), o0 = reinterpret_cast<uintptr_t>(coef);
    if (c0 < o0 + ob && o0 < c0 + cb) return DRT3D_ERR_INVALID_ARG;   // overlap
    return d3::run_adjoint(transform, coef, N, n, table_rows(o.table, transform), mask, o.batch, o.out_dtype, cube, ws,
                           reinterpret_cast<cudaStream_t>(stream), o.launches);
}

drt3d_status drt3d_planes_adjoint_workspace_size(int N, uint32_t mask, const drt3d_opts *opts, size_t *bytes) {
    return adjoint_ws(0, N, mask, opts, bytes);
}
drt3d_status drt3d_planes_adjoint(const void *coef, int N, uint32_t mask, void *cube, const drt3d_opts *opts,
                                  void *ws, size_t ws_bytes, void *stream) {
    return adjoint_run(0, coef, N, mask, cube, opts, ws, ws_bytes, stream);
}
drt3d_status djt3d_lines_adjoint_workspace_size(int N, uint32_t mask, const drt3d_opts *opts, size_t *bytes) {
    return adjoint_ws(1, N, mask, opts, bytes);
}
drt3d_status djt3d_lines_adjoint(const void *coef, int N, uint32_t mask, void *cube, const drt3d_opts *opts,
                                 void *ws, size_t ws_bytes, void *stream) {
    return adjoint_run(1, coef, N, mask, cube, opts, ws, ws_bytes, stream);
}

static drt3d_status host_variant(int transform, const void *host_cube, int N, uint32_t mask, void *host_out,
                                 const drt3d_opts *opts, void *dev_cube, void *dev_out, void *ws, size_t ws_bytes,
                                 void *stream) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    Plan P;
    drt3d_status s = make_plan(transform, N, mask, o, P);
    if (s != DRT3D_OK) return s;
    if (!host_cube || !host_out) return DRT3D_ERR_INVALID_ARG;
    s = check_ptrs(dev_cube, dev_out, ws, ws_bytes, P, o, transform);
    if (s != DRT3D_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t cb = (size_t)P.batch * N * N * N * in_bytes(o.in_dtype);
    const size_t ob = out_elems(transform, P, o) * 4;
    if (cudaMemcpyAsync(dev_cube, host_cube, cb, cudaMemcpyHostToDevice, st) != cudaSuccess) return DRT3D_ERR_CUDA;
    // One cube, stacked layout, several dodecants: transform them in groups and copy each group's
    // output slice to the host on a copy stream while the next group computes (the result's
    // device-to-host copy is PCIe-bound, ~57 GB/s; this hides the transform behind it).
    AuxLease lease(P.batch == 1 && o.layout == DRT3D_LAYOUT_STACKED && P.ndod >= 2 && !o.events);
    Aux *ax = lease.get();
    if (ax) {
        JoinGuard join{st, ax->cp, ax->cpdone};      // the caller's stream resumes after the last copy
        const int K = P.ndod, G = K < kHostGroups ? K : kHostGroups;
        const size_t per_dod = ob / (size_t)K;
        int kl[12], nk = 0;
        for (int k = 0; k < 12; ++k)
            if ((mask >> k) & 1) kl[nk++] = k;
        int j0 = 0, launches = 0;
        for (int g = 0; g < G; ++g) {
            const int d = K / G + (g < K % G ? 1 : 0);
            uint32_t mg = 0;
            for (int j = j0; j < j0 + d; ++j) mg |= 1u << kl[j];
            Plan Pg;
            s = make_plan(transform, N, mg, o, Pg);
            if (s != DRT3D_OK) return s;
            if (Pg.ws_bytes > ws_bytes) return DRT3D_ERR_WORKSPACE;      // cannot happen: fewer instances
            unsigned char *og = reinterpret_cast<unsigned char *>(dev_out) + per_dod * j0;
            s = transform == 0 ? run_drt(dev_cube, mg, og, o, Pg, ws, st) : run_djt(dev_cube, mg, og, o, Pg, ws, st);
            if (s != DRT3D_OK) return s;
            if (o.launches) launches += *o.launches;
            if (cudaEventRecord(ax->gdone[g], st) != cudaSuccess) return DRT3D_ERR_CUDA;
            if (cudaStreamWaitEvent(ax->cp, ax->gdone[g], 0) != cudaSuccess) return DRT3D_ERR_CUDA;
            if (cudaMemcpyAsync(reinterpret_cast<unsigned char *>(host_out) + per_dod * j0, og, per_dod * d,
                                cudaMemcpyDeviceToHost, ax->cp) != cudaSuccess)
                return DRT3D_ERR_CUDA;
            j0 += d;
        }
        if (o.launches) *o.launches = launches;
        return DRT3D_OK;
    }
    s = transform == 0 ? run_drt(dev_cube, mask, dev_out, o, P, ws, st) : run_djt(dev_cube, mask, dev_out, o, P, ws, st);
    if (s != DRT3D_OK) return s;
    if (cudaMemcpyAsync(host_out, dev_out, ob, cudaMemcpyDeviceToHost, st) != cudaSuccess) return DRT3D_ERR_CUDA;
    return DRT3D_OK;
}

drt3d_status drt3d_planes_host(const void *host_cube, int N, uint32_t mask, void *host_out, const drt3d_opts *opts,
                               void *dev_cube, void *dev_out, void *ws, size_t ws_bytes, void *stream) {
    return host_variant(0, host_cube, N, mask, host_out, opts, dev_cube, dev_out, ws, ws_bytes, stream);
}

drt3d_status djt3d_lines_host(const void *host_cube, int N, uint32_t mask, void *host_out, const drt3d_opts *opts,
                              void *dev_cube, void *dev_out, void *ws, size_t ws_bytes, void *stream) {
    return host_variant(1, host_cube, N, mask, host_out, opts, dev_cube, dev_out, ws, ws_bytes, stream);
}

}  // extern "C"

namespace d3 {
// Internal entry (C++ linkage, not part of the C ABI): r <- r - A f for an fp32 cube, stacked
// layout, enqueued on `stream`.  The final pass adds -A f into r with a TMA reduce-add per output
// tile (its all-zero tiles add nothing), so the residual update of the inverse (invert.cu) needs no
// separate elementwise pass over A f.  DRT3D_ERR_UNSUPPORTED, with nothing enqueued, for plans
// without that final pass (N < 64: the on-chip kernels, the tiny single passes).
drt3d_status planes_residual(const void *cube, int N, uint32_t mask, float *r, const drt3d_opts *opts,
                             void *workspace, size_t workspace_bytes, void *stream) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    if (o.in_dtype != DRT3D_F32 || o.out_dtype != DRT3D_F32 || o.layout != DRT3D_LAYOUT_STACKED || N < 64)
        return DRT3D_ERR_UNSUPPORTED;
    Plan P;
    drt3d_status s = make_plan(0, N, mask, o, P);
    if (s != DRT3D_OK) return s;
    if (P.small) return DRT3D_ERR_UNSUPPORTED;
    s = check_ptrs(cube, r, workspace, workspace_bytes, P, o, 0);
    if (s != DRT3D_OK) return s;
    return run_drt(cube, mask, r, o, P, workspace, reinterpret_cast<cudaStream_t>(stream), true);
}

// Internal entry: out = A f (fp32, stacked) and, fused into the final pass, per-CTA sums of out^2 in
// fp64 at sq_part[0 .. *sq_count) (the count is written by the kernel; at most
// planes_sumsq_parts(N, batch x dodecants) entries).  DRT3D_ERR_UNSUPPORTED, nothing enqueued, as for
// planes_residual.
size_t planes_sumsq_parts(int N, int instances) {
    // final passes with K >= 2: groups x tiles <= N^2 / 16 x 3N / 96 (the smallest group and tile)
    return (size_t)instances * N * N / 16 * ((3 * (size_t)N + 95) / 96) + 1;
}
drt3d_status planes_sumsq(const void *cube, int N, uint32_t mask, float *out, const drt3d_opts *opts,
                          void *workspace, size_t workspace_bytes, void *stream, double *sq_part, int *sq_count) {
    drt3d_opts tmp;
    const drt3d_opts &o = opts_or_default(opts, tmp);
    if (o.in_dtype != DRT3D_F32 || o.out_dtype != DRT3D_F32 || o.layout != DRT3D_LAYOUT_STACKED || N < 64 || !sq_part ||
        !sq_count)
        return DRT3D_ERR_UNSUPPORTED;
    Plan P;
    drt3d_status s = make_plan(0, N, mask, o, P);
    if (s != DRT3D_OK) return s;
    if (P.small) return DRT3D_ERR_UNSUPPORTED;
    s = check_ptrs(cube, out, workspace, workspace_bytes, P, o, 0);
    if (s != DRT3D_OK) return s;
    return run_drt(cube, mask, out, o, P, workspace, reinterpret_cast<cudaStream_t>(stream), false, sq_part, sq_count);
}
}  // namespace d3
