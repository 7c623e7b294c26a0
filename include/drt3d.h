/*
 * drt3d.h -- C ABI of the B200 (sm_100a) library for the forward hot path of
 * arXiv 2501.13664 (Marichal-Hernandez et al., "Multiscale 3D discrete Radon
 * transform of planes and discrete John transform of lines").
 *
 * Citations are /root/reference/PAPER.md line numbers with the section,
 * equation label or algorithm they fall in.
 *
 * Common rules for every entry point
 * ----------------------------------
 *  - All data pointers (`cube`, `out`, `workspace`) are DEVICE pointers unless
 *    the function name ends in `_host`.  The caller owns every buffer; the
 *    library never allocates device memory, frees, or synchronises, and enqueues
 *    its kernels on `stream` (a cudaStream_t passed as void*, NULL = legacy
 *    default stream).  Multi-chunk DRT calls may also run passes on an internal
 *    auxiliary stream, and the `_host` calls copy finished dodecant groups to the
 *    host on an internal copy stream (both one per host thread and device,
 *    created on first use); each is forked from and joined back into `stream`
 *    within the call, so ordering with respect to `stream` is unchanged.  The
 *    inverse captures one iteration as a CUDA graph on an internal stream and
 *    replays it on `stream` (graphs cached per device, shapes and buffers).
 *  - N must be a power of two, 2 <= N <= 1024 (non-cubic / non-dyadic volumes are
 *    out of scope).
 *  - cube layout: C order [batch][x][y][z], z fastest; element type opts->in_dtype.
 *  - Validation happens synchronously before any launch; on error nothing is
 *    written and no kernel is enqueued.  Launch failures return
 *    DRT3D_ERR_CUDA; asynchronous faults surface at the caller's next sync.
 *  - Results are deterministic and bit-identical across runs.
 *  - opts may be NULL: {batch=1, U8 -> I32, STACKED, HEMISPHERE}.
 */
#ifndef DRT3D_H
#define DRT3D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DRT3D_OK = 0,
    DRT3D_ERR_INVALID_ARG = 1,   /* bad N, mask, pointer, dtype pair, alignment */
    DRT3D_ERR_UNSUPPORTED = 2,   /* valid request this build does not implement */
    DRT3D_ERR_WORKSPACE = 3,     /* workspace NULL or smaller than queried     */
    DRT3D_ERR_CUDA = 4           /* a CUDA launch/attribute call failed         */
} drt3d_status;

typedef enum { DRT3D_U8 = 0, DRT3D_I32 = 1, DRT3D_F32 = 2 } drt3d_dtype;

typedef enum {
    DRT3D_LAYOUT_STACKED = 0,    /* out[batch][j][s1][s2][D]  (j = rank of dodecant in mask) */
    DRT3D_LAYOUT_MOSAIC = 1      /* DRT only, mask 0xFFF: out[batch][4N][4N][3N-2], Alg. 2  */
} drt3d_layout;

typedef enum {
    DRT3D_TABLE_HEMISPHERE = 0,  /* DRT: printed InOrder with rows 5, 9 repaired; DJT: complete
                                    identity-anchored line table (R7, R8)          */
    DRT3D_TABLE_PRINTED = 1,     /* InOrder of Alg. 2 verbatim, both      */
    DRT3D_TABLE_SHARED = 2       /* one table complete for planes and lines (R8)   */
} drt3d_table;

typedef struct {
    int batch;        /* number of independent cubes, >= 1                        */
    int in_dtype;     /* drt3d_dtype of cube: U8, I32 or F32                      */
    int out_dtype;    /* I32 for U8/I32 input (exact sum mod 2^32), F32 for F32   */
    int layout;       /* drt3d_layout                                             */
    int table;        /* drt3d_table                                              */
    /* Optional instrumentation (NULL = off).  When `events` is non-NULL it points
     * to 2*max_events cudaEvent_t handles; the library records events[2i] and
     * events[2i+1] around its i-th kernel launch on `stream` (i < max_events).
     * When `launches` is non-NULL the number of kernels enqueued is written.
     * `launch_kind` (optional, max_events entries) receives the pass kind of
     * each launch: 0 = first pass, 1 = middle pass, 2 = final pass, 3 = fill. */
    void **events;
    int max_events;
    int *launches;
    int *launch_kind;
} drt3d_opts;

/* Human-readable name of a status code (static string). */
const char *drt3d_status_string(drt3d_status s);

/* Orientation table rows used for `table` and `transform` (0 = DRT, 1 = DJT):
 * rows[3k + j] = signed 1-based axis p_j of dodecant k (reading A: oriented
 * axis j is original axis |p_j|, reversed when p_j < 0; Alg. 2). */
drt3d_status drt3d_orientation_table(int table, int transform, int8_t rows[36]);

/* ---------------------------------------------------------------- planes --
 * 3D DRT of planes over the dodecants set in dodecant_mask (bit k = dodecant k,
 * 1 <= mask < 2^12), Alg. 1 per dodecant, Alg. 2 dodecant
 * loop with the orientation applied as an index remap.
 * Definition eq:3DfDRT:
 *   out(s1, s2, D) = sum_{x,y} f_k(x, y, l_{s1}(x) + l_{s2}(y) + D - 2N),
 * s1, s2 in [0, N), D in [0, 3N) (D = 0, 1 and D < 2N - s1 - s2 are 0).
 * STACKED output: [batch][popcount(mask)][N][N][3N] of out_dtype.
 * MOSAIC output (mask must be 0xFFF): [batch][4N][4N][3N-2], block
 * DodecantCoords[k] holds dodecant k with OutOrder[k] applied to (s1, s2) by
 * reading A, d = D - 2; 4 unused blocks are 0.  OutOrder rows 0-3 are the
 * repaired rows (-1,-2,3), (-2,1,3), (1,2,3), (2,-1,3) of DESIGN.md reading
 * R13: with them, and only them, the boundary planes neighbouring dodecants
 * share lie on facing block edges ("rotated so that all of them fit
 * accurately", fig:shapeOutput; HEMISPHERE table).
 * Workspace: drt3d_planes_workspace_size() bytes (device, 256-byte aligned);
 * 0 for N = 16 and N = 32 in the STACKED layout (every stage on chip), where
 * workspace may be NULL.                                                      */
size_t drt3d_planes_out_elems(int N, uint32_t dodecant_mask, const drt3d_opts *opts);
drt3d_status drt3d_planes_workspace_size(int N, uint32_t dodecant_mask, const drt3d_opts *opts,
                                         size_t *bytes);
drt3d_status drt3d_planes(const void *cube, int N, uint32_t dodecant_mask, void *out,
                          const drt3d_opts *opts, void *workspace, size_t workspace_bytes,
                          void *stream);

/* ----------------------------------------------------------------- lines --
 * 3D DJT of lines, Alg. 3 per dodecant; the dodecants of
 * dodecant_mask use the DJT orientation table.  Definition
 * eq:3DfDJT:
 *   out(s1, s2, D1, D2) = sum_u f_k(u, l_{s1}(u) + D1 - N, l_{s2}(u) + D2 - N),
 * Di in [0, 2N).  Output [batch][popcount(mask)][N][N][2N][2N] (STACKED only;
 * the paper defines no DJT mosaic).                             */
size_t djt3d_lines_out_elems(int N, uint32_t dodecant_mask, const drt3d_opts *opts);
drt3d_status djt3d_lines_workspace_size(int N, uint32_t dodecant_mask, const drt3d_opts *opts,
                                        size_t *bytes);
drt3d_status djt3d_lines(const void *cube, int N, uint32_t dodecant_mask, void *out,
                         const drt3d_opts *opts, void *workspace, size_t workspace_bytes,
                         void *stream);

/* ------------------------------------------------------------- adjoints --
 * Backprojection = the transpose of the transforms above:
 * eq:invmap3Dsummation / eq:invmap3DJsummation
 * run in reversed stage order, then the
 * transposes of the seeding step and of the dodecant orientation.
 *   cube(c) = sum_{k in mask} sum_{s1,s2,D} coef_k(s1,s2,D) [c on plane (s1,s2,D) of k]
 * (lines likewise), i.e. <A f, coef> = <f, A^T coef> for every f.
 * coef: the stacked output layout of the forward call ([batch][K][N][N][3N] for
 * planes, [batch][K][N][N][2N][2N] for lines) with element type opts->out_dtype
 * (I32: exact sums mod 2^32; F32: fp32 accumulation); cube: [batch][N][N][N]
 * of the same element type (opts->in_dtype is ignored).  STACKED layout only.
 * coef and cube must be 16-byte aligned, the workspace 256-byte aligned
 * (DRT3D_ERR_INVALID_ARG / DRT3D_ERR_WORKSPACE otherwise).
 * Workspace: query the size (it depends on N and on the number of dodecants:
 * the DRT runs the dodecants of a chunk together, up to 4 GB of level
 * buffers -- all 12 at N = 256, 1.7 GB).                                     */
drt3d_status drt3d_planes_adjoint_workspace_size(int N, uint32_t dodecant_mask, const drt3d_opts *opts,
                                                 size_t *bytes);
drt3d_status drt3d_planes_adjoint(const void *coef, int N, uint32_t dodecant_mask, void *cube,
                                  const drt3d_opts *opts, void *workspace, size_t workspace_bytes,
                                  void *stream);
drt3d_status djt3d_lines_adjoint_workspace_size(int N, uint32_t dodecant_mask, const drt3d_opts *opts,
                                                size_t *bytes);
drt3d_status djt3d_lines_adjoint(const void *coef, int N, uint32_t dodecant_mask, void *cube,
                                 const drt3d_opts *opts, void *workspace, size_t workspace_bytes,
                                 void *stream);

/* ---------------------------------------------------- iterative inverse --
 * Iterative inverse of the 3D DRT: Press's
 * iterative improvement x <- x + B (b - A x), x_0 = 0, where B is the multigrid
 * approximate inverse built from the 3D high-pass filter h,
 * the prolongation P and the restriction S.  Readings
 * (R15-R18): at size n, B r = e + alpha h*(A^T (r - A e)) with
 * e = P B_{n/2}(S r) and alpha = <r', A p> / <A p, A p> (r' the remainder, p the
 * filtered backprojection: the residual-minimising step); at n = n_min,
 * B r = alpha h*(A^T r).  h uses zero padding.  n_min = N is the single-grid
 * iteration x <- x + alpha h*(A^T r).
 * coef: [K][N][N][3N] fp32 device (the stacked forward layout, K = popcount
 * of the mask); n_min: coarsest grid, a power of two in [2, N]; cube: [N][N][N]
 * fp32 device, receives x_iters; rnorm: NULL or a device array of iters+1
 * doubles receiving ||b - A x_k||_2, k = 0..iters.
 * opts: NULL or batch = 1, out_dtype = F32, STACKED (in_dtype ignored).
 * Workspace: per level n = N, N/2, .., n_min three coefficient-sized and three
 * cube-sized fp32 buffers, plus the larger of the size-N forward / adjoint
 * workspaces (query the size; 256-byte aligned).
 * Enqueue only: every iteration runs on `stream` with no host synchronisation
 * (the step sizes live in the workspace).
 * Errors: DRT3D_ERR_INVALID_ARG (N, n_min, mask, opts, NULL or not 16-byte
 * aligned coef / cube, iters < 0), DRT3D_ERR_WORKSPACE, DRT3D_ERR_CUDA.      */
drt3d_status drt3d_planes_invert_workspace_size(int N, int n_min, uint32_t dodecant_mask,
                                                const drt3d_opts *opts, size_t *bytes);
drt3d_status drt3d_planes_invert(const void *coef, int N, int n_min, uint32_t dodecant_mask, int iters,
                                 void *cube, double *rnorm, const drt3d_opts *opts, void *workspace,
                                 size_t workspace_bytes, void *stream);

/* --------------------------------------------------------- applications --
 * SURVEY §8(f) F-4, on int32 coefficient arrays in device memory (any layout
 * for argmax / threshold; the stacked DRT layout [K][N][N][3N] for planes).
 * Workspace: drt3d_apps_workspace_size() bytes, 256-byte aligned, device.
 * All enqueue on `stream`; results are deterministic (fixed-order reductions).
 *
 * drt3d_coef_argmax: *index (device int64) = flat index of the largest
 *   coefficient, the smallest index among ties (R20).
 * drt3d_coef_threshold: out[i] = coef[i] if coef[i] * den >= num * max(coef)
 *   else 0, tested exactly in int64 (R19; "a thresholding of the
 *   highest amplitude coefficients, and subsequent backprojection"); out may
 *   alias coef.  num >= 0, den > 0.
 * drt3d_detect_planes: flags[i] (device uint8, same shape
 *   as coef) = 1 for the argmax plane and for every coefficient that passes
 *   the R19 threshold, is a relative maximum of its dodecant's (s1, s2, D)
 *   26-neighbourhood (R21) and whose plane is orthogonal to the argmax plane,
 *   |cos| <= onum/oden, with integer normals through the orientation table
 *   opts->table (R22); *argmax (device int64, may be NULL) receives R20's index.
 * drt3d_coef_select: out[i] = flags[i] ? coef[i] : 0 (no workspace): with
 *   drt3d_planes_adjoint it back-projects the detected planes ("When those
 *   planes are backprojected, they correspond to the walls").
 * Errors: DRT3D_ERR_INVALID_ARG (NULL pointers, n = 0, N, mask, num < 0,
 *   den <= 0, onum < 0, oden <= 0), DRT3D_ERR_WORKSPACE, DRT3D_ERR_CUDA.      */
size_t drt3d_apps_workspace_size(void);
drt3d_status drt3d_coef_argmax(const int32_t *coef, size_t n, long long *index, void *workspace,
                               size_t workspace_bytes, void *stream);
drt3d_status drt3d_coef_threshold(const int32_t *coef, size_t n, int num, int den, int32_t *out,
                                  void *workspace, size_t workspace_bytes, void *stream);
drt3d_status drt3d_coef_select(const int32_t *coef, const uint8_t *flags, size_t n, int32_t *out,
                               void *stream);
drt3d_status drt3d_detect_planes(const int32_t *coef, int N, uint32_t dodecant_mask, int num, int den,
                                 int onum, int oden, const drt3d_opts *opts, uint8_t *flags,
                                 long long *argmax, void *workspace, size_t workspace_bytes, void *stream);

/* --------------------------------------------------------- host buffers --
 * End-to-end variants: `host_cube` and `host_out` are HOST pointers (pinned
 * for full speed); `dev_cube` (>= cube bytes), `dev_out` (>= out bytes) and
 * `workspace` are caller-provided device scratch.  Copies the cube in, runs
 * the transform, copies the result out, all on `stream`; returns after
 * enqueueing (synchronise the stream before reading host_out).               */
drt3d_status drt3d_planes_host(const void *host_cube, int N, uint32_t dodecant_mask, void *host_out,
                               const drt3d_opts *opts, void *dev_cube, void *dev_out,
                               void *workspace, size_t workspace_bytes, void *stream);
drt3d_status djt3d_lines_host(const void *host_cube, int N, uint32_t dodecant_mask, void *host_out,
                              const drt3d_opts *opts, void *dev_cube, void *dev_out,
                              void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DRT3D_H */
