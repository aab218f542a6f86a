/*
 * wect.h -- C ABI of libwect.so, the B200 (sm_100a) hot path of arXiv 2511.03909
 * ("Vectorized Computation of Euler Characteristic Functions and Transforms").
 *
 * Citation keys: P:a-b = lines of the paper text, with the section /
 * equation / algorithm named.  Readings A1..A12 are listed in DESIGN.md.
 *
 * What every entry point computes (Algorithm 1 "ComputeWECFs", and
 * its closed form P:769-776):
 *
 *     out[p, q] = sum over cells s of K with  max_{v in s} f_p(v) <= beta(q)
 *                 of (-1)^{dim s} * w(s)
 *
 *   with beta(q) = lo + q (hi - lo) / (T - 1)
 *   and, by default, lo = -M, hi = M, M = max_{p, v} |f_p(v)|.
 *   The height grid is applied through alpha (eq. left-adjoint):
 *       alpha(t) = clamp(ceil(((T-1) * (t - lo)) / (hi - lo)), 0, T-1),
 *   evaluated so that every bin equals the IEEE binary64 evaluation of that
 *   expression in the order written (reading A1).  The WECT uses the height
 *   filters f_p(v) = <l(v), s_p> (Example "wect" P:778-794),
 *   summed in axis order in binary64.  The ECF uses the caller's filter values.
 *
 * Conventions shared by all calls
 *   - Pointers: every array pointer may be CUDA device memory or host memory
 *     (pageable or pinned); the library detects which.  Host inputs are staged
 *     to the device and host outputs are copied back inside the call; a call
 *     with any host array synchronises the stream before returning, so host
 *     buffers may be reused at once.  Device-only calls are asynchronous on
 *     `stream` (device inputs must stay untouched until the stream completes).
 *   - Ownership: the caller owns every array.  The library keeps no pointer
 *     after the call's stream work completes; it allocates its scratch with
 *     cudaMallocAsync on `stream` and frees it stream-ordered.
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Output is fully overwritten, never accumulated.  Layout row-major.
 *   - Errors: argument/shape errors return synchronously BEFORE anything is
 *     enqueued (WECT_EINVAL / WECT_EOVERFLOW / WECT_ENOTSUP).  An out-of-range
 *     vertex index found by a kernel sets a per-device error word and the cell
 *     is skipped; wect_sync_status() reports it as WECT_ERANGE (output then
 *     unspecified).  With WECT_VALIDATE the indices are checked synchronously
 *     first and WECT_ERANGE is returned with nothing written.
 *   - wect_last_error() returns a thread-local message for the last failure.
 *   - Reentrant; distinct calls may run concurrently on distinct streams.  The
 *     deferred-error word (WECT_ERANGE) and the repair counter are PER DEVICE,
 *     not per call: with concurrent calls on one device, wect_sync_status() on
 *     one stream can report an out-of-range index found by another call.
 */
#ifndef WECT_H_
#define WECT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WECT_ABI_VERSION 1

#if defined(__GNUC__)
#define WECT_API __attribute__((visibility("default")))
#else
#define WECT_API
#endif

typedef enum {
  WECT_OK = 0,
  WECT_EINVAL = -1,    /* bad argument or shape */
  WECT_ERANGE = -2,    /* vertex index outside [0, k0) */
  WECT_EOVERFLOW = -3, /* requested output dtype cannot hold the result */
  WECT_ECUDA = -4,     /* CUDA runtime error (message in wect_last_error) */
  WECT_ENOMEM = -5,    /* device allocation failed */
  WECT_ENOTSUP = -6    /* valid request this build does not support */
} wect_status;

typedef enum { WECT_U8 = 1, WECT_I32 = 2, WECT_I64 = 3, WECT_F32 = 4, WECT_F64 = 5 } wect_dtype;

/* flags for wect_grid.flags */
#define WECT_VALIDATE 1u   /* synchronous index pre-check before any write */
#define WECT_FP32_ONLY 2u  /* skip the binary64 near-edge repair (experiments only; bins may then
                              differ from reading A1 for heights within rounding of a bin edge) */
#define WECT_TIME_MAIN 4u  /* instrumentation: record CUDA events around the call's dominant kernel on
                              `stream` (read with wect_stats); adds no synchronisation */
#define WECT_FREUDENTHAL 8u /* wect_images, ndim = 2 only: the image as a weighted Freudenthal complex
                               instead of a cubical one -- horizontal, vertical
                              and (r,c)-(r+1,c+1) diagonal edges, two triangles per unit square, each
                              simplex weighted by the max of its vertices, sign (-1)^dim */

/* One dimension i >= 1 of K: the pair (i-SimplexVertices, i-SimplexWeights) of the
 * Complex list.  verts: [count, arity] int32 row-major, values in [0, k0).
 * arity = i+1 for simplices, 2^i for cubes ("cubical complexes with no
 * modifications").  weights: [count] of the complex's weight dtype, or NULL for unit
 * weights (the EC).  count == 0 skips the dimension.  sign = (-1)^dim. */
typedef struct {
  const int32_t* verts;
  const void* weights;
  int64_t count;
  int32_t arity; /* 1..32 */
  int32_t dim;   /* >= 1 */
} wect_cells;

/* The Complex of Algorithm 1 plus vertex coordinates (Example "wect").
 * coords: [k0, n] fp32 vertex embedding l(v) (unused by ecf_complex, may be NULL there).
 * vweights: [k0] VertexWeights or NULL (unit).  cells: HOST array of ncell_dims
 * descriptors.  wdtype: WECT_I32 (integer weights, exact int64 accumulation) or
 * WECT_F32 (float weights, fp32 shared-memory partials merged in binary64, reading A8). */
typedef struct {
  const float* coords;
  int64_t k0;
  int32_t n; /* ambient dimension, 1..8 */
  const void* vweights;
  const wect_cells* cells;
  int32_t ncell_dims;
  wect_dtype wdtype;
} wect_complex_desc;

/* The discretisation grid and the row range to compute.
 * T = numvals >= 2 (beta divides by T-1).
 * d_begin, d_count: compute output rows [d_begin, d_begin + d_count) of the full filter
 *   set; d_count == 0 means all rows from d_begin.  M is ALWAYS taken over the full set
 *   (reading A2), so row-sharded calls agree with an unsharded call bit for bit.
 * maxheight > 0: use it as M (a shared grid across inputs); <= 0: compute M.
 * lo < hi: use the explicit grid [lo, hi] instead of [-M, M] (reading A9); otherwise ignored.
 * flags: WECT_VALIDATE | WECT_FP32_ONLY. */
typedef struct {
  int32_t T;
  int32_t d_begin;
  int32_t d_count;
  double maxheight;
  double lo;
  double hi;
  uint32_t flags;
} wect_grid;

/* WECT of an explicit weighted complex (P:351-362 Def. wect; Alg. 1 with FVals = V D^T,
 * P:778-794).  dirs: [D, n] fp32 directions s_p (need not be unit).  out: [d_count, T]
 * of odtype: WECT_I64 for integer weights (WECT_I32 is refused: no bound), WECT_F64 for
 * float weights. */
WECT_API wect_status wect_complex(const wect_complex_desc* K, const float* dirs, int32_t D, const wect_grid* grid,
                         void* out, wect_dtype odtype, void* stream);

/* WECT of a batch of uint8 images (ndim = 2, dims = {H, W}) or voxel volumes (ndim = 3,
 * dims = {Z, Y, X}) as weighted cubical complexes (P:213-215, P:273-289 pipeline (ii)).
 * Pixels are vertices; every axis-aligned unit i-cube of the grid is a cell of sign
 * (-1)^i (reading A7) with weight = max of its corner intensities (reading A5);
 * vertex weight = intensity.  Vertex l(v) per reading A3: grid index g on an axis of
 * length L maps to (g - (L-1)/2) / max(max_dim - 1, 1) (binary64, rounded once to fp32);
 * column -> axis 0, row -> axis 1, slice -> axis 2.  No cell lists touch memory.
 * img: [B, dims...] uint8.  dims: HOST array.  dirs: [D, ndim] fp32.
 * out: [B, d_count, T] of WECT_I32 (refused with WECT_EOVERFLOW when
 * 255 * #cells >= 2^31) or WECT_I64.
 * grid->flags & WECT_FREUDENTHAL (ndim = 2): the Freudenthal triangulation of each image
 * instead (same vertices and coordinates, same M; every simplex binned exactly). */
WECT_API wect_status wect_images(const uint8_t* img, int64_t B, int32_t ndim, const int64_t* dims, const float* dirs,
                        int32_t D, const wect_grid* grid, void* out, wect_dtype odtype, void* stream);

/* WECFs of a weighted complex for m given vertex filters (Algorithm 1 verbatim,
 * P:654-687; with unit weights the ECF).  fvals: [k0, m] fp32,
 * FVals[a, p] = f_p(v_a).  K->coords is not used.  out: [d_count, T]. */
WECT_API wect_status ecf_complex(const wect_complex_desc* K, const float* fvals, int32_t m, const wect_grid* grid,
                        void* out, wect_dtype odtype, void* stream);

/* ECF of a batch of uint8 images (ndim = 2, dims = {H, W}) or voxel volumes (ndim = 3,
 * dims = {Z, Y, X}): Remark "which-ecf" -- the pixel intensities are the
 * vertex filter and each entry is the unweighted Euler characteristic of the lower-star
 * filtration of the image's cubical V-construction (every unit
 * i-cube a cell of sign (-1)^i, reading A7; a cell's filter value = max of its corners).
 * This is Algorithm 1 with m = 1 and unit weights, each image its own complex:
 *     out[b, q] = sum over cells s of image b with max_{v in s} img_b(v) <= beta_b(q) of (-1)^dim s.
 * Grid (reading A9), in priority order:
 *   grid->lo < grid->hi  -> the same grid [lo, hi] for every image (e.g. [0, 255] with
 *                           T = 256: beta(q) = q, one bin per intensity);
 *   grid->maxheight > 0  -> [-maxheight, maxheight] for every image;
 *   otherwise            -> the paper's grid [-M_b, M_b], M_b = max intensity of image b
 *                           (M_b = 0 puts every cell in bin 0, reading A6).
 * Bins equal the binary64 evaluation of alpha (reading A1), so results are exact integers.
 * img: [B, dims...] uint8.  dims: HOST array.  grid->d_begin must be 0 and grid->d_count
 * 0 or 1 (one filter per image); flags other than WECT_TIME_MAIN are ignored.
 * out: [B, T] of WECT_I32 (refused with WECT_EOVERFLOW when #cells >= 2^31) or WECT_I64.
 * T in [2, 65536]; image sides <= 65535; B <= 65535 for images of more than 4096 pixels
 * (WECT_ENOTSUP otherwise).  Errors as for wect_images. */
WECT_API wect_status ecf_images(const uint8_t* img, int64_t B, int32_t ndim, const int64_t* dims,
                                const wect_grid* grid, void* out, wect_dtype odtype, void* stream);

/* Gradient of a scalar loss L with respect to the weights, through wect_complex /
 * ecf_complex (the paper's differentiability claim).
 * Alg. 1 is linear in the weights (closed form P:769-776), so with G = dL/dout,
 *     dL/dw(s) = (-1)^dim s * sum_p sum_{q >= bin(s, p)} G[p, q]
 * where bin(s, p) is the forward's cell bin (max of its vertices' alpha, eq. msi P:713-723,
 * evaluated exactly per reading A1).  Coordinates / filter values receive no gradient
 * (the output is piecewise constant in them).
 * K, dirs / fvals, D / m, grid: exactly as for the forward call (M over ALL rows, A2);
 *   K->wdtype and the weight arrays are not read.
 * G: [d_count, T] fp64, the rows d_begin .. d_begin + d_count of dL/dout.
 * grad_vweights: [k0] fp64 output or NULL (skip).
 * grad_cells: HOST array of K->ncell_dims pointers (or NULL), entry i an [cells[i].count] fp64
 *   output or NULL (skip).  Outputs are overwritten.  Cells of arity > 8: WECT_ENOTSUP.
 * Accumulation: RC = reverse cumsum of each G row in binary64 from q = T-1 down, then the
 *   sum over rows in a fixed order (tiles of 32 rows, or 64 when T <= 320; a shuffle tree
 *   within a tile):
 *   deterministic, within binary64 rounding of the exact sum (reading A13).
 * Errors as for wect_complex; an out-of-range vertex index is reported by wect_sync_status. */
WECT_API wect_status wect_complex_backward(const wect_complex_desc* K, const float* dirs, int32_t D,
                                           const wect_grid* grid, const double* G, double* grad_vweights,
                                           double* const* grad_cells, void* stream);
WECT_API wect_status ecf_complex_backward(const wect_complex_desc* K, const float* fvals, int32_t m,
                                          const wect_grid* grid, const double* G, double* grad_vweights,
                                          double* const* grad_cells, void* stream);

/* M = max_{p, v} |<l(v), s_p>| over all k0 vertices and all D directions, in binary64
 * (P:624-628), the value wect_complex uses when grid->maxheight <= 0.  Synchronous
 * (writes *M_host).  For direction-sharded runs each rank may call this and the
 * results agree exactly. */
WECT_API wect_status wect_maxheight(const float* coords, int64_t k0, int32_t n, const float* dirs, int32_t D,
                           double* M_host, void* stream);

/* Synchronises `stream` and returns WECT_ERANGE if any kernel since the last call
 * recorded an out-of-range vertex index on this device (and clears the word),
 * WECT_ECUDA on a CUDA error, WECT_OK otherwise. */
WECT_API wect_status wect_sync_status(void* stream);

/* Thread-local description of the last error ("" if none). */
WECT_API const char* wect_last_error(void);

/* Counters of the binary64 near-edge repairs since the last reset (reading A1:
 * "near-edge cases, counted and reported").  Reads synchronously. */
WECT_API wect_status wect_repair_count(uint64_t* count_host, int reset);

/* Instrumentation: *launches = kernels this library launched since the last reset;
 * *timed_launches / *timed_ms = count and summed device time of the dominant-kernel launches
 * recorded under WECT_TIME_MAIN (synchronises on their events).  reset != 0 clears all. */
WECT_API wect_status wect_stats(uint64_t* launches, uint64_t* timed_launches, double* timed_ms, int reset);

WECT_API int32_t wect_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WECT_H_ */
