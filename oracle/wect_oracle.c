/*
 * wect_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the WECT / WECF hot path of
 * arXiv 2511.03909 ("Vectorized Computation of Euler Characteristic Functions
 * and Transforms").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA path in
 * paper_2511_03909_b200/ and never includes include/wect.h.
 *
 * Citation keys: P:a-b = /root/reference/PAPER.md lines a-b (section/equation
 * named beside each).  Readings of the paper that are not fixed by the text are
 * the ones listed in DESIGN.md "Readings" (A1..A12).
 *
 * Arithmetic: IEEE binary64, built with -O2 -ffp-contract=off so that every
 * product and sum below is rounded exactly as written (A1).
 *
 * Arms:
 *   O1  orc_wecfs_naive   -- the naive discretised WECT: for every
 *                            filter p and height beta(q), enumerate the
 *                            sublevel complex and sum (-1)^dim * w directly.
 *   O2  orc_wecfs_alg1    -- Algorithm 1 ComputeWECFs, step by step:
 *                            VIndices = alpha(FVals); scatter_add; per
 *                            dimension gather + rmax + signed scatter_add;
 *                            cumsum.  OpenMP over filters p only.
 *   plus the builders the tests need: FVals = V * D^T and the
 *   explicit cubical complex of an image / voxel volume (P:213-215,
 *   P:273-289; readings A3, A5, A7).
 *
 * Parity pins for every function live in tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Example "wect": FVals = V * D^T, (V*D^T)[a,p] = h_{s_p}(v_a)   */
/* with h_s(v) = l(v) . s.  Summed in axis order i = 0..n-1;    */
/* each product of two fp32 values is exact in binary64.                     */
/* ------------------------------------------------------------------------ */
ORC_API void orc_heights(const float* coords, int64_t k0, int32_t n,
                         const float* dirs, int32_t D, double* fvals /* [k0, D] */) {
  for (int64_t a = 0; a < k0; ++a) {
    for (int32_t p = 0; p < D; ++p) {
      double h = 0.0;
      for (int32_t i = 0; i < n; ++i) {
        double prod = (double)coords[a * n + i] * (double)dirs[p * n + i];
        h = (i == 0) ? prod : h + prod;
      }
      fvals[a * D + p] = h;
    }
  }
}

/* maxheight = max_{p, v} |f_p(v)| over ALL filters and vertices. */
ORC_API double orc_maxheight(const double* fvals, int64_t k0, int32_t m) {
  double M = 0.0;
  for (int64_t i = 0; i < k0 * (int64_t)m; ++i) {
    double a = fabs(fvals[i]);
    if (a > M) M = a;
  }
  return M;
}

/* alpha(t) = ceil((numvals-1)(maxheight + t) / (2 maxheight))  (eq. left-adjoint,
 * P:637-645), written for a general grid [lo, hi] as
 *     u = ((T-1) * (t - lo)) / (hi - lo),  alpha = clamp(ceil(u), 0, T-1).
 * With lo = -M, hi = M this is the paper's expression operation for operation:
 * t - (-M) rounds exactly like M + t, and M - (-M) = 2M exactly.
 * Degenerate grid hi == lo (maxheight = 0): every value goes to index 0 (A6). */
ORC_API int32_t orc_alpha(double t, double lo, double hi, int32_t T) {
  if (!(hi > lo)) return 0;
  double u = ((double)(T - 1) * (t - lo)) / (hi - lo);
  double c = ceil(u);
  if (c < 0.0) return 0;
  if (c > (double)(T - 1)) return T - 1;
  return (int32_t)c;
}

/* beta(q) = q * 2M/(T-1) - M; endpoints are exactly lo and hi. */
ORC_API double orc_beta(int32_t q, double lo, double hi, int32_t T) {
  if (q == 0) return lo;
  if (q == T - 1) return hi;
  return (double)q * (hi - lo) / (double)(T - 1) + lo;
}

/* ------------------------------------------------------------------------ */
/* Complex descriptor (the Complex list of tuples).              */
/*   dimension 0: k0 vertices with weights vw[k0]                           */
/*   dimension i: cells[i] = (verts [count, arity] row-major, weights,      */
/*                dim) -- arity i+1 for simplices, 2^i for cubes */
/* Weights are int64 or double, selected by is_float.                        */
/* ------------------------------------------------------------------------ */
typedef struct {
  const int32_t* verts;
  const void* weights; /* int64_t* or double*; NULL => unit weights */
  int64_t count;
  int32_t arity;
  int32_t dim;
} orc_cells;

static double w_f(const void* w, int is_float, int64_t i) {
  if (!w) return 1.0;
  return is_float ? ((const double*)w)[i] : (double)((const int64_t*)w)[i];
}
static int64_t w_i(const void* w, int64_t i) {
  return w ? ((const int64_t*)w)[i] : 1;
}

/* Neumaier-compensated add for float weights (A8). */
static void kahan_add(double* s, double* c, double x) {
  double t = *s + x;
  if (fabs(*s) >= fabs(x)) *c += (*s - t) + x;
  else *c += (x - t) + *s;
  *s = t;
}

/* ------------------------------------------------------------------------ */
/* O2: Algorithm 1 ComputeWECFs(Complex, numvals).             */
/* out: [m, T]; int64 for integer weights, double for float weights.        */
/* Returns 0, or -2 if a vertex index is out of range (nothing written).    */
/* ------------------------------------------------------------------------ */
ORC_API int orc_wecfs_alg1(const double* fvals, int64_t k0, int32_t m,
                           const void* vweights, const orc_cells* cells, int32_t ncell_dims,
                           int is_float, int32_t T, double lo, double hi, void* out) {
  for (int32_t c = 0; c < ncell_dims; ++c)
    for (int64_t e = 0; e < cells[c].count * (int64_t)cells[c].arity; ++e)
      if (cells[c].verts[e] < 0 || cells[c].verts[e] >= k0) return -2;

#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t p = 0; p < m; ++p) {
    /* line 2: DiffWECFs <- zeros(m, numvals)   (row p only) */
    int64_t* diff_i = (int64_t*)calloc((size_t)T, sizeof(int64_t));
    double* diff_f = (double*)calloc((size_t)T, sizeof(double));
    double* diff_c = (double*)calloc((size_t)T, sizeof(double));
    /* line 3: VIndices <- alpha(FVals)  (eq. v-inds) */
    int32_t* vind = (int32_t*)malloc((size_t)(k0 > 0 ? k0 : 1) * sizeof(int32_t));
    for (int64_t a = 0; a < k0; ++a) vind[a] = orc_alpha(fvals[a * m + p], lo, hi, T);
    /* line 4: scatter_add(VIndices^T, VertexWeights)(DiffWECFs)  (D_0) */
    for (int64_t a = 0; a < k0; ++a) {
      if (is_float) kahan_add(&diff_f[vind[a]], &diff_c[vind[a]], w_f(vweights, 1, a));
      else diff_i[vind[a]] += w_i(vweights, a);
    }
    /* lines 5-10: for i = 1..dim(K) */
    for (int32_t c = 0; c < ncell_dims; ++c) {
      const orc_cells* C = &cells[c];
      int sign = (C->dim % 2 == 0) ? 1 : -1; /* (-1)^i */
      for (int64_t b = 0; b < C->count; ++b) {
        /* lines 7-8: SimpIndices = VIndices[SimplexVertices]; MSI = rmax(., 1)  (eq. msi) */
        int32_t msi = 0;
        for (int32_t j = 0; j < C->arity; ++j) {
          int32_t vi = vind[C->verts[b * C->arity + j]];
          if (j == 0 || vi > msi) msi = vi;
        }
        /* line 9: scatter_add(MSI^T, (-1)^i * SimplexWeights) */
        if (is_float) kahan_add(&diff_f[msi], &diff_c[msi], sign * w_f(C->weights, 1, b));
        else diff_i[msi] += sign * w_i(C->weights, b);
      }
    }
    /* line 11: WECFs <- cumsum(DiffWECFs) */
    if (is_float) {
      double s = 0.0, cc = 0.0;
      for (int32_t q = 0; q < T; ++q) {
        kahan_add(&s, &cc, diff_f[q]);
        kahan_add(&s, &cc, diff_c[q]);
        ((double*)out)[(int64_t)p * T + q] = s + cc;
      }
    } else {
      int64_t s = 0;
      for (int32_t q = 0; q < T; ++q) {
        s += diff_i[q];
        ((int64_t*)out)[(int64_t)p * T + q] = s;
      }
    }
    free(vind); free(diff_i); free(diff_f); free(diff_c);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O1: the naive discretised WECF, straight from the definitions */
/*   F(t) = { sigma : max_{v in sigma} f(v) <= t }        */
/*   wecf_f(t) = chi(F(t), w) = sum_{sigma in F(t)} (-1)^dim w(sigma)          */
/*                                                       */
/* evaluated at t = beta(q) for every q.  Theta(T * m * |K|).                 */
/* q_lo..q_hi-1 lets callers evaluate a subset of columns (sampled parity).  */
/* ------------------------------------------------------------------------ */
ORC_API int orc_wecfs_naive(const double* fvals, int64_t k0, int32_t m,
                            const void* vweights, const orc_cells* cells, int32_t ncell_dims,
                            int is_float, int32_t T, double lo, double hi, void* out) {
  for (int32_t c = 0; c < ncell_dims; ++c)
    for (int64_t e = 0; e < cells[c].count * (int64_t)cells[c].arity; ++e)
      if (cells[c].verts[e] < 0 || cells[c].verts[e] >= k0) return -2;
  int degenerate = !(hi > lo);
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t p = 0; p < m; ++p) {
    for (int32_t q = 0; q < T; ++q) {
      double t = degenerate ? lo : orc_beta(q, lo, hi, T);
      int64_t si = 0;
      double sf = 0.0, sc = 0.0;
      /* vertices (dimension 0) */
      for (int64_t a = 0; a < k0; ++a) {
        if (degenerate || fvals[a * m + p] <= t) {
          if (is_float) kahan_add(&sf, &sc, w_f(vweights, 1, a));
          else si += w_i(vweights, a);
        }
      }
      for (int32_t c = 0; c < ncell_dims; ++c) {
        const orc_cells* C = &cells[c];
        int sign = (C->dim % 2 == 0) ? 1 : -1;
        for (int64_t b = 0; b < C->count; ++b) {
          double fmax = fvals[(int64_t)C->verts[b * C->arity] * m + p];
          for (int32_t j = 1; j < C->arity; ++j) {
            double f = fvals[(int64_t)C->verts[b * C->arity + j] * m + p];
            if (f > fmax) fmax = f;
          }
          if (degenerate || fmax <= t) {
            if (is_float) kahan_add(&sf, &sc, sign * w_f(C->weights, 1, b));
            else si += sign * w_i(C->weights, b);
          }
        }
      }
      if (is_float) ((double*)out)[(int64_t)p * T + q] = sf + sc;
      else ((int64_t*)out)[(int64_t)p * T + q] = si;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Image embedding (reading A3; the paper fixes none): grid index g along an  */
/* axis of length L becomes (g - (L-1)/2) / S with S = max(max_dim - 1, 1),    */
/* evaluated in binary64 and rounded once to fp32.  Column -> axis 0, row ->   */
/* axis 1 (2D); column -> 0, row -> 1, slice -> 2 (3D).                       */
/* ------------------------------------------------------------------------ */
static float axis_coord(int64_t g, int64_t L, double S) {
  return (float)(((double)g - (double)(L - 1) / 2.0) / S);
}

/* Vertex coordinates of an image grid with ndim dims (slowest first:        */
/* 2D = (H, W), 3D = (Z, Y, X)); coords [prod(dims), ndim].                  */
ORC_API void orc_grid_coords(int32_t ndim, const int64_t* dims, float* coords) {
  int64_t maxd = 1;
  for (int i = 0; i < ndim; ++i) if (dims[i] > maxd) maxd = dims[i];
  double S = (double)(maxd - 1 > 1 ? maxd - 1 : 1);
  int64_t nv = 1;
  for (int i = 0; i < ndim; ++i) nv *= dims[i];
  for (int64_t v = 0; v < nv; ++v) {
    int64_t rem = v;
    /* axis k of the coordinate = grid dim (ndim-1-k): fastest dim -> axis 0 */
    for (int k = 0; k < ndim; ++k) {
      int d = ndim - 1 - k;
      int64_t g = rem % dims[d];
      rem /= dims[d];
      coords[v * ndim + k] = axis_coord(g, dims[d], S);
    }
  }
}

/* Cubical complex (V-construction) of an image (P:213-215;       */
/* cells stored by their 2^i corners).  Every i-cube is the product   */
/* of one unit step along each axis in a subset of i axes.  Its weight is the */
/* max of its corner intensities (reading A5).                    */
/* This function returns the number of cells of each dimension in counts[]   */
/* (counts[0..ndim]) when verts == NULL; otherwise fills, per dimension i,   */
/* verts_i [k_i, 2^i] and weights_i [k_i] (int64) in the order: axis subsets */
/* by increasing bitmask, then lower corner in row-major order.             */
ORC_API void orc_grid_cells(int32_t ndim, const int64_t* dims, const uint8_t* img,
                            int64_t* counts, int32_t** verts, int64_t** weights) {
  int64_t nv = 1;
  for (int i = 0; i < ndim; ++i) nv *= dims[i];
  int64_t fill[4] = {0, 0, 0, 0};
  if (!verts) {
    for (int i = 0; i <= ndim; ++i) counts[i] = 0;
  }
  for (int mask = 0; mask < (1 << ndim); ++mask) {
    int dim = __builtin_popcount(mask);
    if (dim == 0) continue;
    int arity = 1 << dim;
    /* axis k <-> grid dim ndim-1-k; a step along axis k adds stride_k */
    int64_t stride[3], ext[3];
    int64_t st = 1;
    for (int d = ndim - 1; d >= 0; --d) { stride[ndim - 1 - d] = st; ext[ndim - 1 - d] = dims[d]; st *= dims[d]; }
    for (int64_t v = 0; v < nv; ++v) {
      /* lower corner v must allow a +1 step on every axis in mask */
      int64_t rem = v; int ok = 1;
      for (int k = 0; k < ndim; ++k) {
        int64_t g = rem % ext[k]; rem /= ext[k];
        if ((mask >> k) & 1) if (g + 1 >= ext[k]) ok = 0;
      }
      if (!ok) continue;
      if (!verts) { counts[dim]++; continue; }
      int64_t idx = fill[dim]++;
      int64_t wmax = 0;
      int j = 0;
      for (int sub = 0; sub < (1 << ndim); ++sub) {
        if ((sub & ~mask) != 0) continue; /* corners: subsets of mask */
        int64_t u = v;
        for (int k = 0; k < ndim; ++k) if ((sub >> k) & 1) u += stride[k];
        verts[dim][idx * arity + j++] = (int32_t)u;
        if (img[u] > wmax) wmax = img[u];
      }
      weights[dim][idx] = wmax;
    }
  }
}

/* Convenience: the full O2 WECT of a batch of images / volumes through the  */
/* explicit cubical complex.  img [B, prod(dims)], dirs [D, ndim] fp32,       */
/* out int64 [B, D, T].  M is max |h| over all vertices and ALL D directions  */
/* (reading A2); maxheight_override > 0 replaces it.              */
/* naive != 0 selects O1 instead of O2.                                       */
ORC_API int orc_wect_images(const uint8_t* img, int64_t B, int32_t ndim, const int64_t* dims,
                            const float* dirs, int32_t D, int32_t T, double maxheight_override,
                            int naive, int64_t* out) {
  int64_t nv = 1;
  for (int i = 0; i < ndim; ++i) nv *= dims[i];
  float* coords = (float*)malloc((size_t)nv * ndim * sizeof(float));
  orc_grid_coords(ndim, dims, coords);
  double* fv = (double*)malloc((size_t)nv * D * sizeof(double));
  orc_heights(coords, nv, ndim, dirs, D, fv);
  double M = maxheight_override > 0 ? maxheight_override : orc_maxheight(fv, nv, D);
  int64_t counts[4];
  orc_grid_cells(ndim, dims, NULL, counts, NULL, NULL);
  int32_t* verts[4] = {0}; int64_t* wts[4] = {0};
  for (int i = 1; i <= ndim; ++i) {
    verts[i] = (int32_t*)malloc((size_t)(counts[i] > 0 ? counts[i] : 1) * (1 << i) * sizeof(int32_t));
    wts[i] = (int64_t*)malloc((size_t)(counts[i] > 0 ? counts[i] : 1) * sizeof(int64_t));
  }
  int64_t* vw = (int64_t*)malloc((size_t)nv * sizeof(int64_t));
  int rc = 0;
  for (int64_t b = 0; b < B && rc == 0; ++b) {
    const uint8_t* im = img + b * nv;
    orc_grid_cells(ndim, dims, im, counts, verts, wts);
    for (int64_t v = 0; v < nv; ++v) vw[v] = im[v];
    orc_cells cl[3];
    int nc = 0;
    for (int i = 1; i <= ndim; ++i) {
      cl[nc].verts = verts[i]; cl[nc].weights = wts[i]; cl[nc].count = counts[i];
      cl[nc].arity = 1 << i; cl[nc].dim = i; ++nc;
    }
    if (naive) rc = orc_wecfs_naive(fv, nv, D, vw, cl, nc, 0, T, -M, M, out + b * (int64_t)D * T);
    else rc = orc_wecfs_alg1(fv, nv, D, vw, cl, nc, 0, T, -M, M, out + b * (int64_t)D * T);
  }
  for (int i = 1; i <= ndim; ++i) { free(verts[i]); free(wts[i]); }
  free(vw); free(fv); free(coords);
  return rc;
}

/* thread count of the OpenMP loops (bench: the single-core baseline) */
ORC_API void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

ORC_API int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
