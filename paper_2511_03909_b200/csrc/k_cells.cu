// k_cells.cu -- thread-per-cell streaming kernels for FEW filters: the ECF (ecf_complex)
// and the WECT of an explicit complex at small D (the HBM-bound end of the D-sweep,
// SURVEY 8(d)).  Alg. 1 with each thread owning cells: gather the filter
// values (MODE 0: FVals[v, p]; MODE 1: <coords[v], s_p> by fp32 FMA), rmax (eq. msi),
// bin (reading A1 guard + binary64 repair), one shared-memory atomic per (cell, filter)
// into a [filters][T+1] histogram, one merge per CTA; k_finalize does the cumsum.
#include <cfloat>

#include "common.cuh"

namespace wect {

constexpr int kCellTile = 8;  // filters per CTA

__device__ __noinline__ int ecf_repair(float hmax, const GridParams* gp) {
  note_repair();
  return alpha64((double)hmax, *gp);  // filter values are exact in binary64
}

// binary64 heights of a cell's vertices (axis order), max, alpha64 (reading A1)
template <int N>
__device__ __noinline__ int wect_repair(const float* x, int ar, const float* s, const GridParams* gp) {
  double hm = -DBL_MAX;
  for (int t = 0; t < ar; ++t) {
    double h = __dmul_rn((double)x[t * N], (double)s[0]);
    for (int i = 1; i < N; ++i) h = __dadd_rn(h, __dmul_rn((double)x[t * N + i], (double)s[i]));
    hm = fmax(hm, h);
  }
  note_repair();
  return alpha64(hm, *gp);
}

__device__ __forceinline__ int fast_bin(float hmax, const GridParams& g, bool& near) {
  const float uu = fmaf(hmax, g.A, g.B);
  int bin = __float2int_ru(uu);
  bin = bin < 0 ? 0 : (bin > g.T - 1 ? g.T - 1 : bin);
  near = !g.fp32_only && fabsf(uu - rintf(uu)) < g.tau;
  return bin;
}

template <typename Acc>
__device__ __forceinline__ void cell_count(int bin, Acc w, int pp, Acc* hist, int TS) {
  if (w != (Acc)0) atomicAdd(&hist[pp * TS + bin], w);
}

// Evaluate NC cells of arity AR whose vertex ids are v[NC*AR] (NC = 1 or 4).
template <int MODE, int N, int AR, int NC, bool FLOATW, typename Acc>
__device__ __forceinline__ void cells_eval(const int* v, const Acc* w, const float* __restrict__ fvals, int m, int p0,
                                           int np, const float* __restrict__ coords, const float* sdir,
                                           const GridParams& g, const GridParams* gp, Acc* hist, int TS) {
  if constexpr (MODE == 0) {
    for (int pp = 0; pp < np; ++pp) {
      float h[NC * AR];
#pragma unroll
      for (int i = 0; i < NC * AR; ++i) h[i] = __ldg(fvals + (int64_t)v[i] * m + p0 + pp);
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        float hmax = h[u * AR];
#pragma unroll
        for (int t = 1; t < AR; ++t) hmax = fmaxf(hmax, h[u * AR + t]);
        bool near;
        int bin = fast_bin(hmax, g, near);
        if (near) bin = ecf_repair(hmax, gp);
        cell_count<Acc>(bin, w[u], pp, hist, TS);
      }
    }
  } else {
    float x[NC * AR * N];
#pragma unroll
    for (int i = 0; i < NC * AR; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) x[i * N + j] = __ldg(coords + (int64_t)v[i] * N + j);
    for (int pp = 0; pp < np; ++pp) {
      const float* s = sdir + pp * N;
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        float hmax = -FLT_MAX;
#pragma unroll
        for (int t = 0; t < AR; ++t) {
          const float* xv = x + (u * AR + t) * N;
          float h = xv[0] * s[0];
#pragma unroll
          for (int i = 1; i < N; ++i) h = fmaf(xv[i], s[i], h);
          hmax = fmaxf(hmax, h);
        }
        bool near;
        int bin = fast_bin(hmax, g, near);
        if (near) bin = wect_repair<N>(x + u * AR * N, AR, s, gp);
        cell_count<Acc>(bin, w[u], pp, hist, TS);
      }
    }
  }
}

// One segment range [b0, b1) of arity AR.  Body: each thread takes 4 consecutive cells
// with 16-byte loads (AR int4 of indices, one of weights), then all their gathers.
template <int MODE, int N, bool FLOATW, int AR, typename Acc>
__device__ __forceinline__ void cell_segment(const Seg& S, int64_t b0, int64_t b1, int64_t k0,
                                             const float* __restrict__ fvals, int m, int p0, int np,
                                             const float* __restrict__ coords, const float* sdir, const GridParams& g,
                                             const GridParams* gp, Acc* hist, int TS) {
  auto scalar_cell = [&](int64_t b) {
    Acc w[1] = {cell_weight<FLOATW, Acc>(S, b)};
    int v[AR];
    bool ok = true;
#pragma unroll
    for (int t = 0; t < AR; ++t) {
      v[t] = S.verts ? __ldg(S.verts + b * AR + t) : (int)b;
      if ((uint64_t)(int64_t)v[t] >= (uint64_t)k0) { ok = false; v[t] = 0; }
    }
    if (!ok) { atomicOr(&g_err_word, 1u); return; }
    cells_eval<MODE, N, AR, 1, FLOATW, Acc>(v, w, fvals, m, p0, np, coords, sdir, g, gp, hist, TS);
  };
  const bool vec_ok = S.verts && (((uintptr_t)S.verts & 15) == 0) && (!S.weights || ((uintptr_t)S.weights & 15) == 0);
  int64_t vb0 = b1, vb1 = b1;
  if (vec_ok) {
    vb0 = (b0 + 3) & ~(int64_t)3;
    vb1 = vb0 + ((b1 - vb0) > 0 ? ((b1 - vb0) & ~(int64_t)3) : 0);
    if (vb0 > b1) vb0 = vb1 = b1;
  }
  for (int64_t b = b0 + threadIdx.x; b < (vec_ok ? vb0 : b1); b += blockDim.x) scalar_cell(b);  // head
  for (int64_t b = vb1 + threadIdx.x; b < b1; b += blockDim.x) scalar_cell(b);                  // tail
  for (int64_t b4 = vb0 + 4 * (int64_t)threadIdx.x; b4 < vb1; b4 += 4 * (int64_t)blockDim.x) {
    int v[4 * AR];
    const int4* vp = (const int4*)(S.verts + b4 * AR);
#pragma unroll
    for (int i = 0; i < AR; ++i) {
      const int4 x = __ldcs(vp + i);  // streamed once: evict-first
      v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
    }
    Acc w[4];
    if (S.weights) {
      if (FLOATW) {
        const float4 x = __ldcs((const float4*)S.weights + (b4 >> 2));
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
      } else {
        const int4 x = __ldcs((const int4*)S.weights + (b4 >> 2));
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
      }
    } else {
      w[0] = w[1] = w[2] = w[3] = (Acc)1;
    }
    if (S.sign < 0) { w[0] = -w[0]; w[1] = -w[1]; w[2] = -w[2]; w[3] = -w[3]; }
    unsigned bad = 0;
#pragma unroll
    for (int i = 0; i < 4 * AR; ++i)
      if ((uint64_t)(int64_t)v[i] >= (uint64_t)k0) { bad |= 1u << (i / AR); v[i] = 0; }
    if (bad) {
      atomicOr(&g_err_word, 1u);
#pragma unroll
      for (int u = 0; u < 4; ++u) if ((bad >> u) & 1u) w[u] = (Acc)0;
    }
    if constexpr (MODE == 1 && AR * N > 12) {  // keep the coordinate registers bounded
#pragma unroll
      for (int u = 0; u < 4; ++u)
        cells_eval<MODE, N, AR, 1, FLOATW, Acc>(v + u * AR, w + u, fvals, m, p0, np, coords, sdir, g, gp, hist, TS);
    } else {
      cells_eval<MODE, N, AR, 4, FLOATW, Acc>(v, w, fvals, m, p0, np, coords, sdir, g, gp, hist, TS);
    }
  }
}

template <int MODE, int N, bool FLOATW>
__global__ void __launch_bounds__(256, MODE == 0 ? 3 : 2) k_cells(Segs segs, int64_t k0, const float* __restrict__ fvals, int m,
                                                  const float* __restrict__ coords, const float* __restrict__ dirs,
                                                  int d_begin, int Dc, const GridParams* __restrict__ gp,
                                                  const unsigned int* __restrict__ wmax_bits, int64_t slice_len,
                                                  int64_t float_chunk, void* __restrict__ diff) {
  using Acc = typename std::conditional<FLOATW, float, int>::type;
  constexpr int NS = N > 0 ? N : 1;
  extern __shared__ __align__(16) unsigned char smraw[];
  const GridParams g = *gp;
  const int T = g.T, TS = T + 1;
  Acc* hist = (Acc*)smraw;  // [kCellTile][T+1]
  __shared__ Seg ssegs[kMaxSegs];
  __shared__ float sdir[kCellTile * NS];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kMaxSegs; ++i) ssegs[i] = segs.s[i];
  }
  const int p0 = d_begin + blockIdx.x * kCellTile;
  const int np = (Dc - (int)blockIdx.x * kCellTile) < kCellTile ? (Dc - (int)blockIdx.x * kCellTile) : kCellTile;
  if (MODE == 1)
    for (int i = threadIdx.x; i < np * NS; i += blockDim.x) sdir[i] = dirs[p0 * NS + i];
  for (int i = threadIdx.x; i < kCellTile * TS; i += blockDim.x) hist[i] = (Acc)0;
  const int64_t c0 = blockIdx.y * slice_len;
  const int64_t c1 = (c0 + slice_len) < segs.total ? (c0 + slice_len) : segs.total;
  const int64_t chunk = chunk_cells(FLOATW, float_chunk, wmax_bits, c1 - c0);
  __syncthreads();
  for (int64_t a0 = c0; a0 < c1; a0 += chunk) {
    const int64_t a1 = (a0 + chunk) < c1 ? (a0 + chunk) : c1;
    for (int sg = 0; sg < kMaxSegs; ++sg) {
      const Seg& S = ssegs[sg];
      const int64_t lo = a0 > S.start ? a0 : S.start;
      const int64_t hi = a1 < S.start + S.count ? a1 : S.start + S.count;
      if (lo >= hi) continue;
      const int64_t b0 = lo - S.start, b1 = hi - S.start;
      switch (S.arity) {
#define WECT_AR(A)                                                                                          \
  case A:                                                                                                   \
    cell_segment<MODE, NS, FLOATW, A>(S, b0, b1, k0, fvals, m, p0, np, coords, sdir, g, gp, hist, TS); \
    break;
        WECT_AR(1) WECT_AR(2) WECT_AR(3) WECT_AR(4)
#undef WECT_AR
        default: {  // other arities: one vertex at a time
          for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
            const Acc w = cell_weight<FLOATW, Acc>(S, b);
            bool bad = false;
            for (int t = 0; t < S.arity; ++t) {
              const int v = S.verts ? __ldg(S.verts + b * S.arity + t) : (int)b;
              bad |= (uint64_t)(int64_t)v >= (uint64_t)k0;
            }
            if (bad) { atomicOr(&g_err_word, 1u); continue; }
            for (int pp = 0; pp < np; ++pp) {
              float hmax = -FLT_MAX;
              for (int t = 0; t < S.arity; ++t) {
                const int v = S.verts ? __ldg(S.verts + b * S.arity + t) : (int)b;
                float h;
                if (MODE == 0) h = __ldg(fvals + (int64_t)v * m + p0 + pp);
                else {
                  h = coords[(int64_t)v * NS] * sdir[pp * NS];
                  for (int i = 1; i < NS; ++i) h = fmaf(coords[(int64_t)v * NS + i], sdir[pp * NS + i], h);
                }
                hmax = fmaxf(hmax, h);
              }
              bool near;
              int bin = fast_bin(hmax, g, near);
              if (near) {
                if (MODE == 0) bin = ecf_repair(hmax, gp);
                else {
                  double hm = -DBL_MAX;
                  for (int t = 0; t < S.arity; ++t) {
                    const int v = S.verts ? __ldg(S.verts + b * S.arity + t) : (int)b;
                    double h = __dmul_rn((double)coords[(int64_t)v * NS], (double)sdir[pp * NS]);
                    for (int i = 1; i < NS; ++i)
                      h = __dadd_rn(h, __dmul_rn((double)coords[(int64_t)v * NS + i], (double)sdir[pp * NS + i]));
                    hm = fmax(hm, h);
                  }
                  note_repair();
                  bin = alpha64(hm, g);
                }
              }
              cell_count<Acc>(bin, w, pp, hist, TS);
            }
          }
        }
      }
    }
    __syncthreads();
    flush_hist<FLOATW, Acc>(hist, np, T, TS, blockIdx.x * kCellTile, Dc, diff);
    __syncthreads();
  }
}

template <int MODE, int N>
static wect_status launch_cells_t(bool floatw, const Segs& segs, int64_t k0, const float* fvals, int m,
                                const float* coords, const float* dirs, int d_begin, int Dc, int T,
                                const GridParams* gp, const unsigned int* wmax, void* diff, cudaStream_t st,
                                int num_sms) {
  const int tiles = (Dc + kCellTile - 1) / kCellTile;
  const size_t smem = (size_t)kCellTile * (T + 1) * 4;
  int per_sm = (int)((220 * 1024) / (smem + 2048));
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const int64_t slice = pick_slice(segs.total, tiles, per_sm, num_sms, (int64_t)1 << 20);
  dim3 grid(tiles, (unsigned)((segs.total + slice - 1) / slice));
  MainTimer timer(st);
  if (floatw) {
    auto k = k_cells<MODE, N, true>;
    WECT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, st>>>(segs, k0, fvals, m, coords, dirs, d_begin, Dc, gp, wmax, slice, 4096, diff);
  } else {
    auto k = k_cells<MODE, N, false>;
    WECT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, st>>>(segs, k0, fvals, m, coords, dirs, d_begin, Dc, gp, wmax, slice, 4096, diff);
  }
  count_launch();
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}


wect_status launch_cells(int mode, int n, bool floatw, const Segs& segs, int64_t k0, const float* fvals, int m,
                         const float* coords, const float* dirs, int d_begin, int Dc, int T, const GridParams* gp,
                         const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms) {
  if (mode == 1)
    return launch_cells_t<0, 0>(floatw, segs, k0, fvals, m, nullptr, nullptr, d_begin, Dc, T, gp, wmax, diff, st,
                                num_sms);
  switch (n) {
#define WECT_CASE(NN) \
  case NN: return launch_cells_t<1, NN>(floatw, segs, k0, nullptr, 0, coords, dirs, d_begin, Dc, T, gp, wmax, diff, st, num_sms);
    WECT_CASE(1) WECT_CASE(2) WECT_CASE(3) WECT_CASE(4) WECT_CASE(5) WECT_CASE(6) WECT_CASE(7) WECT_CASE(8)
#undef WECT_CASE
  }
  return fail(WECT_EINVAL, "ambient dimension n=%d outside [1,8]", n);
}

}  // namespace wect
