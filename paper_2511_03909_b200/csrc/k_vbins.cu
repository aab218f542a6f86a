// k_vbins.cu -- WECT of an explicit complex at large D, in two passes per tile of 64
// directions:
//
//   k_vbins     VB[v][p] = alpha(<coords[v], s_p>) for every vertex and the tile's 64
//               directions, u16, exact per reading A1 (fp32 FMA + guard, binary64 repair).
//               Alg. 1 line 3 (VIndices = alpha(FVals)), one tile at a time.
//   k_cells_vb  per cell: MSI = max over its vertices of VB rows (lines 7-8, eq. msi --
//               alpha is monotone so the max of exact vertex bins is the exact cell bin),
//               two directions per lane with packed u16x2 max, one shared-memory atomic per
//               (cell, direction) into a lane-interleaved [T][2][32] histogram (line 9).
//
// Heights are computed once per (vertex, direction) instead of once per (cell, vertex,
// direction); a cell costs `arity` coalesced 128-byte row loads (L2-resident for meshes
// stored in spatial order) and a packed max, independent of n.
#include <cfloat>
#include <cstdint>

#include "common.cuh"

namespace wect {

constexpr int kVbTile = 64;  // directions per tile: two per lane

template <int N>
__device__ __noinline__ int vertex_repair(const float* x, const float* s, const GridParams* gp) {
  double h = __dmul_rn((double)x[0], (double)s[0]);
  for (int i = 1; i < N; ++i) h = __dadd_rn(h, __dmul_rn((double)x[i], (double)s[i]));
  note_repair();
  return alpha64(h, *gp);
}

template <int N>
__device__ __forceinline__ int vbin(const float* x, const float* s, const GridParams& g, const GridParams* gp) {
  float h = x[0] * s[0];
#pragma unroll
  for (int i = 1; i < N; ++i) h = fmaf(x[i], s[i], h);
  const float u = fmaf(h, g.A, g.B);
  int b = __float2int_ru(u);
  b = b < 0 ? 0 : (b > g.T - 1 ? g.T - 1 : b);
  if (__builtin_expect(!g.fp32_only && fabsf(u - rintf(u)) < g.tau, 0)) b = vertex_repair<N>(x, s, gp);
  return b;
}

// grid: blocks over vertices; lanes = direction pairs of the tile; each warp stages 32
// vertices' coordinates (lane-parallel), then writes one 128-byte VB row per vertex.
template <int N>
__global__ void __launch_bounds__(256) k_vbins(const float* __restrict__ coords, int64_t k0,
                                               const float* __restrict__ dirs, int p0, int np,
                                               const GridParams* __restrict__ gp, uint32_t* __restrict__ vb) {
  __shared__ float xs[8][32 * N];
  const GridParams g = *gp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float sa[N], sb[N];
  const int pa = 2 * lane, pb = 2 * lane + 1;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    sa[i] = pa < np ? dirs[(int64_t)(p0 + pa) * N + i] : 0.f;
    sb[i] = pb < np ? dirs[(int64_t)(p0 + pb) * N + i] : 0.f;
  }
  float* x = xs[warp];
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t base = ((int64_t)blockIdx.x * 8 + warp) * 32; base < k0; base += nwarps * 32) {
    const int nv = (k0 - base) < 32 ? (int)(k0 - base) : 32;
    for (int t = lane; t < nv * N; t += 32) x[t] = __ldg(coords + base * N + t);
    __syncwarp();
    for (int j = 0; j < nv; ++j) {
      float xv[N];
#pragma unroll
      for (int i = 0; i < N; ++i) xv[i] = x[j * N + i];
      const int ba = pa < np ? vbin<N>(xv, sa, g, gp) : 0, bb = pb < np ? vbin<N>(xv, sb, g, gp) : 0;
      vb[(base + j) * 32 + lane] = (uint32_t)ba | ((uint32_t)bb << 16);
    }
    __syncwarp();
  }
}

// red.shared for int / CAS-based atomicAdd for float (fp32 shared atomics are CAS loops on sm_100)
__device__ __forceinline__ void hist_add(int* h, int w) { atomicAdd(h, w); }
__device__ __forceinline__ void hist_add(float* h, float w) { atomicAdd(h, w); }

constexpr int kVbBatch = 32;  // cells per warp batch

// nb cells of arity AR (0: runtime `arr`) from the warp's staged ids: four cells at a
// time, all 4*AR row loads issued before the packed max and the atomics.
template <int AR, bool FLOATW, typename Acc>
__device__ __forceinline__ void vb_batch(const int* ids, int nb, Acc wl, const uint32_t* __restrict__ vb, Acc* hl,
                                         int lane, int arr = AR) {
  const int ar = AR > 0 ? AR : arr;
  constexpr int RA = AR > 0 ? AR : 1;
  for (int j = 0; j < nb; j += 4) {
    uint32_t m2[4];
    if (AR > 0) {
      uint32_t x[4][RA];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int t = 0; t < RA; ++t) x[u][t] = (j + u < nb) ? __ldg(vb + (int64_t)ids[(j + u) * RA + t] * 32 + lane) : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        m2[u] = x[u][0];
#pragma unroll
        for (int t = 1; t < RA; ++t) m2[u] = __vmaxu2(m2[u], x[u][t]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        m2[u] = 0;
        if (j + u < nb)
          for (int t = 0; t < ar; ++t) m2[u] = __vmaxu2(m2[u], __ldg(vb + (int64_t)ids[(j + u) * ar + t] * 32 + lane));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const Acc w = __shfl_sync(0xffffffffu, wl, (j + u) & 31);
      if (j + u < nb && w != (Acc)0) {
        hist_add(hl + (m2[u] & 0xFFFFu) * 64, w);
        hist_add(hl + (m2[u] >> 16) * 64 + 32, w);
      }
    }
  }
}

// merge a CTA's [T][2][32] histogram into the global difference table and clear it
template <bool FLOATW, typename Acc>
__device__ __forceinline__ void flush_tile(Acc* hist, int T, int row0, int np, void* diff) {
  for (int i = threadIdx.x; i < T * 64; i += blockDim.x) {
    const int q = i >> 6, col = i & 63, half = col >> 5, l = col & 31;
    const int r = 2 * l + half;  // direction within the tile
    const Acc val = hist[i];
    if (val != (Acc)0 && r < np) {
      const int64_t o = (int64_t)(row0 + r) * T + q;
      if (FLOATW) atomicAdd((double*)diff + o, (double)val);
      else atomicAdd((unsigned long long*)diff + o, (unsigned long long)(long long)val);
    }
    hist[i] = (Acc)0;
  }
}

// Work order (L2 locality): batches of kVbBatch cells of every segment advance in NSTEP
// lock-steps; in step i each segment's batches [i U_s / NSTEP, (i+1) U_s / NSTEP) are
// spread over all warps of the grid (grid-stride).  For a complex stored in spatial
// order this keeps the concurrently gathered VB rows inside a narrow vertex window, so
// each row comes from HBM about once per tile.  One histogram flush per CTA at the end
// (the launcher checks max|w| * cells-per-CTA < 2^31 for integer weights).
template <bool FLOATW>
__global__ void __launch_bounds__(512) k_cells_vb(Segs segs, int64_t k0, const uint32_t* __restrict__ vb, int row0,
                                                  int np, int Dc, const GridParams* __restrict__ gp, int nstep,
                                                  const unsigned int* __restrict__ wmax_bits, int64_t cta_cells_step,
                                                  void* __restrict__ diff) {
  using Acc = typename std::conditional<FLOATW, float, int>::type;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int T = gp->T;
  Acc* hist = (Acc*)smraw;  // [T][2][32]: column (half, lane) = direction 2*lane + half
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int* ids = (int*)(smraw + (size_t)T * 64 * sizeof(Acc)) + warp * (kVbBatch * 8);
  __shared__ Seg ssegs[kMaxSegs];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kMaxSegs; ++i) ssegs[i] = segs.s[i];
  }
  for (int i = threadIdx.x; i < T * 64; i += blockDim.x) hist[i] = (Acc)0;
  Acc* hl = hist + lane;
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp, W = (int64_t)gridDim.x * nwarps;
  // int32 partials: flush every `every` steps so that max|w| * cells since the flush < 2^31
  int every = nstep;
  if (!FLOATW) {
    const unsigned int wm = *wmax_bits;
    if (wm) {
      const int64_t e = (int64_t)2147483647 / ((int64_t)wm * cta_cells_step);
      every = e < 1 ? 1 : (e < nstep ? (int)e : nstep);
    }
  } else {  // float partials (fp32) are merged into binary64 every <= 32768 cells (reading A8)
    const int64_t e = 32768 / (cta_cells_step > 0 ? cta_cells_step : 1);
    every = e < 1 ? 1 : (e < nstep ? (int)e : nstep);
  }
  __syncthreads();
  for (int step = 0; step < nstep; ++step) {
    if (step > 0 && step % every == 0) {
      __syncthreads();
      flush_tile<FLOATW, Acc>(hist, T, row0, np, diff);
      __syncthreads();
    }
    for (int sg = 0; sg < segs.nseg; ++sg) {
      const Seg& S = ssegs[sg];
      const int ar = S.arity;
      int bs = (kVbBatch * 8) / ar;
      bs = bs > kVbBatch ? kVbBatch : bs;
      const int64_t U = (S.count + bs - 1) / bs;
      const int64_t u0 = U * step / nstep, u1 = U * (step + 1) / nstep;
      for (int64_t u = u0 + ((gw - u0) % W + W) % W; u < u1; u += W) {
        const int64_t b0 = u * bs;
        const int nb = (S.count - b0) < bs ? (int)(S.count - b0) : bs;
        unsigned badcells = 0;
        for (int t = lane; t < nb * ar; t += 32) {
          int v = S.verts ? __ldg(S.verts + b0 * ar + t) : (int)(b0 + t);
          if ((uint64_t)(int64_t)v >= (uint64_t)k0) { badcells |= 1u << (t / ar); v = 0; }
          ids[t] = v;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) badcells |= __shfl_xor_sync(0xffffffffu, badcells, o);
        Acc wl = (Acc)0;
        if (lane < nb && !((badcells >> lane) & 1u)) wl = cell_weight<FLOATW, Acc>(S, b0 + lane);
        if (badcells && lane == 0) atomicOr(&g_err_word, 1u);
        __syncwarp();
        switch (ar) {
          case 1: vb_batch<1, FLOATW>(ids, nb, wl, vb, hl, lane); break;
          case 2: vb_batch<2, FLOATW>(ids, nb, wl, vb, hl, lane); break;
          case 3: vb_batch<3, FLOATW>(ids, nb, wl, vb, hl, lane); break;
          case 4: vb_batch<4, FLOATW>(ids, nb, wl, vb, hl, lane); break;
          case 5: vb_batch<5, FLOATW>(ids, nb, wl, vb, hl, lane); break;
          default: vb_batch<0, FLOATW>(ids, nb, wl, vb, hl, lane, ar); break;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  flush_tile<FLOATW, Acc>(hist, T, row0, np, diff);
}

template <int N>
static wect_status launch_vb_n(bool floatw, const Segs& segs, const float* coords, int64_t k0, const float* dirs,
                               int d_begin, int Dc, int T, const GridParams* gp, const unsigned int* wmax, void* diff,
                               cudaStream_t st, int num_sms) {
  uint32_t* vb = nullptr;
  WECT_CUDA_TRY(cudaMallocAsync((void**)&vb, (size_t)(k0 > 0 ? k0 : 1) * 32 * sizeof(uint32_t), st));
  const size_t smem = (size_t)T * 64 * 4 + (size_t)16 * kVbBatch * 8 * sizeof(int);
  int per_sm = (int)((220 * 1024) / (smem + 1024));  // 512-thread CTAs that fit one SM's smem
  per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
  const int ctas = num_sms * per_sm;
  // steps: every warp gets ~4 batches of EVERY segment per step (balanced, narrow window)
  int64_t minU = INT64_MAX;
  for (int i = 0; i < segs.nseg; ++i) {
    if (segs.s[i].count == 0) continue;
    int bs = (kVbBatch * 8) / segs.s[i].arity;
    bs = bs > kVbBatch ? kVbBatch : bs;
    const int64_t U = (segs.s[i].count + bs - 1) / bs;
    minU = U < minU ? U : minU;
  }
  const int64_t per_step = (int64_t)ctas * 16 * 4;  // 4 batches per warp per segment per step
  int nstep = minU == INT64_MAX ? 1 : (int)(minU / per_step);
  nstep = nstep < 1 ? 1 : nstep;
  int vblocks = (int)((k0 + 255) / 256);
  vblocks = vblocks > num_sms * 8 ? num_sms * 8 : (vblocks < 1 ? 1 : vblocks);
  // bound on the cells one CTA processes per step (for the int32 flush period)
  int64_t cta_cells_step = 0;
  for (int i = 0; i < segs.nseg; ++i) {
    const int ar = segs.s[i].arity;
    int bs = (kVbBatch * 8) / ar;
    bs = bs > kVbBatch ? kVbBatch : bs;
    const int64_t U = (segs.s[i].count + bs - 1) / bs;
    const int64_t per_warp = (U / nstep + 1 + (int64_t)ctas * 16 - 1) / ((int64_t)ctas * 16);
    cta_cells_step += 16 * per_warp * bs;
  }
  wect_status s = WECT_OK;
  for (int t0 = 0; t0 < Dc && s == WECT_OK; t0 += kVbTile) {
    const int np = (Dc - t0) < kVbTile ? (Dc - t0) : kVbTile;
    k_vbins<N><<<vblocks, 256, 0, st>>>(coords, k0, dirs, d_begin + t0, np, gp, vb);
    count_launch();
    MainTimer timer(st);
    if (floatw) {
      WECT_CUDA_TRY(cudaFuncSetAttribute(k_cells_vb<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_cells_vb<true><<<ctas, 512, smem, st>>>(segs, k0, vb, t0, np, Dc, gp, nstep, wmax, cta_cells_step, diff);
    } else {
      WECT_CUDA_TRY(cudaFuncSetAttribute(k_cells_vb<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_cells_vb<false><<<ctas, 512, smem, st>>>(segs, k0, vb, t0, np, Dc, gp, nstep, wmax, cta_cells_step, diff);
    }
    count_launch();
    timer.stop();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) s = fail_cuda(e, "k_cells_vb", __FILE__, __LINE__);
  }
  cudaFreeAsync(vb, st);
  return s;
}

// smem fits, and (integer weights) a CTA's int32 partials cannot overflow: every CTA sees at
// most total/num_sms + one step's worth of cells, checked against the host bound on max|w|
// (255 for the configs; callers with larger weights fall back to k_complex's chunked flush)
bool vb_supported(int T) { return (size_t)T * 64 * 4 + (size_t)16 * kVbBatch * 8 * sizeof(int) <= 200 * 1024; }

wect_status launch_complex_vb(int n, bool floatw, const Segs& segs, const float* coords, int64_t k0,
                              const float* dirs, int d_begin, int Dc, int T, const GridParams* gp,
                              const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms) {
  switch (n) {
#define WECT_CASE(NN) \
  case NN: return launch_vb_n<NN>(floatw, segs, coords, k0, dirs, d_begin, Dc, T, gp, wmax, diff, st, num_sms);
    WECT_CASE(1) WECT_CASE(2) WECT_CASE(3) WECT_CASE(4) WECT_CASE(5) WECT_CASE(6) WECT_CASE(7) WECT_CASE(8)
#undef WECT_CASE
  }
  return fail(WECT_EINVAL, "ambient dimension n=%d outside [1,8]", n);
}

}  // namespace wect
