// k_complex.cu -- explicit weighted complexes (wect_complex, ecf_complex), the
// binary64 maxheight, and the cumsum epilogue shared with the image histogram path.
//
// Algorithm 1 fused into one streaming pass per direction tile:
//   line 3  VIndices = alpha(FVals)           -> per (cell, filter) in registers
//   line 7  SimpIndices = VIndices[verts]     -> gathered heights, never materialised
//   line 8  MSI = rmax(SimpIndices, 1)        -> max of the gathered heights (alpha is
//                                                monotone, eq. msi)
//   line 9  scatter_add(MSI^T, (-1)^i w)       -> shared-memory histogram, lanes = filters
//   line 11 cumsum                             -> k_finalize (warp-shuffle scan)
// The paper's Theta(k m) intermediates never exist: FVals for cfg4 would be
// 41 GB of fp32.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"

namespace wect {

__device__ unsigned int g_err_word = 0;
__device__ unsigned long long g_repair_count = 0;


// ---------------------------------------------------------------- maxheight
// pass 1: per vertex vmax32[v] = max_p |h32(v, p)| (fp32), global max M32 and
// R1 = max_v sum_i |x_vi| (for the guard).  pass 2 recomputes in binary64 every vertex
// whose fp32 max is within 2 err of M32 (err bounds |h32 - h64|), so the exact M64 =
// max |h64| is found (reading A2).
constexpr int kVmaxChunk = 4096;  // directions per shared-memory chunk of k_vmax_pass1 (<= 128 KB)

template <int N>
__global__ void __launch_bounds__(256) k_vmax_pass1(const float* __restrict__ coords, int64_t k0,
                                                    const float* __restrict__ dirs, int D, float* __restrict__ vmax,
                                                    unsigned int* __restrict__ m32_bits, unsigned int* __restrict__ r1_bits,
                                                    unsigned int* __restrict__ smax_bits) {
  extern __shared__ float sdir[];  // [KC][NP]: N <= 4 zero-padded to float4 rows (one LDS.128 per direction)
  constexpr int NP = N <= 4 ? 4 : N;
  constexpr int KC = kVmaxChunk;     // directions per shared-memory chunk
  float sm = 0.f, bm = 0.f, br = 0.f;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int p0 = 0; p0 < D; p0 += KC) {
    const int dc = (D - p0) < KC ? (D - p0) : KC;
    const bool first = p0 == 0;
    __syncthreads();  // the previous chunk is consumed
    for (int i = threadIdx.x; i < dc * NP; i += blockDim.x) {
      const int p = i / NP, k = i - p * NP;
      const float d = k < N ? dirs[(int64_t)(p0 + p) * N + k] : 0.f;
      sdir[i] = d;
      sm = fmaxf(sm, fabsf(d));
    }
    __syncthreads();
    if constexpr (N <= 4) {
      // two vertices per thread share every direction load
      for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < k0; v += 2 * nt) {
        const int64_t v1 = v + nt;
        const bool has1 = v1 < k0;
        float x0[N], x1[N];
        float r0 = 0.f, r1 = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          x0[i] = coords[v * N + i];
          x1[i] = has1 ? coords[v1 * N + i] : x0[i];
          r0 += fabsf(x0[i]);
          r1 += fabsf(x1[i]);
        }
        float m0 = first ? 0.f : vmax[v], m1 = (first || !has1) ? 0.f : vmax[v1];
        const float4* sd4 = (const float4*)sdir;
#pragma unroll 4
        for (int p = 0; p < dc; ++p) {
          const float4 d = sd4[p];
          const float dv[4] = {d.x, d.y, d.z, d.w};
          float h0 = x0[0] * dv[0], h1 = x1[0] * dv[0];
#pragma unroll
          for (int i = 1; i < N; ++i) {
            h0 = fmaf(x0[i], dv[i], h0);
            h1 = fmaf(x1[i], dv[i], h1);
          }
          m0 = fmaxf(m0, fabsf(h0));
          m1 = fmaxf(m1, fabsf(h1));
        }
        vmax[v] = m0;
        if (has1) vmax[v1] = m1;
        bm = fmaxf(bm, has1 ? fmaxf(m0, m1) : m0);
        br = fmaxf(br, fmaxf(r0, r1));
      }
    } else {
      for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < k0; v += nt) {
        float x[N];
        float r1 = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) { x[i] = coords[v * N + i]; r1 += fabsf(x[i]); }
        float m = first ? 0.f : vmax[v];
        for (int p = 0; p < dc; ++p) {
          float h = x[0] * sdir[p * N];
#pragma unroll
          for (int i = 1; i < N; ++i) h = fmaf(x[i], sdir[p * N + i], h);
          m = fmaxf(m, fabsf(h));
        }
        vmax[v] = m;
        bm = fmaxf(bm, m);
        br = fmaxf(br, r1);
      }
    }
  }
  if (blockIdx.x == 0) {
    for (int o = 16; o; o >>= 1) sm = fmaxf(sm, __shfl_xor_sync(0xffffffffu, sm, o));
    if ((threadIdx.x & 31) == 0) atomicMax(smax_bits, __float_as_uint(sm));
  }
  for (int o = 16; o; o >>= 1) {
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
    br = fmaxf(br, __shfl_xor_sync(0xffffffffu, br, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(m32_bits, __float_as_uint(bm));
    atomicMax(r1_bits, __float_as_uint(br));
  }
}

template <int N>
__global__ void __launch_bounds__(256) k_vmax_pass2(const float* __restrict__ coords, int64_t k0,
                                                    const float* __restrict__ dirs, int D, const float* __restrict__ vmax,
                                                    const unsigned int* __restrict__ m32_bits,
                                                    const unsigned int* __restrict__ r1_bits,
                                                    const unsigned int* __restrict__ smax_bits,
                                                    unsigned long long* __restrict__ m64_bits) {
  const float M32 = __uint_as_float(*m32_bits);
  const float R = __uint_as_float(*r1_bits) * __uint_as_float(*smax_bits);
  const float err = (N + 2) * kEps32 * R * 1.001f + FLT_MIN;
  const float thresh = M32 - 2.f * err;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < k0; v += (int64_t)gridDim.x * blockDim.x) {
    if (vmax[v] < thresh) continue;
    double m = 0.0;
    for (int p = 0; p < D; ++p) {
      double h = __dmul_rn((double)coords[v * N], (double)dirs[p * N]);
      for (int i = 1; i < N; ++i) h = __dadd_rn(h, __dmul_rn((double)coords[v * N + i], (double)dirs[p * N + i]));
      m = fmax(m, fabs(h));
    }
    atomicMax(m64_bits, dbits(m));
  }
}

// ECF: M = max |f| over FVals (exact in fp32, so no refinement)
__global__ void k_absmax_f32(const float* __restrict__ f, int64_t n, unsigned int* __restrict__ bits) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(f[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(bits, __float_as_uint(m));
}

// max |w| of integer weights (sizes the int32 shared-memory partials)
__global__ void k_absmax_i32(const int32_t* __restrict__ w, int64_t n, unsigned int* __restrict__ out) {
  unsigned int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int x = w[i];
    unsigned int a = x < 0 ? 0u - (unsigned int)x : (unsigned int)x;
    m = a > m ? a : m;
  }
  for (int o = 16; o; o >>= 1) { unsigned int t = __shfl_xor_sync(0xffffffffu, m, o); m = t > m ? t : m; }
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// mode 0: WECT (M64 bits + R from pass 1), mode 1: ECF (M32 bits)
__global__ void k_params_complex(int mode, int n, const unsigned long long* __restrict__ m64_bits,
                                 const unsigned int* __restrict__ m32_bits, const unsigned int* __restrict__ r1_bits,
                                 const unsigned int* __restrict__ smax_bits, int T, double maxheight, double lo_in, double hi_in, uint32_t flags,
                                 GridParams* __restrict__ out) {
  GridParams g;
  double Mc = mode == 0 ? __longlong_as_double((long long)*m64_bits) : (double)__uint_as_float(*m32_bits);
  double R = mode == 0 ? (double)__uint_as_float(*r1_bits) * (double)__uint_as_float(*smax_bits) * (1.0 + 1e-6) : Mc;
  g.M = maxheight > 0 ? maxheight : Mc;
  if (lo_in < hi_in) { g.lo = lo_in; g.hi = hi_in; } else { g.lo = -g.M; g.hi = g.M; }
  g.T = T;
  g.Tm1 = (double)(T - 1);
  g.degenerate = !(g.hi > g.lo);
  g.fp32_only = (flags & WECT_FP32_ONLY) ? 1 : 0;
  double A = g.degenerate ? 0.0 : g.Tm1 / (g.hi - g.lo);
  double Bc = -g.lo * A;
  int nn = mode == 0 ? n : 0;
  g.A = (float)A;
  g.B = (float)Bc;
  g.tau = (float)(2.0 * (double)kEps32 * (A * (nn + 2) * R + 2.0 * fabs(Bc) + T + 1.0));
  g.covers = 0;
  *out = g;
}

// ----------------------------------------------------------- index validation
__global__ void k_check_indices(const int32_t* __restrict__ v, int64_t n, int64_t k0, unsigned int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if ((uint32_t)v[i] >= (uint64_t)k0 || v[i] < 0) { atomicOr(flag, 1u); return; }
}

// --------------------------------------------------------------- main kernels
// Flush of a lane-interleaved histogram hist[q * 32 + lane] (lanes = 32 filter rows):
// every lane's atomics hit its own bank, whatever the bins.
template <bool FLOATW, typename Acc>
__device__ __forceinline__ void flush_hist_t(Acc* hist, int T, int row0, int Dc, void* diff) {
  for (int i = threadIdx.x; i < 32 * T; i += blockDim.x) {
    const int q = i >> 5, r = i & 31;
    const Acc val = hist[i];
    if (val != (Acc)0 && row0 + r < Dc) {
      const int64_t o = (int64_t)(row0 + r) * T + q;
      if (FLOATW) atomicAdd((double*)diff + o, (double)val);
      else atomicAdd((unsigned long long*)diff + o, (unsigned long long)(long long)val);
    }
    hist[i] = (Acc)0;
  }
}

// WECT of an explicit complex.  grid = (direction tiles of 32, cell slices); lanes =
// directions, warps = contiguous cell streams.  Cells are taken in batches: the warp
// first gathers a batch's vertex coordinates lane-parallel into a private smem buffer
// (many independent loads in flight), then each lane evaluates the batch against its own
// direction from broadcast reads: h = <x, s> by fp32 FMA (binary64 repair near bin
// edges, reading A1), cell height = max over its vertices (rmax, eq. msi),
// one shared-memory atomic per (cell, direction) (scatter_add).
constexpr int kBatchFloats = 1536;  // per-warp coordinate buffer (6 KB)

// binary64 repair of one cell's bin: exact heights of its vertices (axis order), max,
// alpha64 (reading A1).  Out of line: it runs for ~0.1% of (cell, direction) pairs.
template <int N, int NP>
__device__ __noinline__ int cell_repair(const float* xs, int ar, const float* s, const GridParams* gp) {
  double hm = -DBL_MAX;
  for (int t = 0; t < ar; ++t) {
    double h = __dmul_rn((double)xs[t * NP], (double)s[0]);
    for (int i = 1; i < N; ++i) h = __dadd_rn(h, __dmul_rn((double)xs[t * NP + i], (double)s[i]));
    hm = fmax(hm, h);
  }
  note_repair();
  return alpha64(hm, *gp);
}

__device__ __forceinline__ void red_shared(uint32_t addr, int w) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(w));
}
__device__ __forceinline__ void red_shared(uint32_t addr, float w) { atomicAdd((float*)__cvta_shared_to_generic(addr), w); }

// One batch of nb cells of arity AR (0: runtime arity `arr`) against this lane's direction.
template <int N, int NP, int AR, bool FLOATW, typename Acc>
__device__ __forceinline__ void batch_eval(const float* xb, int nb, unsigned badcells, Acc wl, const float* s,
                                           const GridParams& g, const GridParams* gp, uint32_t hlane, bool active,
                                           int arr = AR) {
  const int ar = AR > 0 ? AR : arr;
  const float A = g.A, Bc = g.B, tau = g.fp32_only ? -1.f : g.tau;
  const int Tm1 = g.T - 1;
  for (int j = 0; j < nb; ++j) {
    const Acc w = __shfl_sync(0xffffffffu, wl, j);
    if ((badcells >> j) & 1u) continue;  // a cell with an out-of-range index is skipped
    const float4* xc = (const float4*)(xb + j * ar * NP);
    float hmax = -FLT_MAX;
#pragma unroll
    for (int t = 0; t < (AR > 0 ? AR : 1); ++t) {
      for (int tt = t; tt < (AR > 0 ? t + 1 : ar); ++tt) {
        float x[NP];
#pragma unroll
        for (int i4 = 0; i4 < NP / 4; ++i4) {
          const float4 q4 = xc[tt * (NP / 4) + i4];  // broadcast LDS.128
          x[4 * i4] = q4.x; x[4 * i4 + 1] = q4.y; x[4 * i4 + 2] = q4.z; x[4 * i4 + 3] = q4.w;
        }
        float h = x[0] * s[0];
#pragma unroll
        for (int i = 1; i < N; ++i) h = fmaf(x[i], s[i], h);
        hmax = fmaxf(hmax, h);
      }
    }
    const float u = fmaf(hmax, A, Bc);
    int bin = __float2int_ru(u);
    if (fabsf(u - rintf(u)) < tau) bin = cell_repair<N, NP>((const float*)xc, ar, s, gp);
    else bin = bin < 0 ? 0 : (bin > Tm1 ? Tm1 : bin);
    if (active && w != (Acc)0) red_shared(hlane + 128u * (uint32_t)bin, w);
  }
}

template <int N, bool FLOATW>
__global__ void __launch_bounds__(256) k_complex(Segs segs, const float* __restrict__ coords, int64_t k0,
                                                 const float* __restrict__ dirs, int d_begin, int Dc,
                                                 const GridParams* __restrict__ gp,
                                                 const unsigned int* __restrict__ wmax_bits, int64_t slice_len,
                                                 int64_t float_chunk, void* __restrict__ diff) {
  using Acc = typename std::conditional<FLOATW, float, int>::type;
  extern __shared__ __align__(16) unsigned char smraw[];
  const GridParams g = *gp;
  const int T = g.T;
  Acc* hist = (Acc*)smraw;  // [T][32] lane-interleaved
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  constexpr int NP = (N + 3) & ~3;  // vertex coordinates padded to whole float4s
  float* xb = (float*)(smraw + (size_t)32 * T * sizeof(Acc)) + warp * kBatchFloats;
  __shared__ Seg ssegs[kMaxSegs];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kMaxSegs; ++i) ssegs[i] = segs.s[i];  // constant indices: no local copy
  }
  for (int i = threadIdx.x; i < 32 * T; i += blockDim.x) hist[i] = (Acc)0;
  const int dl = blockIdx.x * 32 + lane;
  const bool active = dl < Dc;
  const int p = d_begin + (active ? dl : 0);
  const uint32_t hlane = (uint32_t)__cvta_generic_to_shared(hist) + 4u * lane;
  float s[N];
#pragma unroll
  for (int i = 0; i < N; ++i) s[i] = dirs[p * N + i];
  const int64_t c0 = blockIdx.y * slice_len;
  const int64_t c1 = (c0 + slice_len) < segs.total ? (c0 + slice_len) : segs.total;
  const int64_t chunk = chunk_cells(FLOATW, float_chunk, wmax_bits, c1 - c0);
  __syncthreads();
  for (int64_t a0 = c0; a0 < c1; a0 += chunk) {
    const int64_t a1 = (a0 + chunk) < c1 ? (a0 + chunk) : c1;
    const int64_t per = (a1 - a0 + nwarps - 1) / nwarps;
    const int64_t w0 = a0 + warp * per, w1 = (w0 + per) < a1 ? (w0 + per) : a1;
    int seg = 0;
    for (int64_t c = w0; c < w1;) {
      while (c >= ssegs[seg].start + ssegs[seg].count) ++seg;
      const Seg& S = ssegs[seg];
      const int ar = S.arity;
      int nb = kBatchFloats / (ar * NP);
      nb = nb > 32 ? 32 : nb;
      const int64_t lim = S.start + S.count < w1 ? S.start + S.count : w1;
      if (c + nb > lim) nb = (int)(lim - c);
      const int64_t b0 = c - S.start;
      // phase A: lane-parallel gathers of the batch's vertex coordinates
      unsigned badcells = 0;  // bit j: cell j has an out-of-range index
      for (int t = lane; t < nb * ar; t += 32) {
        int v = S.verts ? __ldg(S.verts + b0 * ar + t) : (int)(b0 + t);
        if ((uint64_t)(int64_t)v >= (uint64_t)k0) { badcells |= 1u << (t / ar); v = 0; }
        const float* x = coords + (int64_t)v * N;
#pragma unroll
        for (int i = 0; i < NP; ++i) xb[t * NP + i] = i < N ? __ldg(x + i) : 0.f;
      }
      Acc wl = (Acc)0;
      if (lane < nb) wl = cell_weight<FLOATW, Acc>(S, b0 + lane);
#pragma unroll
      for (int o = 16; o; o >>= 1) badcells |= __shfl_xor_sync(0xffffffffu, badcells, o);
      if (badcells && lane == 0) atomicOr(&g_err_word, 1u);
      __syncwarp();
      // phase B: lanes = directions (arity specialised so the vertex loops unroll)
      switch (ar) {
        case 1: batch_eval<N, NP, 1, FLOATW>(xb, nb, badcells, wl, s, g, gp, hlane, active); break;
        case 2: batch_eval<N, NP, 2, FLOATW>(xb, nb, badcells, wl, s, g, gp, hlane, active); break;
        case 3: batch_eval<N, NP, 3, FLOATW>(xb, nb, badcells, wl, s, g, gp, hlane, active); break;
        case 4: batch_eval<N, NP, 4, FLOATW>(xb, nb, badcells, wl, s, g, gp, hlane, active); break;
        case 5: batch_eval<N, NP, 5, FLOATW>(xb, nb, badcells, wl, s, g, gp, hlane, active); break;
        case 8: batch_eval<N, NP, 8, FLOATW>(xb, nb, badcells, wl, s, g, gp, hlane, active); break;
        default: batch_eval<N, NP, 0, FLOATW>(xb, nb, badcells, wl, s, g, gp, hlane, active, ar); break;
      }
      __syncwarp();
      c += nb;
    }
    __syncthreads();
    flush_hist_t<FLOATW, Acc>(hist, T, blockIdx.x * 32, Dc, diff);
    __syncthreads();
  }
}

// ------------------------------------------------------------ cumsum epilogue
// Alg. 1 line 11: one warp per row, 32-wide shuffle scan with carry.
template <typename In, typename Out>
__global__ void k_finalize(const In* __restrict__ diff, int64_t rows, int T, Out* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const In* d = diff + row * T;
  Out* o = out + row * T;
  In carry = 0;
  for (int q0 = 0; q0 < T; q0 += 32) {
    In x = (q0 + lane < T) ? d[q0 + lane] : (In)0;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      In y = __shfl_up_sync(0xffffffffu, x, k);
      if (lane >= k) x += y;
    }
    x += carry;
    if (q0 + lane < T) o[q0 + lane] = (Out)x;
    carry = __shfl_sync(0xffffffffu, x, 31);
  }
}

// ------------------------------------------------------------------ launchers

template <int N>
static wect_status launch_complex_n(bool floatw, const Segs& segs, const float* coords, int64_t k0, const float* dirs,
                                    int d_begin, int Dc, int T, const GridParams* gp, const unsigned int* wmax,
                                    void* diff, cudaStream_t st, int num_sms) {
  const int tiles = (Dc + 31) / 32;
  const size_t smem = (size_t)32 * T * 4 + (size_t)8 * kBatchFloats * 4;
  int per_sm = (int)((220 * 1024) / (smem + 2048));
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const int64_t slice = pick_slice(segs.total, tiles, per_sm, num_sms, (int64_t)1 << 20);
  dim3 grid(tiles, (unsigned)((segs.total + slice - 1) / slice));
  MainTimer timer(st);
  if (floatw) {
    auto k = k_complex<N, true>;
    WECT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, st>>>(segs, coords, k0, dirs, d_begin, Dc, gp, wmax, slice, 4096, diff);
  } else {
    auto k = k_complex<N, false>;
    WECT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, st>>>(segs, coords, k0, dirs, d_begin, Dc, gp, wmax, slice, 4096, diff);
  }
  count_launch();
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_cells(int mode, int n, bool floatw, const Segs& segs, int64_t k0, const float* fvals, int m,
                         const float* coords, const float* dirs, int d_begin, int Dc, int T, const GridParams* gp,
                         const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms);
constexpr int kCellTile = 8;  // filters per CTA of the thread-per-cell kernels (k_cells.cu)
bool vb_supported(int T);
wect_status launch_stream(int mode, int n, bool floatw, const Segs& segs, int64_t k0, const float* fvals, int m,
                          const float* coords, const float* dirs, int d_begin, int Dc, int T, const GridParams* gp,
                          const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms);
wect_status launch_complex_vb(int n, bool floatw, const Segs& segs, const float* coords, int64_t k0,
                              const float* dirs, int d_begin, int Dc, int T, const GridParams* gp,
                              const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms);

wect_status launch_absmax_i32(const int32_t* w, int64_t n, unsigned int* out, cudaStream_t st, int num_sms);

// max|w| over the integer weight arrays into the (zeroed) device word *wmax: the int32
// partial-flush bound of k_cells / k_cells_vb / k_complex.  (k_stream checks its weights per
// unit in-kernel instead, so the streaming path skips this pass over the weights.)
static wect_status ensure_wmax(bool floatw, const Segs& segs, const unsigned int* wmax, cudaStream_t st,
                               int num_sms) {
  if (floatw) return WECT_OK;
  for (int i = 0; i < segs.nseg; ++i)
    if (segs.s[i].weights) {
      const wect_status s = launch_absmax_i32((const int32_t*)segs.s[i].weights, segs.s[i].count,
                                              const_cast<unsigned int*>(wmax), st, num_sms);
      if (s != WECT_OK) return s;
    }
  return WECT_OK;
}

wect_status launch_complex(int mode, int n, bool floatw, const Segs& segs, const float* coords, int64_t k0,
                           const float* fsrc, int m_or_D, int d_begin, int Dc, int T, const GridParams* gp,
                           const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms) {
  if (mode == 1 || Dc <= 3 * kCellTile) {  // ECF, or D <= 24: streaming passes (tiles of 8 filters), thread per cell
    const wect_status s = launch_stream(mode, n, floatw, segs, k0, fsrc, m_or_D, coords, fsrc, d_begin, Dc, T, gp,
                                        nullptr, diff, st, num_sms);
    if (s != WECT_ENOTSUP) return s;
    const wect_status sw = ensure_wmax(floatw, segs, wmax, st, num_sms);
    if (sw != WECT_OK) return sw;
    return launch_cells(mode, n, floatw, segs, k0, fsrc, m_or_D, coords, fsrc, d_begin, Dc, T, gp, wmax, diff, st,
                        num_sms);
  }
  {
    const wect_status sw = ensure_wmax(floatw, segs, wmax, st, num_sms);
    if (sw != WECT_OK) return sw;
  }
  if (vb_supported(T) && !getenv("WECT_DISABLE_VB")) {  // vertex bins once per tile, cells from packed rows
    const wect_status s = launch_complex_vb(n, floatw, segs, coords, k0, fsrc, d_begin, Dc, T, gp, wmax, diff, st,
                                            num_sms);
    if (s != WECT_ENOTSUP) return s;
  }
  switch (n) {
#define WECT_CASE(NN) \
  case NN: return launch_complex_n<NN>(floatw, segs, coords, k0, fsrc, d_begin, Dc, T, gp, wmax, diff, st, num_sms);
    WECT_CASE(1) WECT_CASE(2) WECT_CASE(3) WECT_CASE(4) WECT_CASE(5) WECT_CASE(6) WECT_CASE(7) WECT_CASE(8)
#undef WECT_CASE
  }
  return fail(WECT_EINVAL, "ambient dimension n=%d outside [1,8]", n);
}

template <int N>
static wect_status launch_vmax_n(const float* coords, int64_t k0, const float* dirs, int D, float* vmax,
                                 unsigned int* m32, unsigned int* r1, unsigned int* smax, unsigned long long* m64,
                                 cudaStream_t st, int num_sms) {
  int blocks = (int)((k0 + 255) / 256);
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  if (blocks < 1) blocks = 1;
  const size_t smem = (size_t)(D < kVmaxChunk ? D : kVmaxChunk) * (N <= 4 ? 4 : N) * sizeof(float);
  if (smem > 48 * 1024) WECT_CUDA_TRY(cudaFuncSetAttribute(k_vmax_pass1<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_vmax_pass1<N><<<blocks, 256, smem, st>>>(coords, k0, dirs, D, vmax, m32, r1, smax); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  k_vmax_pass2<N><<<blocks, 256, 0, st>>>(coords, k0, dirs, D, vmax, m32, r1, smax, m64); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_vmax(int n, const float* coords, int64_t k0, const float* dirs, int D, float* vmax,
                        unsigned int* m32, unsigned int* r1, unsigned int* smax, unsigned long long* m64, cudaStream_t st,
                        int num_sms) {
  switch (n) {
#define WECT_CASE(NN) \
  case NN: return launch_vmax_n<NN>(coords, k0, dirs, D, vmax, m32, r1, smax, m64, st, num_sms);
    WECT_CASE(1) WECT_CASE(2) WECT_CASE(3) WECT_CASE(4) WECT_CASE(5) WECT_CASE(6) WECT_CASE(7) WECT_CASE(8)
#undef WECT_CASE
  }
  return fail(WECT_EINVAL, "ambient dimension n=%d outside [1,8]", n);
}

wect_status launch_complex_params(int mode, int n, const unsigned long long* m64, const unsigned int* m32,
                                  const unsigned int* r1, const unsigned int* smax, const wect_grid& grid,
                                  GridParams* gp, cudaStream_t st) {
  k_params_complex<<<1, 1, 0, st>>>(mode, n, m64, m32, r1, smax, grid.T, grid.maxheight, grid.lo, grid.hi,
                                    grid.flags, gp); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_absmax_f32(const float* f, int64_t n, unsigned int* bits, cudaStream_t st, int num_sms) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  if (blocks < 1) blocks = 1;
  k_absmax_f32<<<blocks, 256, 0, st>>>(f, n, bits); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_absmax_i32(const int32_t* w, int64_t n, unsigned int* out, cudaStream_t st, int num_sms) {
  if (n <= 0) return WECT_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  k_absmax_i32<<<blocks, 256, 0, st>>>(w, n, out); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_check_indices(const int32_t* v, int64_t n, int64_t k0, unsigned int* flag, cudaStream_t st,
                                 int num_sms) {
  if (n <= 0) return WECT_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  k_check_indices<<<blocks, 256, 0, st>>>(v, n, k0, flag); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_finalize(const void* diff, bool is_float, int64_t rows, int T, void* out, wect_dtype odtype,
                            cudaStream_t st) {
  if (rows <= 0) return WECT_OK;
  const int wpb = 8;
  const unsigned blocks = (unsigned)((rows + wpb - 1) / wpb);
  if (is_float) {
    k_finalize<double, double><<<blocks, wpb * 32, 0, st>>>((const double*)diff, rows, T, (double*)out); count_launch();
  } else if (odtype == WECT_I32) {
    k_finalize<long long, int><<<blocks, wpb * 32, 0, st>>>((const long long*)diff, rows, T, (int*)out); count_launch();
  } else {
    k_finalize<long long, long long><<<blocks, wpb * 32, 0, st>>>((const long long*)diff, rows, T, (long long*)out); count_launch();
  }
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

}  // namespace wect
