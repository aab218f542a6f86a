// k_grad.cu -- gradient of a scalar loss through the WECT / WECFs with respect to the
// weights (wect_complex_backward, ecf_complex_backward).
//
// The paper's framework is differentiable with respect to the weights (P:114-115,
// P:493-494).  Alg. 1 is linear in the weights:
//   out[p, q] = sum over cells s of w(s) (-1)^dim s [bin(s, p) <= q]     (closed form P:769-776)
// so for G = dL/dout,
//   dL/dw(s) = (-1)^dim s * sum_p RC[p, bin(s, p)],   RC[p, q] = sum_{q' >= q} G[p, q'].
// (Heights / coordinates enter only through the piecewise-constant bins: gradient 0 a.e.)
//
// Passes: k_rcumsum (RC, one thread per row, q from T-1 down); per tile of 64 filters the
// exact vertex-bin table VB (k_vbins of the forward for directions, k_vbins_f here for
// given filter values); then k_grad_cells twice per tile (32 filters each, one per lane):
// a warp takes 16 cells, the cell bin per lane is the max of its vertices' VB entries
// (eq. msi, exact because alpha is monotone), each lane gathers RC[bin] from a
// shared-memory tile, and a 31-shuffle transpose-reduction leaves lanes 2c, 2c+1 with
// cell c's sum over the 32 filters.  Tiles add into the fp64 gradient in a fixed order, so the
// result is deterministic.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace wect {

constexpr int kGradWarps = 16;  // one 512-thread CTA per SM shares the RC tile


__global__ void k_rcumsum(const double* __restrict__ G, int64_t rows, int T, double* __restrict__ RC) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double acc = 0.0;
  for (int q = T - 1; q >= 0; --q) {
    acc = __dadd_rn(acc, G[r * T + q]);
    RC[r * T + q] = acc;
  }
}

// VB rows for given filter values (ECF): VB[v] word l = alpha(f[v, p0+2l]) | alpha(f[v, p0+2l+1]) << 16,
// alpha in binary64 on the fp32 value (reading A1; no fast path needed here).
__global__ void __launch_bounds__(256) k_vbins_f(const float* __restrict__ f, int64_t k0, int m, int p0, int np,
                                                 const GridParams* __restrict__ gp, uint32_t* __restrict__ vb) {
  const GridParams g = *gp;
  const int lane = threadIdx.x & 31;
  const int pa = 2 * lane, pb = 2 * lane + 1;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < k0; v += nwarps) {
    const int ba = pa < np ? alpha64((double)__ldg(f + v * m + p0 + pa), g) : 0;
    const int bb = pb < np ? alpha64((double)__ldg(f + v * m + p0 + pb), g) : 0;
    vb[v * 32 + lane] = (uint32_t)ba | ((uint32_t)bb << 16);
  }
}

// Recursive halving over 16 per-lane values v[c] (c = cell of the batch): after the
// offsets 16, 8, 4, 2 lane l holds the partial sum of cell l >> 1 over half of the lanes,
// and the last xor-1 step completes it in both lanes 2c and 2c + 1 (16 + 8 + 4 + 2 + 1
// shuffles for 16 cells).
__device__ __forceinline__ double transpose_reduce16(double (&v)[16], int lane) {
#pragma unroll
  for (int o = 16, n = 8; o >= 2; o >>= 1, n >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const double send = up ? v[k] : v[k + n];
      const double keep = up ? v[k + n] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// One pass: filters [row0, row0 + np) of the tile (np <= 32), lane = filter; batches of
// 16 cells, 8 cells x AR VB loads in flight at a time (AR = 0: runtime arity <= 8).
template <bool SMEM_RC, bool PAIR, int AR>
__device__ __forceinline__ void grad_segment(const Seg& S, double* __restrict__ go, int64_t k0,
                                             const uint16_t* __restrict__ vb16, int np, const double* __restrict__ rcs,
                                             const double* __restrict__ RC, int row0, int T, int first, int64_t gw,
                                             int64_t nwarps, int lane) {
  constexpr int MA = AR > 0 ? AR : 8;
  const int ar = AR > 0 ? AR : S.arity;
  for (int64_t base = gw * 16; base < S.count; base += nwarps * 16) {
    const int64_t mycell = base + (lane & 15);
    int ids[MA];
#pragma unroll
    for (int j = 0; j < MA; ++j) {
      int id = 0;
      if (j < ar && mycell < S.count) {
        id = S.verts ? __ldg(S.verts + mycell * ar + j) : (int)mycell;
        if ((unsigned)id >= (unsigned)k0) {
          if (lane < 16) atomicOr(&g_err_word, 1u);
          id = -1;
        }
      }
      ids[j] = id;
    }
    double v[16];
#pragma unroll
    for (int c0 = 0; c0 < 16; c0 += 8) {
      int b[8][MA];
      bool ok[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        ok[c] = true;
#pragma unroll
        for (int j = 0; j < MA; ++j) {
          if (AR == 0 && j >= ar) { b[c][j] = 0; continue; }
          const int id = __shfl_sync(0xffffffffu, ids[j], c0 + c);
          ok[c] &= id >= 0;
          // PAIR: the lane's two directions (2 lane, 2 lane + 1) as one u16x2 word of the row
          b[c][j] = PAIR ? (int)__ldg((const uint32_t*)vb16 + (int64_t)(id < 0 ? 0 : id) * 32)
                         : (int)__ldg(vb16 + (int64_t)(id < 0 ? 0 : id) * 64);
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double x = 0.0;
        if (PAIR) {  // SMEM_RC is implied: rcs[q][half][32]
          uint32_t m2 = (uint32_t)b[c][0];
#pragma unroll
          for (int j = 1; j < MA; ++j) m2 = __vmaxu2(m2, (uint32_t)b[c][j]);
          if (ok[c]) x = rcs[(m2 & 0xFFFFu) * 64 + lane] + rcs[(m2 >> 16) * 64 + 32 + lane];
        } else {
          int bin = b[c][0];
#pragma unroll
          for (int j = 1; j < MA; ++j) bin = max(bin, b[c][j]);
          if (ok[c] && lane < np) x = SMEM_RC ? rcs[bin * 32 + lane] : __ldg(RC + (int64_t)(row0 + lane) * T + bin);
        }
        v[c0 + c] = x;
      }
    }
    const double sum = transpose_reduce16(v, lane);
    const int64_t cell = base + (lane >> 1);
    if ((lane & 1) == 0 && cell < S.count) {
      const double gcell = S.sign < 0 ? -sum : sum;
      go[cell] = first ? gcell : go[cell] + gcell;
    }
  }
}

// PAIR (T small enough for a [T][2][32] fp64 tile): one pass per 64-filter tile, lane =
// filters (2 lane, 2 lane + 1); otherwise two passes of 32 (half), lane = filter.
template <bool SMEM_RC, bool PAIR>
__global__ void __launch_bounds__(kGradWarps * 32, 1) k_grad_cells(Segs segs, int64_t k0, const uint32_t* __restrict__ vb,
                                                                   int half, int np, const double* __restrict__ RC,
                                                                   int row0, int T, GradOut gout, int first) {
  extern __shared__ __align__(16) double rcs[];  // [T][32], PAIR: [T][2][32] (column half * 32 + l = filter 2 l + half)
  const int lane = threadIdx.x & 31;
  if (PAIR) {
    for (int i = threadIdx.x; i < T * 64; i += blockDim.x) {
      const int q = i >> 6, col = i & 63, f = 2 * (col & 31) + (col >> 5);
      rcs[i] = f < np ? RC[(int64_t)(row0 + f) * T + q] : 0.0;
    }
    __syncthreads();
  } else if (SMEM_RC) {
    for (int i = threadIdx.x; i < T * 32; i += blockDim.x) {
      const int q = i >> 5, l = i & 31;
      rcs[i] = l < np ? RC[(int64_t)(row0 + l) * T + q] : 0.0;
    }
    __syncthreads();
  }
  const uint16_t* vb16 = PAIR ? (const uint16_t*)(vb + lane) : (const uint16_t*)vb + half * 32 + lane;
  const int64_t gw = (int64_t)blockIdx.x * kGradWarps + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kGradWarps;
  for (int si = 0; si < segs.nseg; ++si) {
    const Seg S = segs.s[si];
    double* go = gout.g[si];
    if (!go || S.count == 0) continue;
    switch (S.arity) {
      case 1: grad_segment<SMEM_RC, PAIR, 1>(S, go, k0, vb16, np, rcs, RC, row0, T, first, gw, nwarps, lane); break;
      case 2: grad_segment<SMEM_RC, PAIR, 2>(S, go, k0, vb16, np, rcs, RC, row0, T, first, gw, nwarps, lane); break;
      case 3: grad_segment<SMEM_RC, PAIR, 3>(S, go, k0, vb16, np, rcs, RC, row0, T, first, gw, nwarps, lane); break;
      case 4: grad_segment<SMEM_RC, PAIR, 4>(S, go, k0, vb16, np, rcs, RC, row0, T, first, gw, nwarps, lane); break;
      default: grad_segment<SMEM_RC, PAIR, 0>(S, go, k0, vb16, np, rcs, RC, row0, T, first, gw, nwarps, lane); break;
    }
  }
}

// ---------------------------------------------------------------------------
wect_status launch_vbins_tile(int n, const float* coords, int64_t k0, const float* dirs, int p0, int np,
                              const GridParams* gp, uint32_t* vb, cudaStream_t st, int num_sms);

wect_status launch_complex_grad(int mode, int n, const Segs& segs, const float* coords, int64_t k0, const float* fsrc,
                                int m_or_D, int d_begin, int Dc, int T, const GridParams* gp, const double* G,
                                const GradOut& gout, cudaStream_t st, int num_sms) {
  for (int i = 0; i < segs.nseg; ++i)
    if (segs.s[i].arity > 8) return fail(WECT_ENOTSUP, "backward supports cells of arity <= 8");
  AsyncScratch mem(st);  // freed on every return path
  double* RC = nullptr;
  uint32_t* vb = nullptr;
  WECT_CUDA_TRY(mem.alloc(&RC, (size_t)Dc * T * sizeof(double)));
  WECT_CUDA_TRY(mem.alloc(&vb, (size_t)(k0 > 0 ? k0 : 1) * 32 * sizeof(uint32_t)));
  k_rcumsum<<<(unsigned)((Dc + 127) / 128), 128, 0, st>>>(G, Dc, T, RC); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  const size_t smem = (size_t)T * 32 * sizeof(double);
  const bool use_smem = smem <= 160 * 1024;
  const bool pair = 2 * smem <= 160 * 1024 && !getenv("WECT_GRAD_NOPAIR");
  if (pair) {
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_grad_cells<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * smem)));
  } else if (use_smem) {
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_grad_cells<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  int64_t maxc = 0;
  for (int i = 0; i < segs.nseg; ++i) maxc = segs.s[i].count > maxc ? segs.s[i].count : maxc;
  int64_t want = (maxc + 16 * kGradWarps - 1) / (16 * kGradWarps);
  const size_t esm = pair ? 2 * smem : smem;
  const int per_sm = use_smem ? (int)((200 * 1024) / esm > 2 ? 2 : ((200 * 1024) / esm < 1 ? 1 : (200 * 1024) / esm)) : 2;
  const int ctas = (int)(want < (int64_t)num_sms * per_sm ? (want < 1 ? 1 : want) : (int64_t)num_sms * per_sm);
  wect_status s = WECT_OK;
  for (int t0 = 0; t0 < Dc && s == WECT_OK; t0 += 64) {
    const int np = (Dc - t0) < 64 ? (Dc - t0) : 64;
    if (mode == 0) {
      s = launch_vbins_tile(n, coords, k0, fsrc, d_begin + t0, np, gp, vb, st, num_sms);
      if (s != WECT_OK) break;
    } else {
      int vblocks = (int)((k0 + 7) / 8);
      vblocks = vblocks > num_sms * 16 ? num_sms * 16 : (vblocks < 1 ? 1 : vblocks);
      k_vbins_f<<<vblocks, 256, 0, st>>>(fsrc, k0, m_or_D, d_begin + t0, np, gp, vb); count_launch();
    }
    if (pair) {
      MainTimer timer(st);
      k_grad_cells<true, true><<<ctas, kGradWarps * 32, 2 * smem, st>>>(segs, k0, vb, 0, np, RC, t0, T, gout,
                                                                         t0 == 0 ? 1 : 0);
      count_launch();
      timer.stop();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) s = fail_cuda(e, "k_grad_cells", __FILE__, __LINE__);
      continue;
    }
    for (int half = 0; half < 2; ++half) {
      const int nph = np - 32 * half;
      if (nph <= 0) break;
      const int first = (t0 == 0 && half == 0) ? 1 : 0;
      MainTimer timer(st);
      if (use_smem)
        k_grad_cells<true, false><<<ctas, kGradWarps * 32, smem, st>>>(segs, k0, vb, half, nph < 32 ? nph : 32, RC,
                                                               t0 + 32 * half, T, gout, first);
      else
        k_grad_cells<false, false><<<ctas, kGradWarps * 32, 0, st>>>(segs, k0, vb, half, nph < 32 ? nph : 32, RC,
                                                             t0 + 32 * half, T, gout, first);
      count_launch();
      timer.stop();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) s = fail_cuda(e, "k_grad_cells", __FILE__, __LINE__);
    }
  }
  return s;
}

}  // namespace wect
