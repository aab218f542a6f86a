// k_images.cu -- implicit image / voxel cubical complexes (wect_images).
//
// Cells are never listed in memory (north_star): every axis-aligned unit i-cube of
// the pixel grid is a cell of sign (-1)^i whose weight is the max of its corners
// (readings A5, A7).
//
// Exact regrouping: for a direction s, a cell's
// height is the height of ONE designated corner -- per extended axis k, the upper
// index when s_k > 0, else the lower -- because the height evaluation (fp32 fast
// path and the binary64 repair alike) is monotone in each coordinate.  So per
// direction every cell lands in the bin of its designated corner, and all cells
// designating vertex v can be summed first into one combined weight cw_o(v), o the
// orthant of s.  |cw| <= 255 in 2D, <= 1020 in 3D.
//
// Two kernels:
//  * k_sweep2d (MNIST-shaped batches, H*W <= 1024): image-independent geometry is
//    preprocessed once per call into, per direction, the vertices sorted by bin
//    (counting sort, k_sort2d).  A CTA then holds 64 images' cw (biased u16, two
//    images per 32-bit word) in shared memory and each warp sweeps one direction:
//    lane l accumulates images 2l, 2l+1 in sorted order and emits the running sum at
//    every bin end.  That running sum IS the cumsum of the difference histogram
//    (Alg. 1 lines 4-11) -- no atomics, no separate scan, exact int32.
//  * k_grid_hist (volumes, large images): lanes = 32 directions, warps stream
//    voxels, shared-memory int32 histograms [32][T+1], one int64 merge per CTA,
//    then k_finalize's cumsum.
#include <cstdio>

#include "common.cuh"

namespace wect {

// ---------------------------------------------------------------------------
// Grid parameters: M = max |h| over the 2^ndim bounding-box corners and ALL D
// directions (reading A2: the binary64 height is monotone per coordinate, so the
// max over the grid is attained at a corner), plus the fp32 guard tau.
// ---------------------------------------------------------------------------
__global__ void k_grid_params(int ndim, int64_t d0, int64_t d1, int64_t d2, const float* __restrict__ dirs,
                              int D, int T, double maxheight, double lo_in, double hi_in, uint32_t flags,
                              GridParams* __restrict__ out) {
  __shared__ double red[256];
  __shared__ float sred[256];
  int64_t dims[3] = {d0, d1, d2};
  int maxd = 1;
  for (int i = 0; i < ndim; ++i) maxd = dims[i] > maxd ? (int)dims[i] : maxd;
  double S = (double)(maxd - 1 > 1 ? maxd - 1 : 1);
  // axis k <-> grid dim ndim-1-k
  float lo_c[3], hi_c[3];
  float R1 = 0.f;
  for (int k = 0; k < ndim; ++k) {
    int L = (int)dims[ndim - 1 - k];
    lo_c[k] = axis_coord(0, L, S);
    hi_c[k] = axis_coord(L - 1, L, S);
    R1 += fmaxf(fabsf(lo_c[k]), fabsf(hi_c[k]));
  }
  double M = 0.0;
  float smax = 0.f;
  int ncorner = 1 << ndim;
  for (int idx = threadIdx.x; idx < D * ncorner; idx += blockDim.x) {
    int p = idx / ncorner, c = idx % ncorner;
    double h = 0.0;
    for (int k = 0; k < ndim; ++k) {
      double x = (double)(((c >> k) & 1) ? hi_c[k] : lo_c[k]);
      double prod = __dmul_rn(x, (double)dirs[p * ndim + k]);
      h = (k == 0) ? prod : __dadd_rn(h, prod);
      smax = fmaxf(smax, fabsf(dirs[p * ndim + k]));
    }
    M = fmax(M, fabs(h));
  }
  red[threadIdx.x] = M;
  sred[threadIdx.x] = smax;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
      sred[threadIdx.x] = fmaxf(sred[threadIdx.x], sred[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    GridParams g;
    g.M = maxheight > 0 ? maxheight : red[0];
    if (lo_in < hi_in) { g.lo = lo_in; g.hi = hi_in; } else { g.lo = -g.M; g.hi = g.M; }
    g.T = T;
    g.Tm1 = (double)(T - 1);
    g.degenerate = !(g.hi > g.lo);
    g.fp32_only = (flags & WECT_FP32_ONLY) ? 1 : 0;
    double A = g.degenerate ? 0.0 : g.Tm1 / (g.hi - g.lo);
    double Bc = -g.lo * A;
    double R = (double)R1 * (double)sred[0] * (1.0 + 1e-6);
    g.A = (float)A;
    g.B = (float)Bc;
    g.tau = (float)(2.0 * (double)kEps32 * (A * (ndim + 2) * R + 2.0 * fabs(Bc) + T + 1.0));
    g.pad = 0;
    *out = g;
  }
}

// ---------------------------------------------------------------------------
// Per local direction: exact bins of all H*W vertices (binary64, alpha64), counting
// sort by bin, and the direction's SWEEP PROGRAM:
//   off[k]  : packets of four u32 byte offsets (id * 128) into the cw table, k < npk;
//             each bin's ids are padded to whole packets with the padding row HW
//             (packed value 0, i.e. weight 0)
//   meta[g]  : one byte per packet of group g (4 packets): bit 0 set on every packet that
//              carries metadata (informational), bits 1..7 emit = number of bins whose
//              value is the running total after this packet (bin q with z empty bins
//              after it emits 1 + z; leading empty bins and emits > kMaxEmit ride on
//              all-padding packets).
//              Loaded with the packets, so no dependent load sits on the run-end path.
// Also records the direction's quadrant o = (s_x > 0) | (s_y > 0) << 1 in qlist.
// ---------------------------------------------------------------------------

constexpr int kMaxEmit = 127;    // emit field of a packet's metadata byte

__host__ __device__ constexpr int sweep_prog_packets(int HW, int T) { return (HW / 4 + T + T / kMaxEmit + 16 + 15) & ~15; }
// u32 words per direction: [off: 4 per packet][meta: 1 per group of 4 packets]
__host__ __device__ constexpr int sweep_prog_words(int HW, int T) {
  return 4 * sweep_prog_packets(HW, T) + sweep_prog_packets(HW, T) / 4;
}

// Freudenthal designated vertex (offset index: 0 self, 1 X = (r,c+1), 2 Y = (r+1,c),
// 3 D = (r+1,c+1)) of simplex type t (1 e_x, 2 e_y, 3 e_diag, 4 U, 5 L) in chamber (A, B, C)
// = (s_x > 0, s_y > 0, s_x + s_y > 0); its vertex set as a bit mask over {self, X, Y, D}.
__host__ __device__ __forceinline__ int freud_des(int t, int A, int B, int C) {
  switch (t) {
    case 1: return A ? 1 : 0;
    case 2: return B ? 2 : 0;
    case 3: return C ? 3 : 0;
    case 4: return (B && C) ? 3 : ((A && !B) ? 1 : 0);
    case 5: return (A && C) ? 3 : ((B && !A) ? 2 : 0);
  }
  return 0;
}
__host__ __device__ __forceinline__ int freud_mask(int t) {
  constexpr int m[6] = {0x1, 0x3, 0x5, 0x9, 0xB, 0xD};
  return m[t];
}

__global__ void __launch_bounds__(256) k_sort2d(int H, int W, const float* __restrict__ dirs, int d_begin, int Dc,
                                                const GridParams* __restrict__ gp, uint32_t* __restrict__ prog,
                                                int* __restrict__ prog_len, int* __restrict__ qlist,
                                                int* __restrict__ qcount, int freud, int4* __restrict__ corr,
                                                int* __restrict__ ncorr, int corr_cap) {
  // smem: counts[T], base[T], meta[Lp] (emit | flag << 16), vbin[HW] (u16)
  extern __shared__ int sh[];
  const GridParams g = *gp;
  const int T = g.T, HW = H * W, dl = blockIdx.x, p = d_begin + dl;
  const int Lp = sweep_prog_packets(HW, T);
  int* counts = sh;
  int* base = sh + T;
  int* meta = sh + 2 * T;
  uint16_t* vbin = (uint16_t*)(sh + 2 * T + Lp);
  __shared__ int npk_total;
  uint32_t* off = prog + (int64_t)dl * sweep_prog_words(HW, T);
  for (int q = threadIdx.x; q < T; q += blockDim.x) counts[q] = 0;
  for (int k = threadIdx.x; k < Lp; k += blockDim.x) meta[k] = 0;
  for (int k = threadIdx.x; k < 4 * Lp; k += blockDim.x) off[k] = (uint32_t)HW * 128u;  // padding row
  const float sx = dirs[2 * p], sy = dirs[2 * p + 1];
  int maxd = H > W ? H : W;
  double S = (double)(maxd - 1 > 1 ? maxd - 1 : 1);
  __syncthreads();
  for (int v = threadIdx.x; v < HW; v += blockDim.x) {
    int r = v / W, c = v % W;
    double h = __dadd_rn(__dmul_rn((double)axis_coord(c, W, S), (double)sx), __dmul_rn((double)axis_coord(r, H, S), (double)sy));
    int bq = alpha64(h, g);
    vbin[v] = (uint16_t)bq;
    atomicAdd(&counts[bq], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // serial over bins: packet bases and per-packet metadata
    int pk = 0, q = 0;
    while (q < T && counts[q] == 0) ++q;
    for (int lead = q; lead > 0;) {  // leading empty bins: all-padding packets
      const int e = lead < kMaxEmit ? lead : kMaxEmit;
      meta[pk++] = e | (1 << 16);
      lead -= e;
    }
    while (q < T) {
      int q2 = q + 1;
      while (q2 < T && counts[q2] == 0) ++q2;
      const int npk = (counts[q] + 3) / 4;
      base[q] = pk;
      int emit = q2 - q;
      int e = emit < kMaxEmit ? emit : kMaxEmit;
      meta[pk + npk - 1] = e | (1 << 16);
      pk += npk;
      for (emit -= e; emit > 0; emit -= e) {  // long gaps: all-padding packets
        e = emit < kMaxEmit ? emit : kMaxEmit;
        meta[pk++] = e | (1 << 16);
      }
      q = q2;
    }
    pk = (pk + 3) & ~3;  // whole groups of 4 packets (the tail packets are padding, no flags)
    npk_total = pk;
    prog_len[dl] = pk;
    // cubical: quadrant (s_x > 0) | (s_y > 0) << 1; Freudenthal: chamber | (s_x + s_y > 0) << 2
    int o = (sx > 0.f ? 1 : 0) | (sy > 0.f ? 2 : 0) | ((freud && sx + sy > 0.f) ? 4 : 0);
    int slot = atomicAdd(&qcount[o], 1);
    qlist[o * Dc + slot] = dl;
  }
  __syncthreads();
  if (freud) {
    // Simplices whose chamber-designated vertex does not carry the simplex's max exact bin
    // (only possible through the rounded diagonal comparison): the sweep counts them from
    // bin lo = vbin[designated]; record [lo, hi) so k_sweep_fix moves them to hi.
    const int A = sx > 0.f, B = sy > 0.f, C = (sx + sy) > 0.f;
    for (int i = threadIdx.x; i < 5 * HW; i += blockDim.x) {
      const int u = i / 5, t = 1 + (i - u * 5), r = u / W, c = u - r * W;
      const bool rt = c + 1 < W, dn = r + 1 < H;
      if ((t == 1 && !rt) || (t == 2 && !dn) || (t >= 3 && !(rt && dn))) continue;
      const int off[4] = {0, 1, W, W + 1};
      const int mask = freud_mask(t);
      int hi = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (mask >> k & 1) hi = max(hi, (int)vbin[u + off[k]]);
      const int lo = vbin[u + off[freud_des(t, A, B, C)]];
      if (hi > lo) {
        const int slot = atomicAdd(ncorr, 1);
        if (slot < corr_cap) corr[slot] = make_int4(dl, u, t, lo | (hi << 16));
      }
    }
  }
  for (int v = threadIdx.x; v < HW; v += blockDim.x) {  // ids: any order within a bin
    const int bq = vbin[v];
    const int r = atomicAdd(&counts[bq], -1) - 1;
    off[4 * base[bq] + r] = (uint32_t)v * 128u;
  }
  const int npk = npk_total;
  uint32_t* metaw = off + 4 * Lp;
  for (int g = threadIdx.x; g < npk / 4; g += blockDim.x) {
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = meta[4 * g + j];
      w |= (uint32_t)(((m & 0xFFFF) << 1) | (m >> 16)) << (8 * j);
    }
    metaw[g] = w;
  }
}

constexpr int kSweepWarps = 16;
constexpr int kSweepImgs = 64;   // images per CTA group: lane l owns images 2l, 2l+1
constexpr int kStageBins = 8;    // bins per staged output chunk
constexpr int kStageStride = 68; // words per staged bin row (68 = 4 mod 32: conflict-free readout)
constexpr int kPixStride = 68;   // bytes per staged pixel row (17 words: conflict-free transpose)

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ constexpr size_t sweep_pix_bytes(int HW) { return align16((size_t)HW * kPixStride); }
// per-warp private area: its direction's sorted vertex ids and bin ends, and the output stage
__host__ __device__ constexpr size_t sweep_warp_bytes(int HW, int T) {
  return (size_t)kStageBins * kStageStride * 4;  // output stage only: programs are read from L2
}
// cwb has HW + 1 rows: row HW is the padding row (bias = weight 0)
__host__ __device__ constexpr size_t sweep_smem_bytes(int HW, int T) {
  return align16((size_t)(HW + 1) * 128) + sweep_pix_bytes(HW) + (size_t)kSweepWarps * sweep_warp_bytes(HW, T);
}

template <typename OutT>
__device__ __forceinline__ void sweep_store_chunk(const int* __restrict__ st, OutT* __restrict__ out, int64_t img0,
                                                  int nimg, int Dc, int dl, int T, int qc, int lane) {
  const int nb = (T - qc) < kStageBins ? (T - qc) : kStageBins;
  if (nb == kStageBins && (T % 4) == 0) {
    if (sizeof(OutT) == 4) {
      // 2 lanes per image (16 B = 4 bins each), 16 images per instruction
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int m = r * 16 + (lane >> 1), j = lane & 1;
        int4 v = make_int4(st[(4 * j + 0) * kStageStride + m], st[(4 * j + 1) * kStageStride + m],
                           st[(4 * j + 2) * kStageStride + m], st[(4 * j + 3) * kStageStride + m]);
        if (m < nimg) __stcs((int4*)(out + ((img0 + m) * Dc + dl) * (int64_t)T + qc + 4 * j), v);
      }
    } else {
      // 4 lanes per image (16 B = 2 bins each), 8 images per instruction
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        int m = r * 8 + (lane >> 2), j = lane & 3;
        longlong2 v = make_longlong2(st[(2 * j) * kStageStride + m], st[(2 * j + 1) * kStageStride + m]);
        if (m < nimg) __stcs((longlong2*)(out + ((img0 + m) * Dc + dl) * (int64_t)T + qc + 2 * j), v);
      }
    }
  } else {
    for (int e = lane; e < kSweepImgs * nb; e += 32) {
      int m = e / nb, k = e % nb;
      if (m < nimg) out[((img0 + m) * Dc + dl) * (int64_t)T + qc + k] = (OutT)st[k * kStageStride + m];
    }
  }
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Signed packed pair: P = S0 + S1 * 2^16 (mod 2^32) with |S0|, |S1| < 2^15 -> (S0, S1).
__device__ __forceinline__ int2 unpack_s16x2(uint32_t P) {
  const int s0 = (int)(int16_t)(P & 0xFFFFu);
  return make_int2(s0, ((int)P - s0) >> 16);
}

// One warp, one direction, the CTA's 64 images: run the direction's sweep program
// (packets of 4 cw-row offsets), accumulating the signed packed weights of images
// (2l, 2l+1) and emitting the running (cumulative) sum for every bin.  Packets are
// consumed four at a time (a group): all 16 gathers are issued first and summed into
// group-local packed partials P[j] (|half| <= 16 * 255, so no carry ever crosses a
// half); emits unpack P[j] onto the int32 base, and the group's total is folded into
// the base once per group.
template <typename OutT>
__device__ __forceinline__ void sweep_direction(uint32_t lane4, const uint32_t* __restrict__ prg, int npk, int Lp,
                                                int* __restrict__ st, OutT* __restrict__ out, int64_t img0, int nimg,
                                                int Dc, int dl, int T, int lane) {
  const uint4* pk = (const uint4*)prg;
  const uint32_t* metaw = prg + 4 * Lp;
  int q = 0, base0 = 0, base1 = 0;
  const bool fast = sizeof(OutT) == 4 && nimg == kSweepImgs && (T % kStageBins) == 0;
  OutT* const lp = out + ((img0 + (lane >> 1)) * Dc + dl) * (int64_t)T + 4 * (lane & 1);
  const int64_t rstride = (int64_t)16 * Dc * T;
  int* const stl = st + 2 * lane;  // this lane's column pair of the stage
  // the program streams from L2: prefetch it into L1 (one 128-byte line per lane)
  if (lane * 8 < npk) asm volatile("prefetch.global.L1 [%0];" ::"l"(pk + lane * 8));
  if (lane * 32 < npk / 4) asm volatile("prefetch.global.L1 [%0];" ::"l"(metaw + lane * 32));
  uint4 w0 = __ldg(pk), w1 = __ldg(pk + 1), w2 = __ldg(pk + 2), w3 = __ldg(pk + 3);
  uint32_t mw = __ldg(metaw);
#pragma unroll 1
  for (int k = 0; k < npk; k += 4) {
    if ((k & 255) == 252 && lane * 8 + k + 4 < npk)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(pk + k + 4 + lane * 8));
    uint32_t P[4];
    P[0] = lds32(lane4 + w0.x) + lds32(lane4 + w0.y) + lds32(lane4 + w0.z) + lds32(lane4 + w0.w);
    P[1] = lds32(lane4 + w1.x) + lds32(lane4 + w1.y) + lds32(lane4 + w1.z) + lds32(lane4 + w1.w);
    P[2] = lds32(lane4 + w2.x) + lds32(lane4 + w2.y) + lds32(lane4 + w2.z) + lds32(lane4 + w2.w);
    P[3] = lds32(lane4 + w3.x) + lds32(lane4 + w3.y) + lds32(lane4 + w3.z) + lds32(lane4 + w3.w);
    P[1] += P[0];
    P[2] += P[1];
    P[3] += P[2];
    const uint32_t m = mw;
    if (k + 4 < npk) {
      w0 = __ldg(pk + k + 4); w1 = __ldg(pk + k + 5); w2 = __ldg(pk + k + 6); w3 = __ldg(pk + k + 7);
      mw = __ldg(metaw + (k >> 2) + 1);
    }
    if (m & 0xFEFEFEFEu) {  // some packet of the group ends a bin
      // one emitted bin: stage the running totals, flush a full 8-bin chunk
      auto emit = [&](const int2 v) {
        *(int2*)(stl + (q & (kStageBins - 1)) * kStageStride) = v;
        if (((++q) & (kStageBins - 1)) == 0) {
          __syncwarp();
          if (fast) {  // full group, int32, whole chunks: unguarded 16-byte stores
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int mm = r * 16 + (lane >> 1), j4 = 4 * (lane & 1);
              const int4 x = make_int4(st[(j4 + 0) * kStageStride + mm], st[(j4 + 1) * kStageStride + mm],
                                       st[(j4 + 2) * kStageStride + mm], st[(j4 + 3) * kStageStride + mm]);
              __stcs((int4*)(lp + r * rstride + (q - kStageBins)), x);
            }
          } else {
            sweep_store_chunk<OutT>(st, out, img0, nimg, Dc, dl, T, q - kStageBins, lane);
          }
          __syncwarp();
        }
      };
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t mj = m & (0xFEu << (8 * j));  // emit count of packet j, in place
        if (mj) {
          const int2 sv = unpack_s16x2(P[j]);
          const int2 v = make_int2(base0 + sv.x, base1 + sv.y);
          emit(v);
          if (__builtin_expect(mj > (2u << (8 * j)), 0))  // empty bins after it: same total
            for (int e = (int)(mj >> (8 * j + 1)) - 1; e > 0; --e) emit(v);
        }
      }
    }
    const int2 s = unpack_s16x2(P[3]);
    base0 += s.x;
    base1 += s.y;
  }
  if (q & (kStageBins - 1)) {  // the last, partial chunk (T not a multiple of 8)
    __syncwarp();
    sweep_store_chunk<OutT>(st, out, img0, nimg, Dc, dl, T, q & ~(kStageBins - 1), lane);
    __syncwarp();
  }
}

// Freudenthal combined weight of vertex (r, c) for chamber (A, B, C): the signed weights of
// the simplices (anchored at v - delta) whose designated vertex is v (freud_des), packed
// u16x2 for images (2l, 2l+1): positives (vertex, U, L) minus negatives (3 edges), each
// sum <= 765 per half.  p0 = this lane's pixel pair of vertex v in the staged rows.
__device__ __forceinline__ uint32_t freud_cw(const uint8_t* p0, int r, int c, int H, int W, int A, int B, int C) {
  auto P = [&](int dr, int dc) -> uint32_t {
    return __byte_perm(*(const uint16_t*)(p0 + (dr * W + dc) * kPixStride), 0, 0x4140);
  };
  const bool up = r > 0, dn = r + 1 < H, lf = c > 0, rt = c + 1 < W;
  const uint32_t a = P(0, 0);
  uint32_t pos = a, neg = 0;
  if (A) { if (lf) neg += __vmaxu2(a, P(0, -1)); } else if (rt) neg += __vmaxu2(a, P(0, 1));          // e_x
  if (B) { if (up) neg += __vmaxu2(a, P(-1, 0)); } else if (dn) neg += __vmaxu2(a, P(1, 0));          // e_y
  if (C) { if (up && lf) neg += __vmaxu2(a, P(-1, -1)); } else if (dn && rt) neg += __vmaxu2(a, P(1, 1));  // e_diag
  if (B && C) { if (up && lf) pos += __vmaxu2(__vmaxu2(a, P(-1, -1)), P(-1, 0)); }                  // U
  else if (A && !B) { if (lf && dn) pos += __vmaxu2(__vmaxu2(a, P(0, -1)), P(1, 0)); }
  else if (rt && dn) pos += __vmaxu2(__vmaxu2(a, P(0, 1)), P(1, 1));
  if (A && C) { if (up && lf) pos += __vmaxu2(__vmaxu2(a, P(-1, -1)), P(0, -1)); }                  // L
  else if (B && !A) { if (up && rt) pos += __vmaxu2(__vmaxu2(a, P(-1, 0)), P(0, 1)); }
  else if (dn && rt) pos += __vmaxu2(__vmaxu2(a, P(1, 0)), P(1, 1));
  return pos - neg;
}

template <typename OutT, bool FREUD>
__global__ void __launch_bounds__(kSweepWarps * 32, 1)
    k_sweep2d(const uint8_t* __restrict__ img, int64_t B, int H, int W, const uint32_t* __restrict__ prog,
              const int* __restrict__ prog_len, const int* __restrict__ qlist, const int* __restrict__ qcount,
              int Dc, int T, OutT* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int HW = H * W;
  uint32_t* cwb = (uint32_t*)smem;                 // [HW][32] words: images (2l, 2l+1) biased u16
  uint8_t* pix = smem + align16((size_t)(HW + 1) * 128);  // [HW][kPixStride] u8 (64 used)
  unsigned char* wbase = pix + sweep_pix_bytes(HW) + (size_t)(threadIdx.x >> 5) * sweep_warp_bytes(HW, T);
  const int Lp = sweep_prog_packets(HW, T), Lw = sweep_prog_words(HW, T);
  int* st = (int*)wbase;                                             // [kStageBins][kStageStride]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lane4 = (uint32_t)__cvta_generic_to_shared(cwb) + 4u * lane;
  const int64_t ngroups = (B + kSweepImgs - 1) / kSweepImgs;
  constexpr int NPH = FREUD ? 8 : 4;  // phase (quadrant / chamber) slots
  const bool phase_split = (int)gridDim.y >= NPH;
  const int ysub = phase_split ? (int)blockIdx.y / NPH : (int)blockIdx.y;
  const int nsub = phase_split ? (int)gridDim.y / NPH : (int)gridDim.y;
  if (threadIdx.x < 32) cwb[HW * 32 + threadIdx.x] = 0u;  // padding row: weight 0

  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int64_t img0 = grp * kSweepImgs;
    const int nimg = (int)((B - img0) < kSweepImgs ? (B - img0) : kSweepImgs);
    __syncthreads();  // the previous group's sweeps are done with pix / cwb
    // stage the group's pixels transposed: pix[v][i] (16-byte global loads when aligned)
    if ((HW & 15) == 0 && ((uintptr_t)img & 15) == 0) {
      // thread -> (image i = t % 64, 16-pixel block); a warp stores 32 images' bytes of one
      // pixel into one staged row: conflict-free byte stores
      const int per = HW >> 4;
      for (int f = threadIdx.x; f < kSweepImgs * per; f += blockDim.x) {
        const int i = f & (kSweepImgs - 1), v = (f >> 6) << 4;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (i < nimg) x = __ldcs((const uint4*)(img + (img0 + i) * HW + v));
        const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 16; ++k) pix[(v + k) * kPixStride + i] = (uint8_t)(wv[k >> 2] >> (8 * (k & 3)));
      }
    } else {
      for (int f = threadIdx.x; f < kSweepImgs * HW; f += blockDim.x) {
        const int i = f & (kSweepImgs - 1), v = f >> 6;
        pix[v * kPixStride + i] = i < nimg ? img[(img0 + i) * HW + v] : (uint8_t)0;
      }
    }
#pragma unroll 1
    for (int o = 0; o < (FREUD ? 8 : 4); ++o) {
      const int qco = qcount[o];
      // small batches: blockIdx.y splits the work over gridDim.y CTAs -- by phase when
      // gridDim.y >= the phase count (then by direction within the phase), else by direction
      if (phase_split && (int)blockIdx.y % NPH != o) continue;
      if (ysub >= qco) continue;
      __syncthreads();  // pix staged / previous quadrant's sweeps done with cwb
      const int dc = (o & 1) ? -1 : 1, dr = (o & 2) ? -1 : 1;
      if (FREUD) {
        int v = threadIdx.x >> 5;
        int r = v / W, c = v - r * W;
        const int step_r = kSweepWarps / W, step_c = kSweepWarps - step_r * W;
        for (; v < HW; v += kSweepWarps) {
          cwb[v * 32 + lane] = freud_cw(pix + v * kPixStride + 2 * lane, r, c, H, W, o & 1, (o >> 1) & 1, (o >> 2) & 1);
          r += step_r;
          c += step_c;
          if (c >= W) { c -= W; ++r; }
        }
      } else {
        // element (v, lane): cw of images 2l, 2l+1 as the signed packed pair
        // cw0 + cw1 * 2^16 (mod 2^32): (a + m_diag) - (m_c + m_r) in plain u32 arithmetic
        // (each operand half <= 510, so the borrow of a negative cw0 lands in cw1's half).
        int v = threadIdx.x >> 5;
        int r = v / W, c = v - r * W;
        const int step_r = kSweepWarps / W, step_c = kSweepWarps - step_r * W;
        for (; v < HW; v += kSweepWarps) {
          const bool vc = (unsigned)(c + dc) < (unsigned)W, vr = (unsigned)(r + dr) < (unsigned)H;
          const uint8_t* p0 = pix + v * kPixStride + 2 * lane;
          const uint32_t A = __byte_perm(*(const uint16_t*)p0, 0, 0x4140);
          uint32_t MC = 0, MR = 0, MD = 0;
          if (vc) MC = __vmaxu2(A, __byte_perm(*(const uint16_t*)(p0 + dc * kPixStride), 0, 0x4140));
          if (vr) MR = __vmaxu2(A, __byte_perm(*(const uint16_t*)(p0 + dr * W * kPixStride), 0, 0x4140));
          if (vc && vr)
            MD = __vmaxu2(__vmaxu2(MC, MR), __byte_perm(*(const uint16_t*)(p0 + (dr * W + dc) * kPixStride), 0, 0x4140));
          cwb[v * 32 + lane] = (A + MD) - (MC + MR);
          r += step_r;
          c += step_c;
          if (c >= W) { c -= W; ++r; }
        }
      }
      __syncthreads();
      for (int k = ysub + warp * nsub; k < qco; k += kSweepWarps * nsub) {
        const int dl = qlist[o * Dc + k];
        sweep_direction<OutT>(lane4, prog + (int64_t)dl * Lw, prog_len[dl], Lp, st, out, img0, nimg, Dc, dl, T, lane);
        __syncwarp();
      }
    }
  }
}

// Freudenthal corrections (after k_sweep2d): simplex (dl, u, t) was counted from bin lo but
// belongs to bin hi > lo: subtract its signed weight from the cumulative bins [lo, hi).
template <typename OutT>
__global__ void __launch_bounds__(256) k_sweep_fix(const uint8_t* __restrict__ img, int64_t B, int H, int W,
                                                   const int4* __restrict__ corr, const int* __restrict__ ncorr,
                                                   int Dc, int T, OutT* __restrict__ out) {
  const int64_t n = (int64_t)*ncorr * B;
  const int64_t HW = (int64_t)H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / B, b = i - e * B;
    const int4 c = corr[e];
    const uint8_t* p = img + b * HW + c.y;
    const int off[4] = {0, 1, W, W + 1};
    const int mask = freud_mask(c.z);
    int mx = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (mask >> k & 1) mx = max(mx, (int)p[off[k]]);
    const int sw = (c.z >= 4) ? mx : -mx;  // (-1)^dim: edges -1, triangles +1
    if (sw == 0) continue;
    OutT* row = out + (b * Dc + c.x) * (int64_t)T;
    for (int q = c.w & 0xFFFF; q < (c.w >> 16); ++q) {
      if (sizeof(OutT) == 4) atomicAdd((int*)(row + q), -sw);
      else atomicAdd((unsigned long long*)(row + q), (unsigned long long)(long long)(-sw));
    }
  }
}

// ---------------------------------------------------------------------------
// Histogram path: orthant-combined weights cwo[b][o][v] (int16, octant-major), o = sum_k (s_k > 0) << k.
// cw_o(v) = sum over axis subsets A (cells anchored at v, extending one step along each
// k in A toward -1 if bit k of o is set, else +1) of (-1)^|A| * max over the cell corners.
// ---------------------------------------------------------------------------
// the NO orthant-combined weights of one voxel (g = its coordinates); INTERIOR: every
// neighbour exists, so no -1 sentinels and no validity tests
template <int ND, bool INTERIOR>
__device__ __forceinline__ void grid_cw_vox(const uint8_t* __restrict__ im, const int (&g)[3], const int (&L)[3],
                                            int16_t (&res)[1 << ND]) {
  constexpr int NO = 1 << ND;
  // 3^ND neighbourhood, -1 where outside the grid
  int nb[ND == 2 ? 9 : 27];
#pragma unroll
  for (int t = 0; t < (ND == 2 ? 9 : 27); ++t) {
    const int o0 = t % 3 - 1, o1 = (t / 3) % 3 - 1, o2 = ND == 3 ? t / 9 - 1 : 0;
    const int x = g[0] + o0, y = g[1] + o1, z = g[2] + o2;
    const bool ok = INTERIOR ||
                    ((unsigned)x < (unsigned)L[0] && (unsigned)y < (unsigned)L[1] && (unsigned)z < (unsigned)L[2]);
    nb[t] = ok ? (int)__ldg(im + (z * L[1] + y) * L[0] + x) : -1;
  }
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    int cw = 0;
#pragma unroll
    for (int A = 0; A < NO; ++A) {
      int m = 0;
      bool valid = true;
#pragma unroll
      for (int S = 0; S < NO; ++S) {
        if ((S & ~A) != 0) continue;  // corners = subsets of A
        int t = 0, mul = 1;
#pragma unroll
        for (int k = 0; k < ND; ++k) {
          int off = ((S >> k) & 1) ? (((o >> k) & 1) ? -1 : 1) : 0;
          t += (off + 1) * mul;
          mul *= 3;
        }
        const int pv = nb[t];
        if (!INTERIOR && pv < 0) valid = false;
        m = pv > m ? pv : m;
      }
      if (INTERIOR || valid) cw += (__popc(A) & 1) ? -m : m;
    }
    res[o] = (int16_t)cw;
  }
}

template <int ND>
__global__ void __launch_bounds__(256) k_grid_cw(const uint8_t* __restrict__ img, int64_t nimg, int64_t d0,
                                                 int64_t d1, int64_t d2, int16_t* __restrict__ cwo) {
  constexpr int NO = 1 << ND;
  int L[3];  // L[k] = length of axis k (axis 0 fastest); one image has < 2^31 voxels
  if (ND == 2) { L[0] = (int)d1; L[1] = (int)d0; L[2] = 1; } else { L[0] = (int)d2; L[1] = (int)d1; L[2] = (int)d0; }
  const int nv = L[0] * L[1] * L[2];
  const int L01 = L[0] * L[1];
  // grid.y walks the images, grid.x x threads the voxels of one image: 32-bit index math
  for (int64_t b = blockIdx.y; b < nimg; b += gridDim.y)
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const int z0 = v / L01, r01 = v - z0 * L01, y0 = r01 / L[0], x0 = r01 - y0 * L[0];
    const int g[3] = {x0, y0, z0};
    const uint8_t* im = img + b * (int64_t)nv;
    int16_t res[NO];
    const bool interior = x0 > 0 && x0 < L[0] - 1 && y0 > 0 && y0 < L[1] - 1 && (ND == 2 || (z0 > 0 && z0 < L[2] - 1));
    if (interior) grid_cw_vox<ND, true>(im, g, L, res);  // ~98 % of a 256^3 volume: no bounds logic
    else grid_cw_vox<ND, false>(im, g, L, res);
#pragma unroll
    for (int o = 0; o < NO; ++o) cwo[(b * NO + o) * nv + v] = res[o];  // octant-major rows
  }
}

// lanes = 32 directions, each warp streams whole grid rows (x fastest).  Per row the
// lane folds everything but the x term into one constant, so a voxel costs one FMA:
//     u = fmaf((float)x, A s0 / S, U0),  U0 = A (y s1 + z s2 - s0 (L0-1)/(2S)) + B,
// an approximation of (T-1)(h - lo)/(hi - lo) within the guard tau (A1:
// tau = 2 eps (A (n+2) R + 2|B| + T + 1) bounds this evaluation's error too); voxels whose
// u lies within tau of an integer recompute h exactly in binary64 from the axis tables.
// The row's orthant weights are staged in smem with coalesced 16-byte loads; the
// histogram is lane-interleaved [T][32] so atomics never bank-conflict.
constexpr int kSegVox = 256;     // voxels per staged row segment
constexpr int kSegStride = 264;  // int16 per staged octant row (132 words = 4 mod 32: conflict-free)

__device__ __noinline__ int grid_repair(float cx, float cy, float cz, float s0, float s1, float s2, int nd,
                                        const GridParams* gp) {
  double h64 = __dadd_rn(__dmul_rn((double)cx, (double)s0), __dmul_rn((double)cy, (double)s1));
  if (nd == 3) h64 = __dadd_rn(h64, __dmul_rn((double)cz, (double)s2));
  note_repair();
  return alpha64(h64, *gp);
}

// predicated shared-memory add (no branch, no reconvergence barrier)
__device__ __forceinline__ void red_shared_add(uint32_t addr, int w) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(w) : "memory");
}
__device__ __forceinline__ void red_shared_nz(uint32_t addr, int w) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %1, 0;\n\t@p red.shared.add.s32 [%0], %1;\n\t}" ::"r"(addr), "r"(w));
}

template <int ND>
__global__ void __launch_bounds__(256) k_grid_hist(const int16_t* __restrict__ cwo, int64_t d0, int64_t d1, int64_t d2,
                                                   const float* __restrict__ dirs, int d_begin, int Dc,
                                                   const GridParams* __restrict__ gp, int64_t slice_rows,
                                                   int64_t b_offset, unsigned long long* __restrict__ diff) {
  constexpr int NO = 1 << ND;
  extern __shared__ __align__(16) int hist[];  // [T][32] lane-interleaved, then per-warp cw segments
  __shared__ float axc[3][1024];
  const GridParams g = *gp;
  const int T = g.T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int16_t* seg = (int16_t*)(hist + 32 * T) + warp * NO * kSegStride;  // [NO][kSegStride]
  int L[3];
  if (ND == 2) { L[0] = (int)d1; L[1] = (int)d0; L[2] = 1; } else { L[0] = (int)d2; L[1] = (int)d1; L[2] = (int)d0; }
  int maxd = L[0] > L[1] ? L[0] : L[1];
  maxd = L[2] > maxd ? L[2] : maxd;
  const double S = (double)(maxd - 1 > 1 ? maxd - 1 : 1);
  for (int k = 0; k < ND; ++k)
    for (int i = threadIdx.x; i < L[k]; i += blockDim.x) axc[k][i] = axis_coord(i, L[k], S);
  for (int i = threadIdx.x; i < 32 * T; i += blockDim.x) hist[i] = 0;
  const int dl = blockIdx.x * 32 + lane;
  const bool active = dl < Dc;
  const int p = d_begin + (active ? dl : 0);
  float s[3] = {0.f, 0.f, 0.f};
  int o = 0;
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    s[k] = dirs[p * ND + k];
    o |= (s[k] > 0.f ? 1 : 0) << k;
  }
  const float A = g.A, Bc = g.B, tau = g.fp32_only ? -1.f : g.tau;
  const float a0 = A * s[0] / (float)S;
  const float c0 = (float)((double)(L[0] - 1) / 2.0);
  const int Tm1 = T - 1;
  const uint32_t hlane = (uint32_t)__cvta_generic_to_shared(hist) + 4u * lane;
  const uint32_t* segw = (const uint32_t*)(seg + o * kSegStride);  // this lane's octant row, 2 voxels per word
  const uint32_t amask = active ? 0xFFFFFFFFu : 0u;  // inactive lanes add nothing
  const int64_t nrows = (int64_t)L[1] * L[2];
  const int64_t nv = nrows * L[0];
  const int64_t b = blockIdx.z;
  const int64_t r0 = blockIdx.y * slice_rows;
  const int64_t r1 = (r0 + slice_rows) < nrows ? (r0 + slice_rows) : nrows;
  const int16_t* cwb = cwo + (b * NO) * nv;
  __syncthreads();
  for (int64_t row = r0 + warp; row < r1; row += nwarps) {
    const int y = (int)(row % L[1]), z = (int)(row / L[1]);
    const float cy = axc[1][y], cz = ND == 3 ? axc[2][z] : 0.f;
    float C = cy * s[1];
    if (ND == 3) C = fmaf(cz, s[2], C);
    const float U0 = fmaf(fmaf(-s[0], c0 / (float)S, C), A, Bc);
    for (int x0 = 0; x0 < L[0]; x0 += kSegVox) {
      const int nx = (L[0] - x0) < kSegVox ? (L[0] - x0) : kSegVox;
      // stage the segment's NO octant rows: seg[oo][0..nx)
      const int64_t src0 = row * L[0] + x0;
      if (((src0 | nx | nv) & 7) == 0) {
        const int per = nx >> 3;  // uint4 per row
        for (int t = lane; t < NO * per; t += 32) {
          const int oo = t / per, k = t - oo * per;
          *(uint4*)(seg + oo * kSegStride + 8 * k) = __ldg((const uint4*)(cwb + oo * nv + src0) + k);
        }
      } else {
        for (int t = lane; t < NO * nx; t += 32) {
          const int oo = t / nx, k = t - oo * nx;
          seg[oo * kSegStride + k] = cwb[oo * nv + src0 + k];
        }
      }
      // zero-pad every octant row to a multiple of 8 voxels (the loop below takes 8 at a time)
      const int nx8 = (nx + 7) & ~7;
      for (int t = lane; t < NO * (nx8 - nx); t += 32) {
        const int oo = t / (nx8 - nx);
        seg[oo * kSegStride + nx + (t - oo * (nx8 - nx))] = 0;
      }
      __syncwarp();
      // 8 voxels per step: one 16-byte load of this lane's octant row, eight fp32 bins
      // (branch-free clamp), one guard test for the group, eight red.shared adds
      for (int xi = 0; xi < nx; xi += 8) {
        const uint4 q = *(const uint4*)(segw + (xi >> 1));
        const uint32_t wd[4] = {q.x & amask, q.y & amask, q.z & amask, q.w & amask};
        const float xf = (float)(x0 + xi);
        int bin[8];
        float dist[8], dmin = 2.f;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const float u = fmaf(xf + (float)h, a0, U0);  // x0 + xi + h is exact in fp32
          bin[h] = max(0, min(__float2int_ru(u), Tm1));
          dist[h] = fabsf(u - rintf(u));
          dmin = fminf(dmin, dist[h]);
        }
        if (__builtin_expect(dmin < tau, 0)) {  // some voxel of the group sits near a bin edge
          const int nvalid = nx - xi;  // padding voxels need no repair
#pragma unroll
          for (int h = 0; h < 8; ++h)
            if (dist[h] < tau && h < nvalid)
              bin[h] = grid_repair(axc[0][x0 + xi + h], cy, cz, s[0], s[1], s[2], ND, gp);
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int w = (h & 1) ? (int)wd[h >> 1] >> 16 : (int)(int16_t)(wd[h >> 1] & 0xFFFFu);
          red_shared_add(hlane + 128u * (uint32_t)bin[h], w);
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * T; i += blockDim.x) {
    int q = i >> 5, r = i & 31;
    int val = hist[i];
    if (val != 0 && blockIdx.x * 32 + r < Dc)
      atomicAdd(diff + ((b_offset + b) * Dc + blockIdx.x * 32 + r) * (int64_t)T + q, (unsigned long long)(long long)val);
  }
}

// ---------------------------------------------------------------------------
// host launchers (called from api.cu)
// ---------------------------------------------------------------------------
wect_status launch_grid_params(int ndim, const int64_t* dims, const float* dirs, int D, const wect_grid& grid,
                               GridParams* gp, cudaStream_t st) {
  k_grid_params<<<1, 256, 0, st>>>(ndim, dims[0], dims[1], ndim == 3 ? dims[2] : 1, dirs, D, grid.T, grid.maxheight,
                                   grid.lo, grid.hi, grid.flags, gp); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

bool sweep2d_supported(int ndim, const int64_t* dims, int T) {
  if (ndim != 2) return false;
  int64_t HW = dims[0] * dims[1];
  return HW >= 1 && HW <= 1023 && T <= 4096 && sweep_smem_bytes((int)HW, T) <= 227 * 1024;
}

wect_status launch_sweep2d(const uint8_t* img, int64_t B, int H, int W, const float* dirs, int d_begin, int Dc,
                           int T, const GridParams* gp, void* scratch, void* out, wect_dtype odtype, cudaStream_t st,
                           int num_sms, int freud) {
  const int HW = H * W;
  const int Lp = sweep_prog_packets(HW, T);
  uint32_t* prog = (uint32_t*)scratch;
  int* ints = (int*)(((uintptr_t)(prog + (size_t)Dc * sweep_prog_words(HW, T)) + 15) & ~(uintptr_t)15);
  int* qcount = ints;           // 8 chamber slots (cubical uses 4)
  int* prog_len = ints + 8;
  int* qlist = prog_len + Dc;   // [8][Dc]
  int* ncorr = qlist + 8 * Dc;
  int4* corr = (int4*)(((uintptr_t)(ncorr + 1) + 15) & ~(uintptr_t)15);
  const int corr_cap = freud ? 5 * HW * Dc : 0;
  WECT_CUDA_TRY(cudaMemsetAsync(qcount, 0, 8 * sizeof(int), st));
  WECT_CUDA_TRY(cudaMemsetAsync(ncorr, 0, sizeof(int), st));
  const size_t sort_smem = (size_t)(2 * T + Lp) * sizeof(int) + align16((size_t)HW * 2);
  if (sort_smem > 48 * 1024) WECT_CUDA_TRY(cudaFuncSetAttribute(k_sort2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem));
  k_sort2d<<<Dc, 256, sort_smem, st>>>(H, W, dirs, d_begin, Dc, gp, prog, prog_len, qlist, qcount, freud, corr, ncorr,
                                       corr_cap); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  const size_t smem = sweep_smem_bytes(HW, T);
  const int64_t ngroups = (B + kSweepImgs - 1) / kSweepImgs;
  // fewer image groups than SMs (small batches): split every phase's directions over CTAs
  const int nph = freud ? 8 : 4;
  int split = (int)(num_sms / (ngroups > 0 ? ngroups : 1));
  split = split < 1 ? 1 : (split > kSweepWarps * nph ? kSweepWarps * nph : split);
  if (split >= nph) split = (split / nph) * nph;  // whole phase rows: y = phase + nph * sub
  const dim3 grid((unsigned)(ngroups < num_sms ? ngroups : num_sms), (unsigned)split);
  MainTimer timer(st);
#define WECT_SWEEP(OT, FR)                                                                                   \
  do {                                                                                                       \
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_sweep2d<OT, FR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_sweep2d<OT, FR><<<grid, kSweepWarps * 32, smem, st>>>(img, B, H, W, prog, prog_len, qlist, qcount, Dc, T,  \
                                                             (OT*)out);                                         \
    count_launch();                                                                                          \
  } while (0)
  if (odtype == WECT_I32) {
    if (freud) WECT_SWEEP(int32_t, true); else WECT_SWEEP(int32_t, false);
  } else {
    if (freud) WECT_SWEEP(long long, true); else WECT_SWEEP(long long, false);
  }
#undef WECT_SWEEP
  timer.stop();
  if (freud) {  // the rare rounded-diagonal simplices (usually none)
    const int fb = num_sms * 4;
    if (odtype == WECT_I32) k_sweep_fix<int32_t><<<fb, 256, 0, st>>>(img, B, H, W, corr, ncorr, Dc, T, (int32_t*)out);
    else k_sweep_fix<long long><<<fb, 256, 0, st>>>(img, B, H, W, corr, ncorr, Dc, T, (long long*)out);
    count_launch();
  }
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

size_t sweep2d_scratch_bytes(int HW, int Dc, int T, int freud) {
  return (size_t)Dc * sweep_prog_words(HW, T) * 4 + 16 + (size_t)(8 + Dc + 8 * Dc + 1) * 4 + 64 +
         (freud ? (size_t)5 * HW * Dc * sizeof(int4) + 16 : 0);
}

// histogram path over a chunk of images [b0, b0 + nb): cwo scratch for nb images, diff rows at b0
wect_status launch_grid_hist(const uint8_t* img, int64_t b0, int64_t nb, int ndim, const int64_t* dims,
                             const float* dirs, int d_begin, int Dc, int T, const GridParams* gp, int16_t* cwo,
                             unsigned long long* diff, cudaStream_t st, int num_sms) {
  const int64_t nv = ndim == 2 ? dims[0] * dims[1] : dims[0] * dims[1] * dims[2];
  const uint8_t* im = img + b0 * nv;
  const int64_t total = nb * nv;
  (void)total;
  const int64_t want_x = (nv + 255) / 256;
  const int gx = (int)(want_x < (int64_t)num_sms * 16 ? want_x : (int64_t)num_sms * 16);
  int64_t gy = ((int64_t)num_sms * 16 + gx - 1) / gx;
  gy = gy < nb ? gy : nb;
  gy = gy < 65535 ? (gy < 1 ? 1 : gy) : 65535;
  dim3 gcw((unsigned)gx, (unsigned)gy);
  if (ndim == 2) k_grid_cw<2><<<gcw, 256, 0, st>>>(im, nb, dims[0], dims[1], 1, cwo);
  else k_grid_cw<3><<<gcw, 256, 0, st>>>(im, nb, dims[0], dims[1], dims[2], cwo);
  count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  const int tiles = (Dc + 31) / 32;
  // slices of whole rows: enough CTAs for >= 4 waves; int32 partials stay below 2^31
  // (a CTA sees <= 2^18 voxels * 1020 |cw| per direction)
  const int64_t L0 = ndim == 2 ? dims[1] : dims[2];
  const int64_t nrows = nv / L0;
  int64_t rows_cap = ((int64_t)1 << 18) / L0;
  if (rows_cap < 1) rows_cap = 1;
  int64_t want = ((int64_t)num_sms * 8 + tiles * nb - 1) / (tiles * nb);
  if (want < 1) want = 1;
  int64_t slice_rows = (nrows + want - 1) / want;
  if (slice_rows > rows_cap) slice_rows = rows_cap;
  if (slice_rows < 1) slice_rows = 1;
  const int64_t nslices = (nrows + slice_rows - 1) / slice_rows;
  const size_t smem = (size_t)32 * T * sizeof(int) + (size_t)8 * (1 << ndim) * kSegStride * sizeof(int16_t);
  dim3 gridd(tiles, (unsigned)nslices, (unsigned)nb);
  MainTimer timer(st);
  if (ndim == 2) {
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_grid_hist<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_grid_hist<2><<<gridd, 256, smem, st>>>(cwo, dims[0], dims[1], 1, dirs, d_begin, Dc, gp, slice_rows, b0, diff); count_launch();
  } else {
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_grid_hist<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_grid_hist<3><<<gridd, 256, smem, st>>>(cwo, dims[0], dims[1], dims[2], dirs, d_begin, Dc, gp, slice_rows, b0, diff); count_launch();
  }
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

}  // namespace wect
