// k_ecf_images.cu -- ECF of batches of uint8 images / voxel volumes (ecf_images;
// SURVEY.md §8(f) NEXT-1).
//
// What is computed (Remark "which-ecf"): the pixel intensities are the
// vertex filter and the result is the unweighted Euler characteristic of the lower-star
// filtration of the cubical V-construction: every axis-aligned
// unit i-cube of the grid is a cell of sign (-1)^i (reading A7) whose filter
// value is the max over its corners (lower star).  That is Algorithm 1
// with m = 1 filter and unit weights, each image its own complex.
//
// Intensities are u8, so the method reduces exactly to, per image,
//   H[c]  = sum over cells with value c of (-1)^dim            (Alg. 1 lines 4-10 by value)
//   C[c]  = H[0] + ... + H[c]                                 (the sublevel-set EC at c)
//   out[q] = C[cstar(q)],  cstar(q) = max{c in 0..255 : alpha(c) <= q}   (0 if none)
// because alpha is monotone (Galois law): the cells in bins <= q are exactly
// the cells with value <= cstar(q).  cstar is a per-call table evaluated in binary64 in
// the order alpha is written (reading A1), one row per possible per-image M = 0..255
// when each image uses its own paper grid [-M, M], else one row.
//
// Pairing (fewer shared atomics): the cells anchored at vertex v (v = their lowest
// corner) are the axis subsets S.  S and S + {x} have opposite signs and
// value(S + {x}) >= value(S); when the two values are equal they cancel and neither is
// added.
//
// Three paths: 2-D images with W % 4 == 0, H*W % 16 == 0, H*W <= 1024 (the
// MNIST-shaped batches): k_ecf_img2d_w4, packed u16x2 (below).  Other images of
// <= kEcfSmallMax vertices (MNIST-shaped batches): one warp per
// image, pixels staged in shared memory, a warp-private 256-entry histogram, scan and
// output in the same warp -- one launch, input read once, output written once.
// Larger images: CTAs over vertex chunks add their histograms into an int64 [B][256]
// table (plus the per-image max), then one warp per image scans and maps.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace wect {

constexpr int kEcfWarps = 8;
constexpr int kEcfSmallMax = 4096;
constexpr int kEcfChunk = 1 << 15;  // vertices (anchors) per CTA on the large path

// ---------------------------------------------------------------------------
// cstar table: row r, bin q -> max{c : alpha_r(c) <= q} or -1.
// mode 0: row r uses the grid [-r, r] (per-image M = r); mode 1: one row, grid [lo, hi].
// alpha(c) = clamp(ceil(((T-1) (c - lo)) / (hi - lo)), 0, T-1); hi <= lo: bin 0 (A6).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ecf_cstar(int mode, double lo_in, double hi_in, int T,
                                                   int16_t* __restrict__ cstar) {
  __shared__ int bins[256];
  const int r = blockIdx.x;
  const double lo = mode == 0 ? -(double)r : lo_in;
  const double hi = mode == 0 ? (double)r : hi_in;
  {
    const int c = threadIdx.x;
    int b = 0;
    if (hi > lo) {
      const double u = __ddiv_rn(__dmul_rn((double)(T - 1), __dsub_rn((double)c, lo)), __dsub_rn(hi, lo));
      const double cu = ceil(u);
      b = cu < 0.0 ? 0 : (cu > (double)(T - 1) ? T - 1 : (int)cu);
    }
    bins[c] = b;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < T; q += blockDim.x) {
    // bins[] is non-decreasing in c: count = #{c : bins[c] <= q} by binary search
    int lo_i = 0, hi_i = 256;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i) >> 1;
      if (bins[mid] <= q) lo_i = mid + 1;
      else hi_i = mid;
    }
    cstar[(int64_t)r * T + q] = (int16_t)(lo_i - 1);
  }
}

// ---------------------------------------------------------------------------
// Signed cell values of the cells anchored at vertex v (see "Pairing" above).
// p: the image's pixels; (x, y, z): v's coordinates; X, Y, Z: dims (Z = 1 in 2D);
// add(c, s): histogram update.
// ---------------------------------------------------------------------------
template <int ND, typename Px, typename Add>
__device__ __forceinline__ void ecf_anchor(Px p, int64_t v, int x, int y, int z, int X, int Y, int Z, Add add) {
  const bool ex = x + 1 < X, ey = y + 1 < Y, ez = ND == 3 && z + 1 < Z;
  const int64_t sy = X, sz = (int64_t)X * Y;
  // face maxima at x (f) and at x + 1 (g) for S in {}, {y}, {z}, {y,z}
  const int a = p(v), a1 = ex ? p(v + 1) : 0;
  int f[4], g[4];
  f[0] = a;
  g[0] = a1;
  if (ey) {
    f[1] = max(a, p(v + sy));
    g[1] = ex ? max(a1, p(v + 1 + sy)) : 0;
  }
  if (ND == 3 && ez) {
    f[2] = max(a, p(v + sz));
    g[2] = ex ? max(a1, p(v + 1 + sz)) : 0;
    if (ey) {
      f[3] = max(max(f[1], f[2]), p(v + sy + sz));
      g[3] = ex ? max(max(g[1], g[2]), p(v + 1 + sy + sz)) : 0;
    }
  }
#pragma unroll
  for (int S = 0; S < (ND == 3 ? 4 : 2); ++S) {
    const bool valid = (!(S & 1) || ey) && (!(S & 2) || ez);
    if (!valid) continue;
    const int s = (__popc(S) & 1) ? -1 : 1;  // (-1)^|S|
    const int m = f[S];
    if (ex) {
      const int mx = max(m, g[S]);
      if (mx != m) {
        add(m, s);
        add(mx, -s);
      }
    } else {
      add(m, s);
    }
  }
}

// Per-image tail (one warp): in-place scan of the 256-entry histogram and the mapped
// output row.  hist: shared, 256 entries of Acc.
template <typename Acc, typename OutT>
__device__ __forceinline__ void ecf_scan_emit(Acc* hist, int lane, const int16_t* __restrict__ cst, int T,
                                              OutT* __restrict__ orow) {
  Acc loc[8];
  Acc run = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    run += hist[8 * lane + k];
    loc[k] = run;
  }
  Acc incl = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Acc y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  const Acc excl = incl - run;
#pragma unroll
  for (int k = 0; k < 8; ++k) hist[8 * lane + k] = excl + loc[k];
  __syncwarp();
  for (int q = lane; q < T; q += 32) {
    const int cs = __ldg(cst + q);
    orow[q] = (OutT)(cs >= 0 ? hist[cs] : (Acc)0);
  }
}

// ---------------------------------------------------------------------------
// Small images: one warp per image.
// smem per warp: hist[256] int32, then the image's pixels (HW bytes, 16-byte aligned).
// ---------------------------------------------------------------------------
template <int ND, typename OutT>
__global__ void __launch_bounds__(kEcfWarps * 32) k_ecf_img_small(const uint8_t* __restrict__ img, int64_t B, int X,
                                                                  int Y, int Z, int per_image_M,
                                                                  const int16_t* __restrict__ cstar, int T,
                                                                  OutT* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int HW = X * Y * Z;
  const int pbytes = (HW + 15) & ~15;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* hist = (int*)(smem + (size_t)warp * (1024 + pbytes));
  uint8_t* pix = (uint8_t*)(hist + 256);
  const bool vec = (HW & 15) == 0 && ((uintptr_t)img & 15) == 0;
  const int64_t nwarps = (int64_t)gridDim.x * kEcfWarps;
  for (int64_t b = (int64_t)blockIdx.x * kEcfWarps + warp; b < B; b += nwarps) {
    const uint8_t* src = img + b * HW;
    unsigned mx = 0;
    if (vec) {
      for (int i = lane; i < (HW >> 4); i += 32) {
        const uint4 w = __ldcs((const uint4*)src + i);
        *((uint4*)pix + i) = w;
        mx = __vmaxu4(mx, __vmaxu4(__vmaxu4(w.x, w.y), __vmaxu4(w.z, w.w)));
      }
    } else {
      for (int i = lane; i < HW; i += 32) {
        const uint8_t w = src[i];
        pix[i] = w;
        mx = w > mx ? w : mx;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) hist[8 * lane + k] = 0;
    mx = max(max(mx & 0xFFu, (mx >> 8) & 0xFFu), max((mx >> 16) & 0xFFu, mx >> 24));
    const int M = (int)__reduce_max_sync(0xffffffffu, mx);
    __syncwarp();
    const uint32_t hs = (uint32_t)__cvta_generic_to_shared(hist);
    auto px = [&](int64_t u) -> int { return pix[u]; };
    auto add = [&](int c, int s) { asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(hs + 4u * c), "r"(s) : "memory"); };
    int x = lane % X, yz = lane / X;
    int y = yz % Y, z = yz / Y;
    const int sx = 32 % X, syz = 32 / X;
    for (int v = lane; v < HW; v += 32) {
      ecf_anchor<ND>(px, v, x, y, z, X, Y, Z, add);
      x += sx;
      y += syz;
      if (x >= X) { x -= X; ++y; }
      while (y >= Y) { y -= Y; ++z; }
    }
    __syncwarp();
    ecf_scan_emit<int, OutT>(hist, lane, cstar + (per_image_M ? (int64_t)M * T : 0), T, out + b * T);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Small 2-D images with W % 4 == 0 (MNIST-shaped): packed u16x2 form of the same pairing.
// The image is staged as u16 values 4*p (byte offsets into the histogram) in rows of
// pitch P = W + 2 with one extra row; the padding column(s) and row hold 4*256, a sink bin
// past the 256 real ones.  Then every anchor is handled alike: a missing x-neighbour
// makes max(a, b) the sink (so +1@a, -1@sink), a missing y-row makes both y-cells the
// sink (they cancel).  A lane takes two anchors (x, x+1) per step: four 32-bit LDS, two
// byte permutes and three u16x2 maxima give a, max(a,b), max(a,c), max(a,b,c,d) for both.
// The warp's histogram sits at a 2048-byte aligned shared address (aligned at run time
// inside the dynamic window) so each histogram address is one LOP3 of the packed value.
// ---------------------------------------------------------------------------
constexpr int kSinkOff = 4 * 256;

template <typename OutT>
__global__ void __launch_bounds__(kEcfWarps * 32) k_ecf_img2d_w4(const uint8_t* __restrict__ img, int64_t B, int H,
                                                                 int W, int per_image_M,
                                                                 const int16_t* __restrict__ cstar, int T,
                                                                 OutT* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int P = W + 2, P2 = P >> 1, W2 = W >> 1, HW = H * W;
  const int pwords = (H + 1) * P2;
  // [pad to a 2048-byte aligned shared address][kEcfWarps x 2048-byte histograms][pixels]
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  unsigned char* hbase = smem + (((s0 + 2047u) & ~2047u) - s0);
  int* hist = (int*)(hbase + (size_t)warp * 2048);
  uint32_t* S = (uint32_t*)(hbase + kEcfWarps * 2048) + (size_t)warp * ((pwords + 3) & ~3);
  const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(hist);
  for (int i = lane; i < pwords; i += 32) S[i] = (uint32_t)kSinkOff | ((uint32_t)kSinkOff << 16);
  // the fixed grid's cstar row in registers (T <= 256)
  int creg[8];
  const bool creg_ok = !per_image_M && T <= 256;
  if (creg_ok) {
#pragma unroll
    for (int k = 0; k < 8; ++k) creg[k] = 32 * k + lane < T ? (int)__ldg(cstar + 32 * k + lane) : -1;
  }
  __syncwarp();
  const int64_t nwarps = (int64_t)gridDim.x * kEcfWarps;
  const int n16 = HW >> 4;  // <= 64: at most two 16-byte loads per lane
  // lane's two 16-pixel blocks: flat pixel index -> staged word index (row pitch P)
  int widx[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int v = 16 * (lane + 32 * j) + 4 * g;
      const int r = v / W;
      widx[j][g] = (r * P + (v - r * W)) >> 1;
    }
  // anchor-pair coordinates advance by 32 items per step: (dr, dx) = divmod(32, W2)
  const int dr = 32 / W2, dx = 32 - dr * W2;
  const int r0 = lane / W2, x0 = lane - r0 * W2;
  int64_t b = (int64_t)blockIdx.x * kEcfWarps + warp;
  uint4 pf[2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
    pf[j] = (b < B && lane + 32 * j < n16) ? __ldcs((const uint4*)(img + b * HW) + lane + 32 * j) : make_uint4(0, 0, 0, 0);
  for (; b < B; b += nwarps) {
    unsigned mx = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (lane + 32 * j < n16) {
        const uint32_t wv[4] = {pf[j].x, pf[j].y, pf[j].z, pf[j].w};
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          S[widx[j][g]] = __byte_perm(wv[g], 0, 0x4140) << 2;
          S[widx[j][g] + 1] = __byte_perm(wv[g], 0, 0x4342) << 2;
          mx = __vmaxu4(mx, wv[g]);
        }
      }
    }
    // the next image's pixels are in flight while this one is processed
    const int64_t bn = b + nwarps;
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (bn < B && lane + 32 * j < n16) pf[j] = __ldcs((const uint4*)(img + bn * HW) + lane + 32 * j);
#pragma unroll
    for (int k = 0; k < 8; ++k) hist[8 * lane + k] = 0;
    mx = max(max(mx & 0xFFu, (mx >> 8) & 0xFFu), max((mx >> 16) & 0xFFu, mx >> 24));
    const int M = (int)__reduce_max_sync(0xffffffffu, mx);
    __syncwarp();
    int r = r0, xp = x0;
    for (int it = lane; it < H * W2; it += 32) {
      const int ai = r * P2 + xp;
      xp += dx;
      r += dr;
      if (xp >= W2) { xp -= W2; ++r; }
      const uint32_t a2 = S[ai], an = S[ai + 1], c2 = S[ai + P2], cn = S[ai + P2 + 1];
      const uint32_t b2 = __byte_perm(a2, an, 0x5432), d2 = __byte_perm(c2, cn, 0x5432);
      const uint32_t m_x = __vmaxu2(a2, b2), m_y = __vmaxu2(a2, c2);
      const uint32_t m_xy = __vmaxu2(m_x, __vmaxu2(c2, d2));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t A = (h ? a2 >> 16 : a2 & 0xFFFFu) | wbase;
        const uint32_t X = (h ? m_x >> 16 : m_x & 0xFFFFu) | wbase;
        const uint32_t Y = (h ? m_y >> 16 : m_y & 0xFFFFu) | wbase;
        const uint32_t XY = (h ? m_xy >> 16 : m_xy & 0xFFFFu) | wbase;
        // equal values cancel and are skipped
        if (X != A) {
          asm volatile("red.shared.add.s32 [%0], 1;" ::"r"(A) : "memory");
          asm volatile("red.shared.add.s32 [%0], -1;" ::"r"(X) : "memory");
        }
        if (XY != Y) {
          asm volatile("red.shared.add.s32 [%0], -1;" ::"r"(Y) : "memory");
          asm volatile("red.shared.add.s32 [%0], 1;" ::"r"(XY) : "memory");
        }
      }
    }
    __syncwarp();
    // in-place inclusive scan of the 256 real bins (lane: bins 8l .. 8l+7)
    int4 h0 = *(int4*)(hist + 8 * lane), h1 = *(int4*)(hist + 8 * lane + 4);
    h0.y += h0.x; h0.z += h0.y; h0.w += h0.z;
    h1.x += h0.w; h1.y += h1.x; h1.z += h1.y; h1.w += h1.z;
    int incl = h1.w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    const int ex = incl - h1.w;
    h0.x += ex; h0.y += ex; h0.z += ex; h0.w += ex;
    h1.x += ex; h1.y += ex; h1.z += ex; h1.w += ex;
    *(int4*)(hist + 8 * lane) = h0;
    *(int4*)(hist + 8 * lane + 4) = h1;
    __syncwarp();
    OutT* orow = out + b * T;
    if (creg_ok) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (32 * k + lane < T) __stcs(orow + 32 * k + lane, (OutT)(creg[k] >= 0 ? hist[creg[k]] : 0));
    } else {
      const int16_t* cst = cstar + (per_image_M ? (int64_t)M * T : 0);
      for (int q = lane; q < T; q += 32) {
        const int cs = __ldg(cst + q);
        orow[q] = (OutT)(cs >= 0 ? hist[cs] : 0);
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Large images: CTA (chunk, image) -> int64 histogram table [B][256] and per-image max.
// ---------------------------------------------------------------------------
template <int ND>
__global__ void __launch_bounds__(256) k_ecf_img_hist(const uint8_t* __restrict__ img, int X, int Y, int Z,
                                                      unsigned long long* __restrict__ ghist,
                                                      unsigned int* __restrict__ gmax) {
  __shared__ int hist[kEcfWarps][256];
  __shared__ unsigned int smax;
  const int64_t HW = (int64_t)X * Y * Z;
  const int64_t b = blockIdx.y;
  const int64_t v0 = (int64_t)blockIdx.x * kEcfChunk;
  const int64_t v1 = v0 + kEcfChunk < HW ? v0 + kEcfChunk : HW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kEcfWarps * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  const uint8_t* src = img + b * HW;
  const uint32_t hs = (uint32_t)__cvta_generic_to_shared(&hist[warp][0]);
  auto px = [&](int64_t u) -> int { return __ldg(src + u); };
  auto add = [&](int c, int s) { asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(hs + 4u * c), "r"(s) : "memory"); };
  unsigned mx = 0;
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    int x, y, z;
    if (HW < ((int64_t)1 << 31)) {  // 32-bit index math (the common case)
      const int vi = (int)v, yz = vi / X;
      x = vi - yz * X;
      y = yz % Y;
      z = yz / Y;
    } else {
      x = (int)(v % X);
      const int64_t yz = v / X;
      y = (int)(yz % Y);
      z = (int)(yz / Y);
    }
    ecf_anchor<ND>(px, v, x, y, z, X, Y, Z, add);
    const unsigned a = src[v];
    mx = a > mx ? a : mx;
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) atomicMax(&smax, mx);
  __syncthreads();
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kEcfWarps; ++w) s += hist[w][c];
    if (s != 0) atomicAdd(ghist + b * 256 + c, (unsigned long long)(long long)s);
  }
  if (threadIdx.x == 0) atomicMax(gmax + b, smax);
}

// Large 2-D images with W % 4 == 0: the packed u16x2 anchor step of k_ecf_img2d_w4 over a
// block of kEcfRows rows per CTA (plus the next row as halo; a sink row below the last),
// staged in shared memory with coalesced 4-byte loads; per-warp histograms merged into the
// int64 [B][256] table, the block's max intensity into gmax.
constexpr int kEcfRows = 16;

__global__ void __launch_bounds__(kEcfWarps * 32) k_ecf_img2d_rows(const uint8_t* __restrict__ img, int H, int W,
                                                                   unsigned long long* __restrict__ ghist,
                                                                   unsigned int* __restrict__ gmax) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int P2 = (W + 2) >> 1, W2 = W >> 1, W4 = W >> 2;
  const int64_t b = blockIdx.y;
  const int r0 = blockIdx.x * kEcfRows;
  const int R = (H - r0) < kEcfRows ? (H - r0) : kEcfRows;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  unsigned char* hbase = smem + (((s0 + 2047u) & ~2047u) - s0);
  int* hist = (int*)(hbase + (size_t)warp * 2048);
  uint32_t* S = (uint32_t*)(hbase + kEcfWarps * 2048);  // [(R + 1)][P2] words
  const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(hist);
  __shared__ unsigned int smax;
  if (threadIdx.x == 0) smax = 0;
  for (int k = lane; k < 256; k += 32) hist[k] = 0;
  // stage rows r0 .. r0 + R (the last one the halo, or the sink row below the image)
  const uint32_t* src = (const uint32_t*)(img + (b * H + r0) * (int64_t)W);
  unsigned mx = 0;
  for (int i = threadIdx.x; i < (R + 1) * W4; i += blockDim.x) {
    const int rr = i / W4, q = i - rr * W4;
    uint32_t lo = (uint32_t)kSinkOff | ((uint32_t)kSinkOff << 16), hi = lo;
    if (r0 + rr < H) {
      const uint32_t wv = __ldcs(src + (int64_t)rr * W4 + q);
      lo = __byte_perm(wv, 0, 0x4140) << 2;
      hi = __byte_perm(wv, 0, 0x4342) << 2;
      if (rr < R) mx = __vmaxu4(mx, wv);
    }
    S[rr * P2 + 2 * q] = lo;
    S[rr * P2 + 2 * q + 1] = hi;
  }
  for (int rr = threadIdx.x; rr < R + 1; rr += blockDim.x)  // the padding column of every row
    S[rr * P2 + W2] = (uint32_t)kSinkOff | ((uint32_t)kSinkOff << 16);
  mx = max(max(mx & 0xFFu, (mx >> 8) & 0xFFu), max((mx >> 16) & 0xFFu, mx >> 24));
  mx = __reduce_max_sync(0xffffffffu, mx);
  __syncthreads();
  if (lane == 0) atomicMax(&smax, mx);
  const int nitems = R * W2;
  for (int it = warp * 32 + lane; it < nitems; it += blockDim.x) {
    const int r = it / W2, xp = it - r * W2;
    const int ai = r * P2 + xp;
    const uint32_t a2 = S[ai], an = S[ai + 1], c2 = S[ai + P2], cn = S[ai + P2 + 1];
    const uint32_t b2 = __byte_perm(a2, an, 0x5432), d2 = __byte_perm(c2, cn, 0x5432);
    const uint32_t m_x = __vmaxu2(a2, b2), m_y = __vmaxu2(a2, c2);
    const uint32_t m_xy = __vmaxu2(m_x, __vmaxu2(c2, d2));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t A = (h ? a2 >> 16 : a2 & 0xFFFFu) | wbase;
      const uint32_t X = (h ? m_x >> 16 : m_x & 0xFFFFu) | wbase;
      const uint32_t Y = (h ? m_y >> 16 : m_y & 0xFFFFu) | wbase;
      const uint32_t XY = (h ? m_xy >> 16 : m_xy & 0xFFFFu) | wbase;
      if (X != A) {
        asm volatile("red.shared.add.s32 [%0], 1;" ::"r"(A) : "memory");
        asm volatile("red.shared.add.s32 [%0], -1;" ::"r"(X) : "memory");
      }
      if (XY != Y) {
        asm volatile("red.shared.add.s32 [%0], -1;" ::"r"(Y) : "memory");
        asm volatile("red.shared.add.s32 [%0], 1;" ::"r"(XY) : "memory");
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    int sum = 0;
#pragma unroll
    for (int w8 = 0; w8 < kEcfWarps; ++w8) sum += ((const int*)(hbase + (size_t)w8 * 2048))[c];
    if (sum != 0) atomicAdd(ghist + b * 256 + c, (unsigned long long)(long long)sum);
  }
  if (threadIdx.x == 0) atomicMax(gmax + b, smax);
}

template <typename OutT>
__global__ void __launch_bounds__(kEcfWarps * 32) k_ecf_img_final(const unsigned long long* __restrict__ ghist,
                                                                  const unsigned int* __restrict__ gmax, int64_t B,
                                                                  int per_image_M, const int16_t* __restrict__ cstar,
                                                                  int T, OutT* __restrict__ out) {
  __shared__ long long hist[kEcfWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kEcfWarps + warp;
  if (b >= B) return;
  for (int c = lane; c < 256; c += 32) hist[warp][c] = (long long)ghist[b * 256 + c];
  __syncwarp();
  const int M = per_image_M ? (int)gmax[b] : 0;
  ecf_scan_emit<long long, OutT>(&hist[warp][0], lane, cstar + (int64_t)M * T, T, out + b * T);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
size_t ecf_images_scratch_bytes(int64_t B, int64_t nv, int T, bool per_image_M) {
  size_t s = (size_t)(per_image_M ? 256 : 1) * T * sizeof(int16_t);
  s = (s + 255) & ~(size_t)255;
  if (nv > kEcfSmallMax) s += (size_t)B * 256 * 8 + (size_t)B * 4 + 256;
  return s;
}

template <typename OutT>
static wect_status launch_ecf_images_t(const uint8_t* img, int64_t B, int ndim, const int64_t* dims, int T, int mode,
                                       double lo, double hi, void* scratch, OutT* out, cudaStream_t st, int num_sms) {
  // dims: {H, W} or {Z, Y, X}; X is the fastest axis
  const int X = (int)dims[ndim - 1], Y = (int)dims[ndim - 2], Z = ndim == 3 ? (int)dims[0] : 1;
  const int64_t nv = (int64_t)X * Y * Z;
  const int per_image_M = mode == 0;
  int16_t* cstar = (int16_t*)scratch;
  k_ecf_cstar<<<per_image_M ? 256 : 1, 256, 0, st>>>(mode, lo, hi, T, cstar); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  size_t off = ((size_t)(per_image_M ? 256 : 1) * T * sizeof(int16_t) + 255) & ~(size_t)255;
  if (ndim == 2 && X % 4 == 0 && nv <= 1024 && nv % 16 == 0 && ((uintptr_t)img & 15) == 0) {
    const int pwords = (Y + 1) * ((X + 2) >> 1);
    const size_t smem = (size_t)kEcfWarps * ((pwords + 3) & ~3) * 4 + 2048 + (size_t)kEcfWarps * 2048;
    const int64_t ctas_needed = (B + kEcfWarps - 1) / kEcfWarps;
    const int64_t cap = (int64_t)num_sms * 8;
    const int grid = (int)(ctas_needed < cap ? ctas_needed : cap);
    MainTimer timer(st);
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_ecf_img2d_w4<OutT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_ecf_img2d_w4<OutT><<<grid, kEcfWarps * 32, smem, st>>>(img, B, Y, X, per_image_M, cstar, T, out);
    count_launch();
    timer.stop();
    WECT_CUDA_TRY(cudaGetLastError());
    return WECT_OK;
  }
  if (nv <= kEcfSmallMax) {
    const int pbytes = (int)((nv + 15) & ~15);
    const size_t smem = (size_t)kEcfWarps * (1024 + pbytes);
    const int64_t ctas_needed = (B + kEcfWarps - 1) / kEcfWarps;
    int per_sm = (int)((200 * 1024) / smem);
    per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
    const int64_t cap = (int64_t)num_sms * per_sm;
    const int grid = (int)(ctas_needed < cap ? ctas_needed : cap);
    MainTimer timer(st);
    if (ndim == 2) {
      WECT_CUDA_TRY(cudaFuncSetAttribute(k_ecf_img_small<2, OutT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_ecf_img_small<2, OutT><<<grid, kEcfWarps * 32, smem, st>>>(img, B, X, Y, 1, per_image_M, cstar, T, out);
    } else {
      WECT_CUDA_TRY(cudaFuncSetAttribute(k_ecf_img_small<3, OutT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_ecf_img_small<3, OutT><<<grid, kEcfWarps * 32, smem, st>>>(img, B, X, Y, Z, per_image_M, cstar, T, out);
    }
    count_launch();
    timer.stop();
    WECT_CUDA_TRY(cudaGetLastError());
    return WECT_OK;
  }
  unsigned long long* ghist = (unsigned long long*)((char*)scratch + off);
  unsigned int* gmax = (unsigned int*)(ghist + (size_t)B * 256);
  WECT_CUDA_TRY(cudaMemsetAsync(ghist, 0, (size_t)B * 256 * 8 + (size_t)B * 4, st));
  // the rows kernel stages kEcfRows + 1 image rows: only when they fit the opt-in shared memory
  const size_t rows_smem = 2048 + (size_t)kEcfWarps * 2048 + (size_t)(kEcfRows + 1) * ((X + 2) >> 1) * 4;
  int smem_optin = 0;
  {
    int dev = 0;
    WECT_CUDA_TRY(cudaGetDevice(&dev));
    WECT_CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  }
  const bool rows_path = ndim == 2 && X % 4 == 0 && X <= 16384 && ((uintptr_t)img & 3) == 0 &&
                         rows_smem <= (size_t)smem_optin && !getenv("WECT_ECF_GENERIC");
  if (rows_path) {
    const size_t smem = rows_smem;
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_ecf_img2d_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 g((unsigned)((Y + kEcfRows - 1) / kEcfRows), (unsigned)B);
    MainTimer timer(st);
    k_ecf_img2d_rows<<<g, kEcfWarps * 32, smem, st>>>(img, Y, X, ghist, gmax);
    count_launch();
    timer.stop();
  } else {
    dim3 g((unsigned)((nv + kEcfChunk - 1) / kEcfChunk), (unsigned)B);
    MainTimer timer(st);
    if (ndim == 2) k_ecf_img_hist<2><<<g, 256, 0, st>>>(img, X, Y, 1, ghist, gmax);
    else k_ecf_img_hist<3><<<g, 256, 0, st>>>(img, X, Y, Z, ghist, gmax);
    count_launch();
    timer.stop();
  }
  WECT_CUDA_TRY(cudaGetLastError());
  k_ecf_img_final<OutT><<<(unsigned)((B + kEcfWarps - 1) / kEcfWarps), kEcfWarps * 32, 0, st>>>(
      ghist, gmax, B, per_image_M, cstar, T, out); count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_ecf_images(const uint8_t* img, int64_t B, int ndim, const int64_t* dims, int T, int mode,
                              double lo, double hi, void* scratch, void* out, wect_dtype odtype, cudaStream_t st,
                              int num_sms) {
  if (odtype == WECT_I32)
    return launch_ecf_images_t<int32_t>(img, B, ndim, dims, T, mode, lo, hi, scratch, (int32_t*)out, st, num_sms);
  return launch_ecf_images_t<long long>(img, B, ndim, dims, T, mode, lo, hi, scratch, (long long*)out, st, num_sms);
}

}  // namespace wect
