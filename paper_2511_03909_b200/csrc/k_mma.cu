// k_mma.cu -- the image-batch WECT (wect_images, 2-D cubical) as a tensor-core contraction
// on the 5th-generation tensor cores (tcgen05 / TMEM), SURVEY §8(f) NEXT-4(ii).  Opt-in
// (WECT_IMAGES_MMA=1): measured slower than the sweep on BASELINE configs[1].
//
// For a direction s the cumulative WECT of image b is (Alg. 1, with the exact
// orthant regrouping of DESIGN.md: every cubical cell lands in the bin of one designated
// corner, so cw_o(b, v) -- the signed weights of the cells designating vertex v, o the
// quadrant of s -- is all that matters):
//
//     out[b, s, q] = sum_v cw_o(b, v) [bin(v, s) <= q]          (q = 0 .. T-1)
//
// i.e. per quadrant one GEMM  C[b, (s, q)] = A_o[b, v] . Ind_o[v, (s, q)]  with M = images,
// K = vertices, N = (direction, bin).  Both operands are exact in fp16 (|cw| <= 510; the
// indicator is 0/1) and every partial sum is an integer below 2^24, exact in the fp32
// accumulator, so the contraction is bit-exact for any summation order.  A holds
// 1536 + cw (its fp16 bit pattern is 0x6600 + cw: an integer add); the constant part,
// 1536 x #{v : bin(v, s) <= q}, is image-independent and removed in the epilogue.
//
//   k_mma_dirs   per direction: exact binary64 vertex bins (alpha64, reading A1), the
//                cumulative vertex counts, the quadrant lists
//   k_mma_passes passes = up to 256 / Tq directions of one quadrant (N = 256 columns)
//   k_mma_bimg   the indicator operand of every (pass, K chunk) in the canonical K-major
//                SWIZZLE_64B layout, and the epilogue constants
//   k_mma2d      persistent CTAs over (128-image tile, quadrant) units, warp-specialised:
//                8 builder warps write A_o chunks (32 vertices, 8 KB fp16) from the staged
//                pixels straight into swizzled shared memory; one thread issues
//                tcgen05.mma (M = 128, N = 256, K = 16) -- each A chunk feeds two passes, into
//                TMEM columns 0-255 and 256-511; one thread streams the B chunks in by
//                cp.async.bulk (3-stage ring); 8 epilogue warps read TMEM (tcgen05.ld),
//                remove the constant with one fp32 add and store int32 / int64.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "async.cuh"

namespace wect {

constexpr int kMmaM = 128;      // images per tile = UMMA M = TMEM lanes
constexpr int kMmaKC = 32;      // vertices per K chunk: 64 bytes of fp16 (one SWIZZLE_64B row)
constexpr int kMmaNmax = 256;   // accumulator columns (UMMA N)
constexpr int kMmaBuildWarps = 8;
constexpr int kMmaEpiWarps = 8;
constexpr int kMmaMmaWarp = kMmaBuildWarps + kMmaEpiWarps;  // the MMA issuer; + 1: the B loader
constexpr int kMmaThreads = (kMmaMmaWarp + 2) * 32;
constexpr int kMmaPassCols = 10;  // pass table row: quadrant, #directions, <= 8 direction ids
constexpr float kMmaMagic = 12582912.0f;  // 1.5 2^23: x + magic has x's integer in its low bits
constexpr uint32_t kMmaOff = 0x66006600u;  // fp16 1536 in both halves

__host__ __device__ constexpr int mma_tq(int T) { return (T + 31) & ~31; }
__host__ __device__ constexpr int mma_dpp(int T) { return kMmaNmax / mma_tq(T); }
__host__ __device__ constexpr int mma_n(int T) { return mma_dpp(T) * mma_tq(T); }
__host__ __device__ constexpr int mma_kc(int HW) { return (HW + kMmaKC - 1) / kMmaKC; }
// pixel row stride: >= HW + 4 (the funnel reads one word past the image), odd word count
// (32 images' words at one offset hit 32 banks)
__host__ __device__ constexpr int mma_ps(int HW) { return ((HW + 4 + 3) & ~3) + ((((HW + 7) >> 2) & 1) ? 0 : 4); }
constexpr size_t kMmaAStageBytes = (size_t)kMmaM * kMmaKC * 2;        // 8 KB
constexpr size_t kMmaBStageBytes = (size_t)kMmaNmax * kMmaKC * 2;     // 16 KB
__host__ __device__ constexpr size_t mma_smem_bytes(int HW) {
  return 1024 + 3 * kMmaAStageBytes + 3 * 2 * kMmaBStageBytes + (size_t)kMmaM * mma_ps(HW) + (size_t)(HW / 4 + 2) * 4 +
         128 + 16;
}

// ---- PTX wrappers (tcgen05, sm_100a)
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  // K-major, SWIZZLE_64B: 8-row atoms of 64-byte rows, atoms 512 B apart (SBO); LBO unused
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bar_builders() { asm volatile("bar.sync 1, %0;" ::"n"(kMmaBuildWarps * 32) : "memory"); }

#define WECT_TMEM_LD32(taddr, r)                                                                                  \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                  \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),     \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),   \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])    \
      : "r"(taddr))

// ---------------------------------------------------------------------------
// per direction (one CTA each): exact vertex bins, cumulative counts, quadrant list
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_mma_dirs(int H, int W, const float* __restrict__ dirs, int d_begin, int Dc,
                                                  const GridParams* __restrict__ gp, uint16_t* __restrict__ vbin,
                                                  int* __restrict__ cum, int* __restrict__ qcount,
                                                  int* __restrict__ qlist) {
  extern __shared__ int cnt[];  // [T]
  const GridParams g = *gp;
  const int T = g.T, HW = H * W, dl = blockIdx.x, p = d_begin + dl;
  const float sx = dirs[2 * p], sy = dirs[2 * p + 1];
  const int maxd = H > W ? H : W;
  const double S = (double)(maxd - 1 > 1 ? maxd - 1 : 1);
  for (int q = threadIdx.x; q < T; q += blockDim.x) cnt[q] = 0;
  __syncthreads();
  for (int v = threadIdx.x; v < HW; v += blockDim.x) {
    const int r = v / W, c = v - r * W;
    const double h = __dadd_rn(__dmul_rn((double)axis_coord(c, W, S), (double)sx),
                               __dmul_rn((double)axis_coord(r, H, S), (double)sy));
    const int bq = alpha64(h, g);
    vbin[(int64_t)dl * HW + v] = (uint16_t)bq;
    atomicAdd(&cnt[bq], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int q = 0; q < T; ++q) {
      run += cnt[q];
      cum[(int64_t)dl * T + q] = run;
    }
    const int o = (sx > 0.f ? 1 : 0) | (sy > 0.f ? 2 : 0);
    qlist[o * Dc + atomicAdd(&qcount[o], 1)] = dl;
  }
}

// pass table: consecutive groups of <= dpp directions of one quadrant, quadrant by
// quadrant; info = {#passes, first pass of quadrant 0..3, #passes of quadrant 0..3}
__global__ void k_mma_passes(const int* __restrict__ qcount, const int* __restrict__ qlist, int Dc, int dpp,
                             int* __restrict__ tab, int* __restrict__ info) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int np = 0;
  for (int o = 0; o < 4; ++o) {
    info[1 + o] = np;
    for (int j = 0; j < qcount[o]; j += dpp) {
      int* t = tab + np * kMmaPassCols;
      const int nd = qcount[o] - j < dpp ? qcount[o] - j : dpp;
      t[0] = o;
      t[1] = nd;
      for (int k = 0; k < nd; ++k) t[2 + k] = qlist[o * Dc + j + k];
      ++np;
    }
    info[5 + o] = np - info[1 + o];
  }
  info[0] = np;
}

// B operand of (pass, K chunk): rows n = j Tq + q, 32 vertices per row, fp16 1.0 where
// bin(v, s_j) <= q; canonical K-major SWIZZLE_64B image (16-byte chunk c of row n at
// n 64 + 16 (c ^ ((n >> 1) & 3))).  Block (p, kc); kc == 0 also writes the epilogue
// constants cfix[p][n] = 1.5 2^23 - 1536 #{v : bin(v, s_j) <= q}.
__global__ void __launch_bounds__(256) k_mma_bimg(int HW, int T, int Tq, int N, int KC, const int* __restrict__ npass,
                                                  const int* __restrict__ tab, const uint16_t* __restrict__ vbin,
                                                  const int* __restrict__ cum, uint4* __restrict__ bimg,
                                                  float* __restrict__ cfix) {
  const int p = blockIdx.x / KC, kc = blockIdx.x - p * KC;
  if (p >= *npass) return;
  const int* t = tab + p * kMmaPassCols;
  const int nd = t[1];
  uint4* img = bimg + ((int64_t)p * KC + kc) * (N * kMmaKC * 2 / 16);
  for (int e = threadIdx.x; e < N * 4; e += blockDim.x) {
    const int n = e >> 2, c = e & 3;
    const int j = n / Tq, q = n - j * Tq;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    if (j < nd && q < T) {
      const uint16_t* vb = vbin + (int64_t)t[2 + j] * HW;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int v = kc * kMmaKC + c * 8 + k;
        if (v < HW && (int)vb[v] <= q) w[k >> 1] |= 0x3C00u << (16 * (k & 1));
      }
    }
    img[n * 4 + (c ^ ((n >> 1) & 3))] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (kc == 0)
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const int j = n / Tq, q = n - j * Tq;
      cfix[(int64_t)p * N + n] =
          (j < nd && q < T) ? kMmaMagic - 1536.f * (float)cum[(int64_t)t[2 + j] * T + q] : kMmaMagic;
    }
}

// ---------------------------------------------------------------------------
// the contraction.  Work unit = (128-image tile, quadrant): its passes run in pairs, one
// A_o chunk feeding two accumulators (TMEM columns 0-255 and 256-511), so every built A
// chunk serves 4 MMAs (2 x K 16, 2 passes).  Iteration i = (unit, pass pair, K chunk) in
// order; A stage i % 3, B stage i % 3 (the B stage holds both passes' 16 KB chunks).
// Barriers: afull[s] (256 builder arrivals), bfull[s] (bulk-copy bytes), adone[s]
// (tcgen05.commit after the MMAs that read stage s: waited by builders and the B loader), accf (commit after a pair's
// last MMAs), tfree (256 arrivals: the epilogue has read TMEM).
// ---------------------------------------------------------------------------
constexpr int kMmaStages = 3;
struct MmaCursor {  // position in this CTA's (unit, pass pair, chunk) sequence
  int64_t unit;
  int pp, kc;
};

template <typename OutT>
__global__ void __launch_bounds__(kMmaThreads, 1)
    k_mma2d(const uint8_t* __restrict__ img, int64_t B, int H, int W, int T, int Tq, int N, int KC, int Dc,
            const int* __restrict__ info, const int* __restrict__ tab, const uint4* __restrict__ bimg,
            const float* __restrict__ cfix, OutT* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  const int HW = H * W, PS = mma_ps(HW), NG = HW >> 2;  // W % 4 == 0: vertex groups of 4 lie in one row
  uint8_t* As = smem;                                              // [3][128 rows][64 B]
  uint8_t* Bs = As + kMmaStages * kMmaAStageBytes;                 // [3][2 passes][N rows][64 B]
  uint8_t* pix = Bs + kMmaStages * 2 * kMmaBStageBytes;            // [128][PS]
  uint32_t* ginfo = (uint32_t*)(pix + (size_t)kMmaM * PS);         // [NG]: r | c << 16
  uint64_t* bars = (uint64_t*)(ginfo + NG + 1 + ((NG + 1) & 1));  // 8-aligned
  uint64_t* afull = bars;
  uint64_t* adone = bars + 3;
  uint64_t* bfull = bars + 6;
  uint64_t* accf = bars + 12;
  uint64_t* tfree = bars + 13;
  uint32_t* tmem_hold = (uint32_t*)(bars + 14);
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int64_t ntiles = (B + kMmaM - 1) / kMmaM, nunits = ntiles * 4;
  const unsigned bbytes = (unsigned)(N * kMmaKC * 2);
  __shared__ int qf[4], qn[4];  // first pass / #passes of each quadrant
  if (tid < 4) {
    qf[tid] = info[1 + tid];
    qn[tid] = info[5 + tid];
  }
  __syncthreads();
  // this CTA's units: a contiguous range, so the 4 quadrant units of a tile mostly follow
  // each other and share one pixel staging; units without passes are skipped
  const int64_t u_end = nunits * (blockIdx.x + 1) / gridDim.x;
  auto npp = [&](int64_t u) { return (qn[(int)(u & 3)] + 1) >> 1; };
  auto first = [&](int64_t u) -> MmaCursor {
    while (u < u_end && npp(u) == 0) ++u;
    return MmaCursor{u < u_end ? u : nunits, 0, 0};
  };
  auto advance = [&](MmaCursor& c) {
    if (++c.kc < KC) return;
    c.kc = 0;
    if (++c.pp < npp(c.unit)) return;
    c = first(c.unit + 1);
  };
  const int64_t u_begin = nunits * blockIdx.x / gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < kMmaStages; ++s) {
      mbar_init(afull + s, kMmaBuildWarps * 32);
      mbar_init(adone + s, 1);
      mbar_init(bfull + s, 1);
    }
    mbar_init(accf, 1);
    mbar_init(tfree, kMmaEpiWarps * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // per vertex group of 4 (one row): bit 0 row r + 1 exists, bit 1 row r - 1 exists, bit 2 the
  // group ends its row (c + 3 = W - 1), bit 3 it starts its row (c = 0)
  for (int gi = tid; gi < NG; gi += blockDim.x) {
    const int v = gi * 4, r = v / W, c = v - r * W;
    ginfo[gi] = (r + 1 < H ? 1u : 0u) | (r >= 1 ? 2u : 0u) | (c + 4 == W ? 4u : 0u) | (c == 0 ? 8u : 0u);
  }
  for (int e = tid; e < kMmaM * (PS >> 2); e += blockDim.x) ((uint32_t*)pix)[e] = 0u;
  if (warp == kMmaMmaWarp) {  // TMEM: 2 x 256 fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_hold)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_hold;

  if (warp == kMmaMmaWarp) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kMmaM >> 4) << 24);
      MmaCursor cur = first(u_begin);
      int s = 0;
      unsigned ph = 0u;
      int64_t pairs = 0;
      for (; cur.unit < nunits; advance(cur)) {
        const int o = (int)(cur.unit & 3);
        const bool two = 2 * cur.pp + 1 < qn[o];
        if (cur.kc == 0 && pairs > 0) mbar_wait(tfree, (unsigned)((pairs - 1) & 1));  // TMEM read out
        mbar_wait(afull + s, ph);
        mbar_wait(bfull + s, ph);
        tc_fence_after();
        const uint32_t a0 = smem_u32(As + s * kMmaAStageBytes), b0 = smem_u32(Bs + s * 2 * kMmaBStageBytes);
#pragma unroll
        for (int k = 0; k < kMmaKC / 16; ++k) {
          const uint64_t ad = umma_desc_sw64(a0 + 32 * k);
          const uint32_t acc = (cur.kc > 0 || k > 0) ? 1u : 0u;
          umma_f16(tmem, ad, umma_desc_sw64(b0 + 32 * k), idesc, acc);
          if (two) umma_f16(tmem + 256, ad, umma_desc_sw64(b0 + (uint32_t)kMmaBStageBytes + 32 * k), idesc, acc);
        }
        umma_commit(adone + s);  // stage s (its A and B halves) free again
        if (cur.kc == KC - 1) {
          umma_commit(accf);
          ++pairs;
        }
        if (++s == kMmaStages) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaMmaWarp + 1) {
    // ---------------- B loader (one thread): stage s refilled once the MMAs that read it are done
    if (lane == 0) {
      MmaCursor ld = first(u_begin);
      int s = 0;
      unsigned ph = 0u;
      bool warm = false;
      for (; ld.unit < nunits; advance(ld)) {
        if (warm) mbar_wait(adone + s, ph);
        const int o = (int)(ld.unit & 3), p0 = qf[o] + 2 * ld.pp;
        const int two = (2 * ld.pp + 1 < qn[o]) ? 2 : 1;
        mbar_arrive_expect_tx(bfull + s, bbytes * two);
        for (int h = 0; h < two; ++h)
          bulk_g2s_plain(Bs + (s * 2 + h) * kMmaBStageBytes, bimg + ((int64_t)(p0 + h) * KC + ld.kc) * (bbytes / 16),
                         bbytes, bfull + s);
        if (++s == kMmaStages) {
          s = 0;
          if (warm) ph ^= 1u;
          warm = true;
        }
      }
    }
    __syncwarp();
  } else if (warp < kMmaBuildWarps) {
    // ---------------- builders (8 warps): A row b, 16-byte chunks 2 (warp / 4) + {0, 1}
    const int b = tid & (kMmaM - 1);
    const uint32_t* pw = (const uint32_t*)(pix + (size_t)b * PS);
    int s = 0;          // A stage of the next iteration
    unsigned aph = 0u;  // parity of the adone completion awaited for stage s
    bool warm = false;  // every stage has been used once (adone waits begin)
    int64_t staged = -1;
    for (MmaCursor cur = first(u_begin); cur.unit < nunits;) {
      const int64_t tile = cur.unit >> 2;
      const int o = (int)(cur.unit & 3);
      const int64_t img0 = tile * kMmaM;
      const int nimg = (int)((B - img0) < kMmaM ? (B - img0) : kMmaM);
      if (staged != tile) {  // stage the tile's pixels (row b = image img0 + b)
        bar_builders();      // the previous unit's builds are done with pix
        // the tile's images are one contiguous block: 16-byte loads, 8 in flight per thread,
        // stored as words into the padded rows (the row pads were zeroed at kernel start)
        if ((HW & 15) == 0 && ((uintptr_t)img & 15) == 0) {
          const int n16 = (int)(((int64_t)nimg * HW) >> 4);
          const uint4* src = (const uint4*)(img + img0 * HW);
          for (int e0 = tid; e0 < n16; e0 += 8 * kMmaBuildWarps * 32) {
            uint4 x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int e = e0 + k * kMmaBuildWarps * 32;
              x[k] = e < n16 ? __ldg(src + e) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int e = e0 + k * kMmaBuildWarps * 32;
              if (e < n16) {
                const int byte = 16 * e, bb = byte / HW, off = byte - bb * HW;  // HW % 16 == 0
                uint32_t* d = (uint32_t*)(pix + (size_t)bb * PS + off);
                d[0] = x[k].x;
                d[1] = x[k].y;
                d[2] = x[k].z;
                d[3] = x[k].w;
              }
            }
          }
        } else {
          for (int e = tid; e < nimg * (HW >> 2); e += kMmaBuildWarps * 32) {
            const int bb = e / (HW >> 2), wi = e - bb * (HW >> 2);
            ((uint32_t*)(pix + (size_t)bb * PS))[wi] = __ldg((const uint32_t*)(img + (img0 + bb) * HW) + wi);
          }
        }
        // rows of missing images (last tile) read as zeros
        for (int e = nimg * (PS >> 2) + tid; e < kMmaM * (PS >> 2); e += kMmaBuildWarps * 32) ((uint32_t*)pix)[e] = 0u;
        bar_builders();
        staged = tile;
      }
      const bool cpos = (o & 1) == 0;  // column neighbour c + 1 (else c - 1)
      const int dr = (o & 2) ? -1 : 1;
      const uint32_t rbit = dr > 0 ? 1u : 2u, cbit = cpos ? 4u : 8u;
      const int rstep = dr * (W >> 2);
      const int np2 = npp(cur.unit);
      for (int pp = 0; pp < np2; ++pp) {
        for (int kc = 0; kc < KC; ++kc) {
          if (warm) mbar_wait(adone + s, aph);  // the MMAs of 3 iterations ago read A stage s
#pragma unroll
          for (int half = 0; half < 2; ++half) {
          const int part = 2 * (warp >> 2) + half;  // warp-uniform
          // vertices v0 .. v0 + 7 (two groups of 4) of image b -> 16-byte chunk `part` of A row b,
          // per vertex pair in u16x2 lanes: fp16 bits 0x6600 + (x + md - mc - mr)
          const int v0 = kc * kMmaKC + 8 * part;
          uint32_t wv[4] = {0u, 0u, 0u, 0u};
          if (v0 < HW) {
            const int g0 = v0 >> 2;
            const bool two = v0 + 4 < HW;
            const uint32_t f0 = ginfo[g0], f1 = two ? ginfo[g0 + 1] : 0u;
            const uint32_t Xm = pw[g0 - 1], Xa = pw[g0], Xb = pw[g0 + 1], Xn = pw[g0 + 2];
            // widened pixels: (b0, b1) / (b2, b3) of each word as u16x2
            const uint32_t A0 = __byte_perm(Xa, 0, 0x4140), A1 = __byte_perm(Xa, 0, 0x4342);
            const uint32_t B0 = __byte_perm(Xb, 0, 0x4140), B1 = __byte_perm(Xb, 0, 0x4342);
            // column neighbours: c + 1 -> (x1, x2), (x3, next x0); c - 1 -> (prev x3, x0), (x1, x2)
            uint32_t CA0, CA1, CB0, CB1;
            if (cpos) {
              CA0 = __byte_perm(Xa, 0, 0x4241);
              CA1 = __byte_perm(Xa, B0, 0x5453);
              CB0 = __byte_perm(Xb, 0, 0x4241);
              CB1 = __byte_perm(Xb, __byte_perm(Xn, 0, 0x4140), 0x5453);
            } else {
              CA0 = __byte_perm(__byte_perm(Xm, 0, 0x4342), Xa, 0x3412);
              CA1 = __byte_perm(Xa, 0, 0x4241);
              CB0 = __byte_perm(A1, Xb, 0x3412);
              CB1 = __byte_perm(Xb, 0, 0x4241);
            }
            uint32_t MCA0 = __vmaxu2(A0, CA0), MCA1 = __vmaxu2(A1, CA1);
            uint32_t MCB0 = __vmaxu2(B0, CB0), MCB1 = __vmaxu2(B1, CB1);
            uint32_t MRA0 = 0u, MRA1 = 0u, MRB0 = 0u, MRB1 = 0u, MDA0 = 0u, MDA1 = 0u, MDB0 = 0u, MDB1 = 0u;
            if ((f0 | f1) & rbit) {  // the neighbour row exists for a group (the two may straddle rows)
              const uint32_t* pr = pw + g0 + rstep;
              const uint32_t Rm = pr[-1], Ra = pr[0], Rb = pr[1], Rn = pr[2];
              const uint32_t RA0 = __byte_perm(Ra, 0, 0x4140), RA1 = __byte_perm(Ra, 0, 0x4342);
              const uint32_t RB0 = __byte_perm(Rb, 0, 0x4140), RB1 = __byte_perm(Rb, 0, 0x4342);
              uint32_t DA0, DA1, DB0, DB1;
              if (cpos) {
                DA0 = __byte_perm(Ra, 0, 0x4241);
                DA1 = __byte_perm(Ra, RB0, 0x5453);
                DB0 = __byte_perm(Rb, 0, 0x4241);
                DB1 = __byte_perm(Rb, __byte_perm(Rn, 0, 0x4140), 0x5453);
              } else {
                DA0 = __byte_perm(__byte_perm(Rm, 0, 0x4342), Ra, 0x3412);
                DA1 = __byte_perm(Ra, 0, 0x4241);
                DB0 = __byte_perm(RA1, Rb, 0x3412);
                DB1 = __byte_perm(Rb, 0, 0x4241);
              }
              MRA0 = __vmaxu2(A0, RA0);
              MRA1 = __vmaxu2(A1, RA1);
              MRB0 = __vmaxu2(B0, RB0);
              MRB1 = __vmaxu2(B1, RB1);
              MDA0 = __vmaxu2(__vmaxu2(MCA0, RA0), DA0);
              MDA1 = __vmaxu2(__vmaxu2(MCA1, RA1), DA1);
              MDB0 = __vmaxu2(__vmaxu2(MCB0, RB0), DB0);
              MDB1 = __vmaxu2(__vmaxu2(MCB1, RB1), DB1);
              if (!(f0 & rbit)) MRA0 = MRA1 = MDA0 = MDA1 = 0u;
              if (!(f1 & rbit)) MRB0 = MRB1 = MDB0 = MDB1 = 0u;
            }
            if ((f0 | f1) & cbit) {  // a group at the row's end: its border vertex has no column neighbour
              const uint32_t keep = cpos ? 0x0000FFFFu : 0xFFFF0000u;
              if (f0 & cbit) {
                if (cpos) { MCA1 &= keep; MDA1 &= keep; } else { MCA0 &= keep; MDA0 &= keep; }
              }
              if (f1 & cbit) {
                if (cpos) { MCB1 &= keep; MDB1 &= keep; } else { MCB0 &= keep; MDB0 &= keep; }
              }
            }
            wv[0] = A0 + MDA0 + kMmaOff - MCA0 - MRA0;
            wv[1] = A1 + MDA1 + kMmaOff - MCA1 - MRA1;
            if (two) {
              wv[2] = B0 + MDB0 + kMmaOff - MCB0 - MRB0;
              wv[3] = B1 + MDB1 + kMmaOff - MCB1 - MRB1;
            }
          }
          *(uint4*)(As + s * kMmaAStageBytes + (size_t)b * 64 + 16 * (part ^ ((b >> 1) & 3))) =
              make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
          fence_async_smem();
          mbar_arrive(afull + s);
          if (++s == kMmaStages) {
            s = 0;
            if (warm) aph ^= 1u;
            warm = true;
          }
        }
      }
      cur = first(cur.unit + 1);
    }
  } else if (warp < kMmaMmaWarp) {
    // ---------------- epilogue (8 warps): warps 8-11 pass p0 (TMEM columns 0-255), 12-15 pass
    // p0 + 1 (256-511); lanes 32 (warp % 4) .. +31 = images of the tile
    const int ew = warp - kMmaBuildWarps;
    const int hp = ew >> 2;
    const int row = 32 * (ew & 3) + lane;
    int64_t pairs = 0;
    for (MmaCursor cur = first(u_begin); cur.unit < nunits;) {
      const int64_t tile = cur.unit >> 2;
      const int o = (int)(cur.unit & 3);
      const int64_t img0 = tile * kMmaM;
      const int nimg = (int)((B - img0) < kMmaM ? (B - img0) : kMmaM);
      const int64_t im = img0 + row;
      const int np2 = npp(cur.unit);
      for (int pp = 0; pp < np2; ++pp) {
        const int p = qf[o] + 2 * pp + hp;
        const bool live = p < qf[o] + qn[o];
        const int nd = live ? tab[p * kMmaPassCols + 1] : 0;
        mbar_wait(accf, (unsigned)(pairs & 1));
        ++pairs;
        tc_fence_after();
        for (int n0 = 0; n0 < N; n0 += 32) {
          uint32_t r[32];
          WECT_TMEM_LD32(tmem + ((uint32_t)(32 * (ew & 3)) << 16) + (uint32_t)(256 * hp + n0), r);
          const int j = n0 / Tq, q0 = n0 - j * Tq;
          const bool st = j < nd && q0 < T && row < nimg;
          float4 f[8];
          int dl = 0;
          if (j < nd && q0 < T) {
            dl = tab[p * kMmaPassCols + 2 + j];
            const float4* cf = (const float4*)(cfix + (int64_t)p * N + n0);
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4) f[k4] = __ldg(cf + k4);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (!st) continue;
          int vals[32];
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) {
            vals[4 * k4 + 0] = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 0]), f[k4].x)) - 0x4B400000;
            vals[4 * k4 + 1] = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 1]), f[k4].y)) - 0x4B400000;
            vals[4 * k4 + 2] = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 2]), f[k4].z)) - 0x4B400000;
            vals[4 * k4 + 3] = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 3]), f[k4].w)) - 0x4B400000;
          }
          OutT* dst = out + (im * Dc + dl) * (int64_t)T + q0;
          const int nq = T - q0 < 32 ? T - q0 : 32;
          if (nq == 32 && ((uintptr_t)dst & 15) == 0) {
            if (sizeof(OutT) == 4) {
#pragma unroll
              for (int k4 = 0; k4 < 8; ++k4)
                __stcs((int4*)dst + k4, make_int4(vals[4 * k4], vals[4 * k4 + 1], vals[4 * k4 + 2], vals[4 * k4 + 3]));
            } else {
#pragma unroll
              for (int k2 = 0; k2 < 16; ++k2)
                __stcs((longlong2*)dst + k2, make_longlong2(vals[2 * k2], vals[2 * k2 + 1]));
            }
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (k < nq) dst[k] = (OutT)vals[k];
          }
        }
        tc_fence_before();
        mbar_arrive(tfree);
      }
      cur = first(cur.unit + 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ===========================================================================
// Version 2 (WECT_IMAGES_MMA=2; v1 above is WECT_IMAGES_MMA=1).  What v1's measurements
// pointed at: the staged pixels (101 KB of shared memory) left room for 3 shallow stages, and
// the epilogue's 16-byte-per-image stores were slow.  v2 keeps no pixels in shared memory:
// a prepass writes each 128-image tile transposed, `pixT[tile][v][128 images]` u8, and the
// builders read it through L1 (lane = 4 images, one coalesced 128-byte line per vertex), so
// A is written MN-major (images contiguous: SWIZZLE_128B atoms of 64 images x 8 vertices).
// K chunks of 64 vertices (A 16 KB, B 32 KB per stage, 4 stages); one pass (N = 256) per
// accumulator, TMEM double-buffered (2 x 256 columns) so the epilogue of a pass overlaps the
// next pass's MMAs; 4 epilogue warps stage 32 images x 32 bins (128-byte rows, 128B swizzle)
// and write them with TMA tensor stores.  Bit-exact, but slower than v1 on cfg2 (3.31 vs
// 1.55 ms): the transposed-pixel reads miss L1 (the 4 stages leave ~30 KB of it) and stall
// the builders on L2 latency (58 % long-scoreboard), and streaming B per 128-image tile is
// 8 KB per M128-N256-K16 MMA, ~62 B/cycle per SM -- at or above the L2 share of an SM, so a
// contraction form needs 2-CTA (cta_group::2) B sharing / multicast before it can compete.
// ===========================================================================
constexpr int kM2K = 64;                                    // vertices per K chunk
constexpr int kM2Stages = 4;
constexpr int kM2Build = 8;                                 // builder warps: 8 vertices each
constexpr int kM2Epi = 4;                                   // epilogue warps: TMEM lanes 32 e ..
constexpr int kM2MmaWarp = kM2Build + kM2Epi;               // + 1: the B loader
constexpr int kM2Threads = (kM2MmaWarp + 2) * 32;
constexpr size_t kM2AStage = (size_t)kMmaM * kM2K * 2;      // 16 KB
constexpr size_t kM2BStage = (size_t)kMmaNmax * kM2K * 2;   // 32 KB
constexpr size_t kM2EStage = 32 * 128;                      // 4 KB: 32 images x 128 bytes
__host__ __device__ constexpr int m2_kc(int HW) { return (HW + kM2K - 1) / kM2K; }
__host__ __device__ constexpr size_t m2_smem_bytes() {
  return 1024 + kM2Stages * (kM2AStage + kM2BStage) + (size_t)kM2Epi * 2 * kM2EStage + 256;
}

// K-major SWIZZLE_128B (B: rows of 64 fp16 = 128 bytes, 8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t umma_desc_k128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// MN-major SWIZZLE_128B (A: atoms of 64 images (128 B) x 8 vertices; the two image atoms
// 1024 B apart (LBO), vertex atoms 2048 B apart (SBO))
__device__ __forceinline__ uint64_t umma_desc_mn128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(1024 >> 4) << 16) | ((uint64_t)(2048 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// transposed tiles: block (tile, 128-vertex slice); pixT[tile][v][i] = img[tile*128 + i][v]
__global__ void __launch_bounds__(256) k_mma2_pixt(const uint8_t* __restrict__ img, int64_t B, int HW,
                                                   uint8_t* __restrict__ pixT) {
  __shared__ uint8_t sm[128][129];
  const int64_t tile = blockIdx.x;
  const int v0 = blockIdx.y * 128;
  const int nv = HW - v0 < 128 ? HW - v0 : 128;
  for (int e = threadIdx.x; e < 128 * 128; e += blockDim.x) {
    const int i = e >> 7, v = e & 127;
    const int64_t im = tile * 128 + i;
    sm[i][v] = (im < B && v < nv) ? img[im * HW + v0 + v] : (uint8_t)0;
  }
  __syncthreads();
  uint32_t* dst = (uint32_t*)(pixT + (tile * HW + v0) * 128);
  for (int e = threadIdx.x; e < nv * 32; e += blockDim.x) {
    const int v = e >> 5, t = e & 31;
    dst[e] = (uint32_t)sm[4 * t][v] | ((uint32_t)sm[4 * t + 1][v] << 8) | ((uint32_t)sm[4 * t + 2][v] << 16) |
             ((uint32_t)sm[4 * t + 3][v] << 24);
  }
}

// vertex flags: bit 0 row r + 1 exists, bit 1 row r - 1, bit 2 column c + 1, bit 3 column c - 1
__global__ void k_mma2_vflags(int H, int W, uint8_t* __restrict__ vf) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < H * W; v += gridDim.x * blockDim.x) {
    const int r = v / W, c = v - r * W;
    vf[v] = (uint8_t)((r + 1 < H ? 1 : 0) | (r >= 1 ? 2 : 0) | (c + 1 < W ? 4 : 0) | (c >= 1 ? 8 : 0));
  }
}

// B operand of (pass, 64-vertex chunk): K-major SWIZZLE_128B rows n = j Tq + q
__global__ void __launch_bounds__(256) k_mma2_bimg(int HW, int T, int Tq, int N, int KC, const int* __restrict__ npass,
                                                   const int* __restrict__ tab, const uint16_t* __restrict__ vbin,
                                                   const int* __restrict__ cum, uint4* __restrict__ bimg,
                                                   float* __restrict__ cfix) {
  const int p = blockIdx.x / KC, kc = blockIdx.x - p * KC;
  if (p >= *npass) return;
  const int* t = tab + p * kMmaPassCols;
  const int nd = t[1];
  uint4* im = bimg + ((int64_t)p * KC + kc) * (N * kM2K * 2 / 16);
  for (int e = threadIdx.x; e < N * 8; e += blockDim.x) {
    const int n = e >> 3, c = e & 7;
    const int j = n / Tq, q = n - j * Tq;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    if (j < nd && q < T) {
      const uint16_t* vb = vbin + (int64_t)t[2 + j] * HW;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int v = kc * kM2K + c * 8 + k;
        if (v < HW && (int)vb[v] <= q) w[k >> 1] |= 0x3C00u << (16 * (k & 1));
      }
    }
    im[n * 8 + (c ^ (n & 7))] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (kc == 0)
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const int j = n / Tq, q = n - j * Tq;
      cfix[(int64_t)p * N + n] =
          (j < nd && q < T) ? kMmaMagic - 1536.f * (float)cum[(int64_t)t[2 + j] * T + q] : kMmaMagic;
    }
}

template <typename OutT>
__global__ void __launch_bounds__(kM2Threads, 1)
    k_mma2(const uint8_t* __restrict__ pixT, const uint8_t* __restrict__ vflags, int64_t B, int H, int W, int T,
           int Tq, int N, int KC, const int* __restrict__ info, const int* __restrict__ tab,
           const uint4* __restrict__ bimg, const float* __restrict__ cfix, const __grid_constant__ CUtensorMap omap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  const int HW = H * W;
  uint8_t* As = smem;                                     // [S][16 KB] MN-major
  uint8_t* Bs = As + kM2Stages * kM2AStage;               // [S][32 KB] K-major
  uint8_t* Es = Bs + kM2Stages * kM2BStage;               // [4 warps][2][4 KB] epilogue stages
  uint64_t* bars = (uint64_t*)(Es + kM2Epi * 2 * kM2EStage);
  uint64_t* afull = bars;                 // [S]
  uint64_t* bfull = bars + kM2Stages;     // [S]
  uint64_t* sdone = bars + 2 * kM2Stages; // [S]
  uint64_t* tfull = bars + 3 * kM2Stages; // [2]
  uint64_t* tempty = tfull + 2;           // [2]
  uint32_t* tmem_hold = (uint32_t*)(tempty + 2);
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int64_t ntiles = (B + kMmaM - 1) / kMmaM, nunits = ntiles * 4;
  const unsigned bbytes = (unsigned)(N * kM2K * 2);
  __shared__ int qf[4], qn[4];
  if (tid < 4) {
    qf[tid] = info[1 + tid];
    qn[tid] = info[5 + tid];
  }
  __syncthreads();
  const int64_t u_begin = nunits * blockIdx.x / gridDim.x, u_end = nunits * (blockIdx.x + 1) / gridDim.x;
  // sequence of (unit, pass, chunk); units without passes skipped
  struct Cur {
    int64_t unit;
    int p, kc;
  };
  auto first = [&](int64_t u) -> Cur {
    while (u < u_end && qn[(int)(u & 3)] == 0) ++u;
    return Cur{u < u_end ? u : nunits, 0, 0};
  };
  auto advance = [&](Cur& c) {
    if (++c.kc < KC) return;
    c.kc = 0;
    if (++c.p < qn[(int)(c.unit & 3)]) return;
    c = first(c.unit + 1);
  };
  if (tid == 0) {
    for (int s = 0; s < kM2Stages; ++s) {
      mbar_init(afull + s, kM2Build * 32);
      mbar_init(bfull + s, 1);
      mbar_init(sdone + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, kM2Epi * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kM2MmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_hold)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_hold;

  if (warp == kM2MmaWarp) {
    // ---------------- MMA issuer
    if (lane == 0) {
      // F32 accumulate, F16 A / B, A MN-major (bit 15), B K-major, N, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kMmaM >> 4) << 24);
      int s = 0;
      unsigned ph = 0u;
      int64_t npass = 0;  // passes started
      for (Cur c = first(u_begin); c.unit < nunits; advance(c)) {
        const int a = (int)(npass & 1);
        if (c.kc == 0 && npass >= 2) mbar_wait(tempty + a, (unsigned)(((npass >> 1) - 1) & 1));  // epilogue of pass - 2
        mbar_wait(afull + s, ph);
        mbar_wait(bfull + s, ph);
        tc_fence_after();
        const uint32_t a0 = smem_u32(As + s * kM2AStage), b0 = smem_u32(Bs + s * kM2BStage);
#pragma unroll
        for (int k = 0; k < kM2K / 16; ++k)
          umma_f16(tmem + 256 * a, umma_desc_mn128(a0 + 4096 * k), umma_desc_k128(b0 + 32 * k), idesc,
                   (c.kc > 0 || k > 0) ? 1u : 0u);
        umma_commit(sdone + s);
        if (c.kc == KC - 1) {
          umma_commit(tfull + a);
          ++npass;
        }
        if (++s == kM2Stages) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == kM2MmaWarp + 1) {
    // ---------------- B loader
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0u;
      bool warm = false;
      for (Cur c = first(u_begin); c.unit < nunits; advance(c)) {
        if (warm) mbar_wait(sdone + s, ph);
        const int p = qf[(int)(c.unit & 3)] + c.p;
        mbar_arrive_expect_tx(bfull + s, bbytes);
        bulk_g2s_plain(Bs + s * kM2BStage, bimg + ((int64_t)p * KC + c.kc) * (bbytes / 16), bbytes, bfull + s);
        if (++s == kM2Stages) {
          s = 0;
          if (warm) ph ^= 1u;
          warm = true;
        }
      }
    }
    __syncwarp();
  } else if (warp < kM2Build) {
    // ---------------- builders: warp w, vertices 8 w .. 8 w + 7 of each chunk; lane t, images 4t..4t+3
    const int t = lane;
    // MN-major A: element (image m, vertex k) at (k/8) 2048 + (m/64) 1024 + (k%8) 128 +
    // (((m%64)/8) ^ (k%8)) 16 + (m%8) 2; this lane's 4 images are 8 contiguous bytes
    const uint32_t mb = (uint32_t)(t >> 4) * 1024u, mc = (uint32_t)((t & 15) >> 1), me = (uint32_t)(t & 1) * 8u;
    int s = 0;
    unsigned ph = 0u;
    bool warm = false;
    for (Cur c = first(u_begin); c.unit < nunits; advance(c)) {
      if (warm) mbar_wait(sdone + s, ph);
      const int o = (int)(c.unit & 3);
      const int dc = (o & 1) ? -1 : 1, dr = (o & 2) ? -1 : 1;
      const uint32_t rbit = dr > 0 ? 1u : 2u, cbit = dc > 0 ? 4u : 8u;
      const uint32_t* px = (const uint32_t*)(pixT + (c.unit >> 2) * (int64_t)HW * 128) + t;  // [v][32 words]
      uint8_t* as = As + s * kM2AStage;
      // the warp's 8 vertices walked against dc: the column neighbour is the previous step
      const int vlo = c.kc * kM2K + 8 * warp;
      uint32_t Cp0 = 0u, Cp1 = 0u, Dp0 = 0u, Dp1 = 0u;
      {  // the first step's column neighbour (v + dc of the walk start)
        const int vs = dc > 0 ? vlo + 7 : vlo;
        const int vn = vs + dc;
        if (vn >= 0 && vn < HW) {
          const uint32_t X = __ldg(px + (int64_t)vn * 32);
          Cp0 = __byte_perm(X, 0, 0x4140);
          Cp1 = __byte_perm(X, 0, 0x4342);
          const int vr = vn + dr * W;
          if (vr >= 0 && vr < HW) {
            const uint32_t R = __ldg(px + (int64_t)vr * 32);
            Dp0 = __byte_perm(R, 0, 0x4140);
            Dp1 = __byte_perm(R, 0, 0x4342);
          }
        }
      }
#pragma unroll
      for (int st = 0; st < 8; ++st) {
        const int v = dc > 0 ? vlo + 7 - st : vlo + st;
        uint32_t lo = 0u, hi = 0u;  // fp16 of images (4t, 4t+1) and (4t+2, 4t+3)
        uint32_t A0 = 0u, A1 = 0u, R0 = 0u, R1 = 0u;
        if (v < HW) {
          const uint32_t f = __ldg(vflags + v);
          const uint32_t X = __ldg(px + (int64_t)v * 32);
          A0 = __byte_perm(X, 0, 0x4140);
          A1 = __byte_perm(X, 0, 0x4342);
          const bool hasr = (f & rbit) != 0, hasc = (f & cbit) != 0;
          if (hasr) {
            const uint32_t Rw = __ldg(px + (int64_t)(v + dr * W) * 32);
            R0 = __byte_perm(Rw, 0, 0x4140);
            R1 = __byte_perm(Rw, 0, 0x4342);
          }
          const uint32_t MC0 = hasc ? __vmaxu2(A0, Cp0) : 0u, MC1 = hasc ? __vmaxu2(A1, Cp1) : 0u;
          const uint32_t MR0 = hasr ? __vmaxu2(A0, R0) : 0u, MR1 = hasr ? __vmaxu2(A1, R1) : 0u;
          const uint32_t MD0 = (hasc && hasr) ? __vmaxu2(__vmaxu2(MC0, MR0), Dp0) : 0u;
          const uint32_t MD1 = (hasc && hasr) ? __vmaxu2(__vmaxu2(MC1, MR1), Dp1) : 0u;
          lo = A0 + MD0 + kMmaOff - MC0 - MR0;
          hi = A1 + MD1 + kMmaOff - MC1 - MR1;
        }
        Cp0 = A0;
        Cp1 = A1;
        Dp0 = R0;
        Dp1 = R1;
        const uint32_t k = (uint32_t)(v - c.kc * kM2K);  // 0..63 within the chunk
        const uint32_t r = k & 7u;
        *(uint2*)(as + (k >> 3) * 2048u + mb + r * 128u + ((mc ^ r) << 4) + me) = make_uint2(lo, hi);
      }
      fence_async_smem();
      mbar_arrive(afull + s);
      if (++s == kM2Stages) {
        s = 0;
        if (warm) ph ^= 1u;
        warm = true;
      }
    }
  } else {
    // ---------------- epilogue: warp e reads TMEM lanes 32 e .. +31 (images), 32 columns at a
    // time, and stores them with TMA (box 32 bins x 1 direction x 32 images)
    const int e = warp - kM2Build;
    uint8_t* es = Es + e * 2 * kM2EStage;
    int eb = 0;  // staging buffer
    int64_t npass = 0;
    for (Cur c = first(u_begin); c.unit < nunits;) {
      const int o = (int)(c.unit & 3);
      const int64_t img0 = (c.unit >> 2) * kMmaM + 32 * e;
      for (int pp = 0; pp < qn[o]; ++pp) {
        const int p = qf[o] + pp;
        const int a = (int)(npass & 1);
        mbar_wait(tfull + a, (unsigned)((npass >> 1) & 1));
        tc_fence_after();
        const int nd = tab[p * kMmaPassCols + 1];
        for (int n0 = 0; n0 < N; n0 += 32) {
          uint32_t r[32];
          WECT_TMEM_LD32(tmem + ((uint32_t)(32 * e) << 16) + (uint32_t)(256 * a + n0), r);
          const int j = n0 / Tq, q0 = n0 - j * Tq;
          const bool live = j < nd && q0 < T;
          float4 f[8];
          int dl = 0;
          if (live) {
            dl = tab[p * kMmaPassCols + 2 + j];
            const float4* cf = (const float4*)(cfix + (int64_t)p * N + n0);
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4) f[k4] = __ldg(cf + k4);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (!live) continue;
          // the staging buffer's previous TMA store has read it
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          uint8_t* sb = es + eb * kM2EStage;
          if (sizeof(OutT) == 4) {
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4) {
              int4 v;
              v.x = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 0]), f[k4].x)) - 0x4B400000;
              v.y = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 1]), f[k4].y)) - 0x4B400000;
              v.z = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 2]), f[k4].z)) - 0x4B400000;
              v.w = __float_as_int(__fadd_rn(__int_as_float(r[4 * k4 + 3]), f[k4].w)) - 0x4B400000;
              // row = lane (image), 16-byte chunk k4 swizzled by (lane & 7)
              *(int4*)(sb + lane * 128 + ((k4 ^ (lane & 7)) << 4)) = v;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(&omap),
                "r"(smem_u32(sb)), "r"(q0), "r"(dl), "r"((int)img0)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          eb ^= 1;
        }
        tc_fence_before();
        mbar_arrive(tempty + a);
        ++npass;
      }
      c = first(c.unit + 1);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kM2MmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool mma2d_supported(int ndim, const int64_t* dims, int T) {
  if (ndim != 2) return false;
  const int64_t H = dims[0], W = dims[1];
  if (H < 2 || W < 4 || (W & 3) != 0 || H * W > 4096) return false;
  return T >= 1 && T <= kMmaNmax && mma_smem_bytes((int)(H * W)) <= 227 * 1024;
}

size_t mma2d_scratch_bytes(int HW, int Dc, int T) {
  const int N = mma_n(T), KC = mma_kc(HW), dpp = mma_dpp(T);
  const int npass_max = (Dc + dpp - 1) / dpp + 4;
  return 256 + (size_t)Dc * HW * 2 + 16 + (size_t)Dc * T * 4 + 16 + (16 + 4 * Dc) * 4 + 16 +
         (size_t)npass_max * kMmaPassCols * 4 + 16 + (size_t)npass_max * KC * N * kMmaKC * 2 + 1024 +
         (size_t)npass_max * N * 4 + 16;
}

wect_status launch_mma2d(const uint8_t* img, int64_t B, int H, int W, const float* dirs, int d_begin, int Dc, int T,
                         const GridParams* gp, void* scratch, void* out, wect_dtype odtype, cudaStream_t st,
                         int num_sms) {
  const int HW = H * W, N = mma_n(T), KC = mma_kc(HW), dpp = mma_dpp(T), Tq = mma_tq(T);
  const int npass_max = (Dc + dpp - 1) / dpp + 4;
  auto al = [](uintptr_t x, uintptr_t a) { return (x + a - 1) & ~(a - 1); };
  uintptr_t cur = al((uintptr_t)scratch, 256);
  uint16_t* vbin = (uint16_t*)cur;
  cur = al(cur + (size_t)Dc * HW * 2, 16);
  int* cum = (int*)cur;
  cur = al(cur + (size_t)Dc * T * 4, 16);
  int* qcount = (int*)cur;  // [4]
  int* info = qcount + 4;   // [9]: #passes, first pass / #passes of each quadrant
  int* qlist = qcount + 16;  // [4][Dc]
  cur = al(cur + (size_t)(16 + 4 * Dc) * 4, 16);
  int* tab = (int*)cur;
  cur = al(cur + (size_t)npass_max * kMmaPassCols * 4, 1024);
  uint4* bimg = (uint4*)cur;
  cur = al(cur + (size_t)npass_max * KC * N * kMmaKC * 2, 16);
  float* cfix = (float*)cur;
  WECT_CUDA_TRY(cudaMemsetAsync(qcount, 0, 16 * sizeof(int), st));
  k_mma_dirs<<<Dc, 256, (size_t)T * 4, st>>>(H, W, dirs, d_begin, Dc, gp, vbin, cum, qcount, qlist);
  k_mma_passes<<<1, 32, 0, st>>>(qcount, qlist, Dc, dpp, tab, info);
  k_mma_bimg<<<npass_max * KC, 256, 0, st>>>(HW, T, Tq, N, KC, info, tab, vbin, cum, bimg, cfix);
  count_launch(3);
  WECT_CUDA_TRY(cudaGetLastError());
  const size_t smem = mma_smem_bytes(HW);
  const int64_t nunits = 4 * ((B + kMmaM - 1) / kMmaM);  // (tile, quadrant)
  const int grid = (int)(nunits < num_sms ? nunits : num_sms);
  MainTimer timer(st);
  if (odtype == WECT_I32) {
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_mma2d<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_mma2d<int32_t><<<grid, kMmaThreads, smem, st>>>(img, B, H, W, T, Tq, N, KC, Dc, info, tab, bimg, cfix,
                                                      (int32_t*)out);
  } else {
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_mma2d<long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_mma2d<long long><<<grid, kMmaThreads, smem, st>>>(img, B, H, W, T, Tq, N, KC, Dc, info, tab, bimg, cfix,
                                                        (long long*)out);
  }
  count_launch();
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

// ---- v2 host side
static PFN_cuTensorMapEncodeTiled_v12000 m2_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;  // calls may come from several host threads
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// v2 needs int32 output that a TMA map can describe, and the B chunks within the scratch cap
bool mma2_usable(void* out, int64_t B, int Dc, int T, wect_dtype odtype) {
  return odtype == WECT_I32 && ((uintptr_t)out & 15) == 0 && ((int64_t)T * 4) % 16 == 0 && B <= 0xFFFFFFFFll &&
         m2_encode() != nullptr;
}

size_t mma2_scratch_bytes(int HW, int Dc, int T, int64_t B) {
  const int N = mma_n(T), KC = m2_kc(HW), dpp = mma_dpp(T);
  const int npass_max = (Dc + dpp - 1) / dpp + 4;
  const int64_t ntiles = (B + kMmaM - 1) / kMmaM;
  return 256 + (size_t)Dc * HW * 2 + 16 + (size_t)Dc * T * 4 + 16 + (16 + 4 * Dc) * 4 + 16 +
         (size_t)npass_max * kMmaPassCols * 4 + 1024 + (size_t)npass_max * KC * N * kM2K * 2 + 16 +
         (size_t)npass_max * N * 4 + 256 + (size_t)ntiles * HW * 128 + 256 + (size_t)HW + 16;
}

wect_status launch_mma2(const uint8_t* img, int64_t B, int H, int W, const float* dirs, int d_begin, int Dc, int T,
                        const GridParams* gp, void* scratch, void* out, cudaStream_t st, int num_sms) {
  const int HW = H * W, N = mma_n(T), KC = m2_kc(HW), dpp = mma_dpp(T), Tq = mma_tq(T);
  const int npass_max = (Dc + dpp - 1) / dpp + 4;
  const int64_t ntiles = (B + kMmaM - 1) / kMmaM;
  auto al = [](uintptr_t x, uintptr_t a) { return (x + a - 1) & ~(a - 1); };
  uintptr_t cur = al((uintptr_t)scratch, 256);
  uint16_t* vbin = (uint16_t*)cur;
  cur = al(cur + (size_t)Dc * HW * 2, 16);
  int* cum = (int*)cur;
  cur = al(cur + (size_t)Dc * T * 4, 16);
  int* qcount = (int*)cur;
  int* info = qcount + 4;
  int* qlist = qcount + 16;
  cur = al(cur + (size_t)(16 + 4 * Dc) * 4, 16);
  int* tab = (int*)cur;
  cur = al(cur + (size_t)npass_max * kMmaPassCols * 4, 1024);
  uint4* bimg = (uint4*)cur;
  cur = al(cur + (size_t)npass_max * KC * N * kM2K * 2, 16);
  float* cfix = (float*)cur;
  cur = al(cur + (size_t)npass_max * N * 4, 256);
  uint8_t* pixT = (uint8_t*)cur;
  cur = al(cur + (size_t)ntiles * HW * 128, 256);
  uint8_t* vflags = (uint8_t*)cur;
  CUtensorMap omap;
  memset(&omap, 0, sizeof(omap));
  {
    const cuuint64_t dims[3] = {(cuuint64_t)T, (cuuint64_t)Dc, (cuuint64_t)B};
    const cuuint64_t strides[2] = {(cuuint64_t)T * 4, (cuuint64_t)Dc * T * 4};
    const cuuint32_t box[3] = {32u, 1u, 32u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = m2_encode()(&omap, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, out, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(WECT_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  WECT_CUDA_TRY(cudaMemsetAsync(qcount, 0, 16 * sizeof(int), st));
  k_mma_dirs<<<Dc, 256, (size_t)T * 4, st>>>(H, W, dirs, d_begin, Dc, gp, vbin, cum, qcount, qlist);
  k_mma_passes<<<1, 32, 0, st>>>(qcount, qlist, Dc, dpp, tab, info);
  k_mma2_bimg<<<npass_max * KC, 256, 0, st>>>(HW, T, Tq, N, KC, info, tab, vbin, cum, bimg, cfix);
  k_mma2_pixt<<<dim3((unsigned)ntiles, (unsigned)((HW + 127) / 128)), 256, 0, st>>>(img, B, HW, pixT);
  k_mma2_vflags<<<(HW + 255) / 256, 256, 0, st>>>(H, W, vflags);
  count_launch(5);
  WECT_CUDA_TRY(cudaGetLastError());
  const size_t smem = m2_smem_bytes();
  const int64_t nunits = 4 * ntiles;
  const int grid = (int)(nunits < num_sms ? nunits : num_sms);
  MainTimer timer(st);
  WECT_CUDA_TRY(cudaFuncSetAttribute(k_mma2<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_mma2<int32_t><<<grid, kM2Threads, smem, st>>>(pixT, vflags, B, H, W, T, Tq, N, KC, info, tab, bimg, cfix, omap);
  count_launch();
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

}  // namespace wect
