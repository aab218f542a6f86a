// k_stream.cu -- the HBM-bound end of the explicit-complex path: the ECF (ecf_complex,
// the ECF-X row) and the WECT at few directions (D <= 8, SURVEY 8(d) D-sweep).
// Alg. 1 with one cell per thread-iteration: gather the filter values of the
// cell's vertices (MODE 0: FVals[v, p]; MODE 1: <coords[v], s_p> by fp32 FMA), take the
// max (eq. msi: alpha is monotone, so the bin of the max height is the max of the vertex
// bins), bin it (reading A1: fp32 + guard, binary64 repair), and add the signed weight into
// a shared-memory histogram (line 9); k_finalize does the cumsum (line 11).
//
// B200 shape: a persistent CTA per SM.  A producer warp streams the index lists and
// weights of 1920-cell units HBM -> shared memory with cp.async.bulk into a 4-stage ring
// (mbarrier complete_tx), so HBM latency is covered by the ring instead of by thread
// occupancy; 15 consumer warps read their cells' ids from shared memory, release the
// stage at once, then gather (L2-resident filter values / coordinates), bin and count.
// Histogram [p][bin][R]: R lane replicas (R = 32 when it fits) so that lanes of a warp
// hitting the same bin -- the common case for spatially coherent heights -- never
// collide in a shared-memory bank.  Units are dealt round-robin over the CTAs, so the
// units in flight at any moment are adjacent in the cell lists (gathers stay in L2).
#include <cfloat>

#include "common.cuh"
#include "async.cuh"

namespace wect {

constexpr int kStreamConsumers = 15;  // consumer warps (+ the producer: 4 warps per SM sub-partition)
constexpr int kStreamThreads = 32 * (kStreamConsumers + 1);  // + 1 producer warp
constexpr int kStreamStages = 4;
constexpr int kStreamMaxAr = 5;
constexpr int kStreamUnit = 4 * 32 * kStreamConsumers;  // 1920 cells (arity <= 4; 960 for arity 5)
constexpr int kStreamIdxBytes = kStreamUnit * 4 * 4;
constexpr int kStreamWBytes = kStreamUnit * 4;
constexpr int kStreamTile = 8;                 // filters per CTA (grid.y tiles)
constexpr int kStreamHistBytes = 64 * 1024;

struct StreamUnits {
  int64_t ustart[kMaxSegs + 1];  // first unit of each segment (prefix sum)
};

__host__ __device__ constexpr int stream_unit_cells(int ar) { return ar <= 4 ? kStreamUnit : kStreamUnit / 2; }

// L2 policy for the streamed index lists and weights: read once, so evict first -- the
// gathered filter values / coordinates (re-read by every cell dimension) keep the L2.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}

// a pointer the compiler cannot re-associate with the 32-bit offsets added to it
__device__ __forceinline__ const float* opaque(const float* p) {
  const float* q;
  asm("mov.b64 %0, %1;" : "=l"(q) : "l"(p));
  return q;
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kStreamConsumers)); }

template <int AR>
struct CellIds {
  int v[AR];
};

template <int MODE, int N, bool FLOATW>
struct StreamCtx {
  using Acc = typename std::conditional<FLOATW, float, int>::type;
  const float* fv;      // MODE 0: fvals + p0
  const uint16_t* vb;   // one filter (np == 1): its exact vertex bins (k_vbin1), gathered per cell
  int m;                // MODE 0: row stride of fvals
  const float* coords;  // MODE 1
  const float* sdir;    // MODE 1: [np][N] in shared memory
  int np, T, rl, rmask, row0;
  float tau;  // near-edge guard; -1 with WECT_FP32_ONLY (never fires)
  bool direct;  // int weights too large for int32 partials: add straight into the int64 table
  uint32_t k0c;
  void* diff;
  GridParams g;
  const GridParams* gp;
  Acc* hist;
};

// int32 partials are flushed every kStreamFlushCells cells per CTA, which is exact while every
// weight added to them has |w| <= kStreamWBound; a warp whose unit holds a larger weight adds
// that unit straight into the int64 table instead (checked per unit in-kernel, so no pre-pass
// over the weights is needed).
constexpr unsigned kStreamWBound = 4095;
constexpr int64_t kStreamFlushCells = 524288;  // 524288 * 4095 < 2^31
template <typename Acc, int CPT>
__device__ __forceinline__ bool unit_needs_direct(const Acc (&w)[CPT]) {
  unsigned m = 0;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int x = (int)w[k];
    m = max(m, (unsigned)(x < 0 ? -x : x));  // |INT_MIN| wraps to 2^31 as unsigned: > bound
  }
  return __reduce_max_sync(0xffffffffu, m) > kStreamWBound;
}

__device__ __noinline__ void stream_add_direct(void* diff, int64_t o, int w) {
  atomicAdd((unsigned long long*)diff + o, (unsigned long long)(long long)w);
}

// KG cells (ids v[KG][AR], already validated; dead cells carry weight 0 and vertex 0):
// every gather of the group is issued before any binning, then one shared-memory atomic
// per (cell, filter).  Near-edge cells are repaired after the fast pass (rare calls).
template <int MODE, int N, bool FLOATW, int AR, int KG>
__device__ __forceinline__ void stream_group(const StreamCtx<MODE, N, FLOATW>& c, const int (*v)[AR],
                                             const typename StreamCtx<MODE, N, FLOATW>::Acc* w, int lane,
                                             bool udirect) {
  if constexpr (MODE == 0) {
    for (int pp = 0; pp < c.np; ++pp) {
      const float* fp = opaque(c.fv + pp);  // keeps each gather one IMAD.WIDE.U32 off the base
      float h[KG][AR];
#pragma unroll
      for (int k = 0; k < KG; ++k)
#pragma unroll
        for (int t = 0; t < AR; ++t) h[k][t] = __ldg(fp + (uint32_t)v[k][t] * (uint32_t)c.m);  // k0*m < 2^32
      float hm[KG], dist[KG], dmin = 2.f;
      int bin[KG];
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        hm[k] = h[k][0];
#pragma unroll
        for (int t = 1; t < AR; ++t) hm[k] = fmaxf(hm[k], h[k][t]);
        const float uu = fmaf(hm[k], c.g.A, c.g.B);
        bin[k] = max(0, min(__float2int_ru(uu), c.T - 1));
        dist[k] = fabsf(uu - rintf(uu));
        dmin = fminf(dmin, dist[k]);
      }
      // some cell of the group sits near a bin edge: warp-uniform repair, binary64 inlined
      // (a divergent repair call would leave the warp split)
      if (__builtin_expect(__any_sync(0xffffffffu, dmin < c.tau), 0)) {
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          const bool nk = dist[k] < c.tau;
          const unsigned bal = __ballot_sync(0xffffffffu, nk);
          if (bal) {
            const int r = alpha64((double)hm[k], c.g);  // filter values are exact in binary64
            if (nk) bin[k] = r;
            if (lane == 0) atomicAdd(&g_repair_count, (unsigned long long)__popc(bal));
          }
        }
      }
      if (!FLOATW && (c.direct || udirect)) {
#pragma unroll
        for (int k = 0; k < KG; ++k) stream_add_direct(c.diff, (int64_t)(c.row0 + pp) * c.T + bin[k], (int)w[k]);
      } else {
#pragma unroll
        for (int k = 0; k < KG; ++k) atomicAdd(c.hist + (((pp * c.T + bin[k]) << c.rl) | (lane & c.rmask)), w[k]);
      }
    }
  } else {
    float x[KG][AR * N];
    const float* cb = opaque(c.coords);
#pragma unroll
    for (int k = 0; k < KG; ++k)
#pragma unroll
      for (int t = 0; t < AR; ++t) {
        const float* xv = cb + (uint32_t)v[k][t] * (uint32_t)N;
#pragma unroll
        for (int i = 0; i < N; ++i) x[k][t * N + i] = __ldg(xv + i);
      }
    for (int pp = 0; pp < c.np; ++pp) {
      const float* s = c.sdir + pp * N;
      float sv[N];
#pragma unroll
      for (int i = 0; i < N; ++i) sv[i] = s[i];
      int bin[KG];
      float dist[KG], dmin = 2.f;
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        float hmax = -FLT_MAX;
#pragma unroll
        for (int t = 0; t < AR; ++t) {
          float h = x[k][t * N] * sv[0];
#pragma unroll
          for (int i = 1; i < N; ++i) h = fmaf(x[k][t * N + i], sv[i], h);
          hmax = fmaxf(hmax, h);
        }
        const float uu = fmaf(hmax, c.g.A, c.g.B);
        bin[k] = max(0, min(__float2int_ru(uu), c.T - 1));
        dist[k] = fabsf(uu - rintf(uu));
        dmin = fminf(dmin, dist[k]);
      }
      if (__builtin_expect(__any_sync(0xffffffffu, dmin < c.tau), 0)) {  // warp-uniform, inlined
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          const bool nk = dist[k] < c.tau;
          const unsigned bal = __ballot_sync(0xffffffffu, nk);
          if (bal) {
            double hm64 = -DBL_MAX;
#pragma unroll
            for (int t = 0; t < AR; ++t) {
              double h = __dmul_rn((double)x[k][t * N], (double)sv[0]);
#pragma unroll
              for (int i = 1; i < N; ++i) h = __dadd_rn(h, __dmul_rn((double)x[k][t * N + i], (double)sv[i]));
              hm64 = fmax(hm64, h);
            }
            const int r = alpha64(hm64, c.g);
            if (nk) bin[k] = r;
            if (lane == 0) atomicAdd(&g_repair_count, (unsigned long long)__popc(bal));
          }
        }
      }
      if (!FLOATW && (c.direct || udirect)) {
#pragma unroll
        for (int k = 0; k < KG; ++k) stream_add_direct(c.diff, (int64_t)(c.row0 + pp) * c.T + bin[k], (int)w[k]);
      } else {
#pragma unroll
        for (int k = 0; k < KG; ++k) atomicAdd(c.hist + (((pp * c.T + bin[k]) << c.rl) | (lane & c.rmask)), w[k]);
      }
    }
  }
}

// Consume one unit of `cells` cells (arity AR) of segment S starting at cell b0; its ids
// and weights are all in the stage (the producer stores a segment's last <= 3 ids /
// weights itself, which a 16-byte bulk copy cannot carry).  Releases the stage (one
// arrive per warp) as soon as the ids are in registers.
// FAST: a full unit of a segment with index lists and weights (the common case): no
// liveness or null-pointer tests, and invalid ids are handled out of line.
template <int MODE, int N, bool FLOATW, int AR, bool FAST>
__device__ __forceinline__ void stream_unit(const StreamCtx<MODE, N, FLOATW>& c, const Seg S, int64_t b0, int cells,
                                            const int* sid, const void* sw, uint64_t* empty, int ctid, int lane) {
  using Acc = typename StreamCtx<MODE, N, FLOATW>::Acc;
  constexpr int CPT = stream_unit_cells(AR) / (32 * kStreamConsumers);  // cells per thread: 4 or 2
  constexpr int KG = (CPT * AR * (MODE == 0 ? 1 : N) <= 40) ? CPT : ((CPT / 2) * AR * (MODE == 0 ? 1 : N) <= 40 ? CPT / 2 : 1);
  int v[CPT][AR];
  Acc w[CPT];
  unsigned bad = 0;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int cl = ctid + k * 32 * kStreamConsumers;  // strided: conflict-free shared loads
    if (FAST || S.verts) {
      const int* p = sid + cl * AR;
      if constexpr (AR == 4) {
        const int4 q = *(const int4*)p;
        v[k][0] = q.x; v[k][1] = q.y; v[k][2] = q.z; v[k][3] = q.w;
      } else if constexpr (AR == 2) {
        const int2 q = *(const int2*)p;
        v[k][0] = q.x; v[k][1] = q.y;
      } else {
#pragma unroll
        for (int t = 0; t < AR; ++t) v[k][t] = p[t];
      }
    } else {
#pragma unroll
      for (int t = 0; t < AR; ++t) v[k][t] = (int)(b0 + cl);
    }
    const Acc wk = (FAST || S.weights) ? ((const Acc*)sw)[cl] : (Acc)1;
    w[k] = S.sign < 0 ? -wk : wk;
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);  // stage free for the producer
  bool anybad = !FAST;
  if (FAST) {
    bool oob = false;
#pragma unroll
    for (int k = 0; k < CPT; ++k)
#pragma unroll
      for (int t = 0; t < AR; ++t) oob |= (uint32_t)v[k][t] >= c.k0c;
    anybad = oob;
  }
  if (anybad)
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int cl = ctid + k * 32 * kStreamConsumers;
    bool ok = cl < cells, oob = false;
#pragma unroll
    for (int t = 0; t < AR; ++t) oob |= (uint32_t)v[k][t] >= c.k0c;
    bad |= (ok && oob) ? 1u : 0u;
    ok = ok && !oob;
    if (!ok) {
      w[k] = (Acc)0;
#pragma unroll
      for (int t = 0; t < AR; ++t) v[k][t] = 0;
    }
  }
  if (bad) atomicOr(&g_err_word, 1u);
#pragma unroll
  const bool udirect = !FLOATW && unit_needs_direct<Acc, CPT>(w);
  for (int k0 = 0; k0 < CPT; k0 += KG) stream_group<MODE, N, FLOATW, AR, KG>(c, v + k0, w + k0, lane, udirect);
}

// ---- ECF with one filter per tile (MODE 0, np == 1): software-pipelined over units.
// ecf_read takes a unit's ids and weights out of its stage, releases the stage and
// issues the unit's gathers; ecf_finish bins and adds a unit whose gathers were issued
// one unit earlier, so the L2 latency of the gathers overlaps the previous unit's work.
template <bool FLOATW, int AR>
__device__ __forceinline__ void ecf_read(const StreamCtx<0, 1, FLOATW>& c, const Seg& S, int64_t b0, int cells,
                                         const int* sid, const void* sw, uint64_t* empty, int ctid, int lane,
                                         int (&h)[stream_unit_cells(AR) / (32 * kStreamConsumers)][AR],
                                         typename StreamCtx<0, 1, FLOATW>::Acc (&w)[stream_unit_cells(AR) / (32 * kStreamConsumers)]) {
  using Acc = typename StreamCtx<0, 1, FLOATW>::Acc;
  constexpr int CPT = stream_unit_cells(AR) / (32 * kStreamConsumers);
  int v[CPT][AR];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int cl = ctid + k * 32 * kStreamConsumers;
    if (S.verts) {
      const int* p = sid + cl * AR;
      if constexpr (AR == 4) {
        const int4 q = *(const int4*)p;
        v[k][0] = q.x; v[k][1] = q.y; v[k][2] = q.z; v[k][3] = q.w;
      } else if constexpr (AR == 2) {
        const int2 q = *(const int2*)p;
        v[k][0] = q.x; v[k][1] = q.y;
      } else {
#pragma unroll
        for (int t = 0; t < AR; ++t) v[k][t] = p[t];
      }
    } else {
#pragma unroll
      for (int t = 0; t < AR; ++t) v[k][t] = (int)(b0 + cl);
    }
    const Acc wk = S.weights ? ((const Acc*)sw)[cl] : (Acc)1;
    w[k] = S.sign < 0 ? -wk : wk;
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);
  bool bad = false;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int cl = ctid + k * 32 * kStreamConsumers;
    bool oob = false;
#pragma unroll
    for (int t = 0; t < AR; ++t) oob |= (uint32_t)v[k][t] >= c.k0c;
    bad |= cl < cells && oob;
    if (cl >= cells || oob) {
      w[k] = (Acc)0;
#pragma unroll
      for (int t = 0; t < AR; ++t) v[k][t] = 0;
    }
  }
  if (bad) atomicOr(&g_err_word, 1u);
  // the cell's vertex bins (exact, k_vbin1): the cell's bin is their max (eq. msi)
#pragma unroll
  for (int k = 0; k < CPT; ++k)
#pragma unroll
    for (int t = 0; t < AR; ++t) h[k][t] = (int)__ldg(c.vb + (uint32_t)v[k][t]);
}

template <bool FLOATW, int AR>
__device__ __forceinline__ void ecf_finish(const StreamCtx<0, 1, FLOATW>& c,
                                           const int (&h)[stream_unit_cells(AR) / (32 * kStreamConsumers)][AR],
                                           const typename StreamCtx<0, 1, FLOATW>::Acc (&w)[stream_unit_cells(AR) / (32 * kStreamConsumers)],
                                           int lane) {
  using Acc = typename StreamCtx<0, 1, FLOATW>::Acc;
  constexpr int CPT = stream_unit_cells(AR) / (32 * kStreamConsumers);
  int bin[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    bin[k] = h[k][0];
#pragma unroll
    for (int t = 1; t < AR; ++t) bin[k] = max(bin[k], h[k][t]);
  }
  if (!FLOATW && (c.direct || unit_needs_direct<Acc, CPT>(w))) {
#pragma unroll
    for (int k = 0; k < CPT; ++k) stream_add_direct(c.diff, (int64_t)c.row0 * c.T + bin[k], (int)w[k]);
  } else {
#pragma unroll
    for (int k = 0; k < CPT; ++k) atomicAdd(c.hist + ((bin[k] << c.rl) | (lane & c.rmask)), w[k]);
  }
}

template <bool FLOATW, typename Acc>
__device__ __forceinline__ void stream_flush(Acc* hist, int np, int T, int rl, int row0, int Dc, void* diff,
                                             int ctid) {
  const int R = 1 << rl;
  for (int i = ctid; i < np * T; i += 32 * kStreamConsumers) {
    Acc s = (Acc)0;
    for (int r = 0; r < R; ++r) {
      const int j = (i << rl) + ((r + i) & (R - 1));  // rotated: lanes hit distinct banks
      s += hist[j];
      hist[j] = (Acc)0;
    }
    const int p = i / T, q = i - p * T;
    if (s != (Acc)0 && row0 + p < Dc) {
      const int64_t o = (int64_t)(row0 + p) * T + q;
      if (FLOATW) atomicAdd((double*)diff + o, (double)s);
      else atomicAdd((unsigned long long*)diff + o, (unsigned long long)(long long)s);
    }
  }
}

template <int MODE, int N, bool FLOATW>
__global__ void __launch_bounds__(kStreamThreads, 1)
    k_stream(Segs segs, StreamUnits su, int64_t k0, const float* __restrict__ fvals, int m,
             const float* __restrict__ coords, const float* __restrict__ dirs, int d_begin, int Dc,
             const GridParams* __restrict__ gp, int rl, const unsigned int* __restrict__ wmax_bits,
             int64_t float_chunk, const char* __restrict__ pf, int64_t pf_bytes, const uint16_t* __restrict__ vbins,
             void* __restrict__ diff) {
  using Acc = typename std::conditional<FLOATW, float, int>::type;
  constexpr int NS = N > 0 ? N : 1;
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned char* sidx = smraw;                                        // [stages][kStreamIdxBytes]
  unsigned char* sw = smraw + kStreamStages * kStreamIdxBytes;        // [stages][kStreamWBytes]
  Acc* hist = (Acc*)(sw + kStreamStages * kStreamWBytes);            // [np][T][R]
  __shared__ __align__(8) uint64_t full[kStreamStages], empty[kStreamStages];
  __shared__ Seg ssegs[kMaxSegs];
  __shared__ int64_t sustart[kMaxSegs + 1];
  __shared__ float sdir[kStreamTile * NS];

  const GridParams g = *gp;
  const int T = g.T, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.y, p0 = d_begin + tile * kStreamTile;
  const int np = (Dc - tile * kStreamTile) < kStreamTile ? (Dc - tile * kStreamTile) : kStreamTile;
  const int R = 1 << rl;
  if (tid < kMaxSegs) ssegs[tid] = segs.s[tid];
  if (tid <= kMaxSegs) sustart[tid] = su.ustart[tid];
  if (MODE == 1)
    for (int i = tid; i < np * NS; i += blockDim.x) sdir[i] = dirs[(int64_t)p0 * NS + i];
  for (int i = tid; i < np * T * R; i += blockDim.x) hist[i] = (Acc)0;
  if (tid == 0) {
    for (int s = 0; s < kStreamStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kStreamConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t nunits = sustart[segs.nseg];
  const int64_t G = gridDim.x;
  const int64_t my_units = nunits > blockIdx.x ? (nunits - blockIdx.x + G - 1) / G : 0;
  // unit j of this CTA = global unit blockIdx.x + j*G; its segment and cell range
  // (units only grow along a CTA's sequence, so each caller keeps a segment cursor sg)
  auto locate = [&](int64_t u, int& sg, int64_t& b0, int& cells) {
    while (sg + 1 < segs.nseg && u >= sustart[sg + 1]) ++sg;
    const int uc = stream_unit_cells(ssegs[sg].arity);
    b0 = (u - sustart[sg]) * uc;
    const int64_t rem = ssegs[sg].count - b0;
    cells = rem < uc ? (int)rem : uc;
  };

  if (warp == kStreamConsumers) {  // ---- producer warp
    if (lane == 0) {
      // warm the L2 with this CTA's share of the gathered array (filter values or
      // coordinates), so that the first touches of the gathers do not wait on HBM
      if (pf_bytes > 0) {
        const int64_t share = ((pf_bytes + G - 1) / G + 15) & ~(int64_t)15;
        const int64_t a0 = (int64_t)blockIdx.x * share;
        const int64_t a1 = (a0 + share) < pf_bytes ? (a0 + share) : (pf_bytes & ~(int64_t)15);
        for (int64_t a = a0; a < a1; a += 32768)
          bulk_prefetch_l2(pf + a, (unsigned)((a1 - a) < 32768 ? (a1 - a) : 32768));
      }
      const uint64_t pol = l2_evict_first();
      int sg = 0;
      for (int64_t j = 0; j < my_units; ++j) {
        const int st = (int)(j % kStreamStages);
        if (j >= kStreamStages) mbar_wait(&empty[st], (unsigned)(((j / kStreamStages) - 1) & 1));
        int cells;
        int64_t b0;
        locate(blockIdx.x + j * G, sg, b0, cells);
        const Seg& S = ssegs[sg];
        const unsigned ib = S.verts ? (unsigned)(((int64_t)cells * S.arity * 4) & ~15ll) : 0u;
        const unsigned wb = S.weights ? (unsigned)(((int64_t)cells * 4) & ~15ll) : 0u;
        // a segment's last 1..3 ids / weights: plain stores, published by the arrive below
        const int ni = S.verts ? cells * S.arity : 0;
        for (int t = (int)(ib >> 2); t < ni; ++t)
          ((int*)(sidx + st * kStreamIdxBytes))[t] = __ldg(S.verts + b0 * S.arity + t);
        if (S.weights)
          for (int t = (int)(wb >> 2); t < cells; ++t)
            ((int*)(sw + st * kStreamWBytes))[t] = __ldg((const int*)S.weights + b0 + t);
        mbar_arrive_expect_tx(&full[st], ib + wb);
        if (ib) bulk_g2s(sidx + st * kStreamIdxBytes, S.verts + b0 * S.arity, ib, &full[st], pol);
        if (wb) bulk_g2s(sw + st * kStreamWBytes, (const char*)S.weights + b0 * 4, wb, &full[st], pol);
      }
    }
    return;
  }

  // ---- consumer warps
  StreamCtx<MODE, NS, FLOATW> c;
  c.fv = MODE == 0 ? fvals + p0 : nullptr;
  c.vb = vbins;
  c.m = m;
  c.coords = coords;
  c.sdir = sdir;
  c.np = np;
  c.T = T;
  c.rl = rl;
  c.rmask = R - 1;
  c.k0c = k0 > 0x80000000ll ? 0x80000000u : (uint32_t)k0;
  c.g = g;
  c.tau = g.fp32_only ? -1.f : g.tau;
  c.gp = gp;
  c.hist = hist;
  c.row0 = tile * kStreamTile;
  c.diff = diff;
  c.direct = false;
  // flush period (units): int32 partials below 2^31 (device max|w|); float every float_chunk cells
  int64_t every_cells;
  if (FLOATW) every_cells = float_chunk;
  else every_cells = kStreamFlushCells;  // + the per-unit weight check (unit_needs_direct)
  int64_t since = 0;
  int sg = 0;
  bool small_ar = true;  // the pipelined path keeps two units of gathers in registers: arity <= 3
  for (int i = 0; i < segs.nseg; ++i) small_ar &= ssegs[i].arity <= 3;
  {
    if (vbins != nullptr && np == 1 && small_ar) {  // one filter: gather exact vertex bins (k_vbin1)
      const StreamCtx<0, 1, FLOATW>& c1 = *reinterpret_cast<const StreamCtx<0, 1, FLOATW>*>(&c);
      int64_t j = 0;
      while (j < my_units) {
        int cells;
        int64_t b0;
        locate(blockIdx.x + j * G, sg, b0, cells);
        const Seg S = ssegs[sg];
        // this CTA's units of segment sg: j in [j, j1)
        const int64_t uend = sustart[sg + 1];
        const int64_t j1 = uend > blockIdx.x ? (uend - blockIdx.x + G - 1) / G : 0;
        const int uc = stream_unit_cells(S.arity);
        auto unit_cells = [&](int64_t jj) {
          const int64_t bb = (blockIdx.x + jj * G - sustart[sg]) * uc;
          return (S.count - bb) < uc ? (int)(S.count - bb) : uc;
        };
        auto flush_if = [&](int ncell) {  // uniform across consumer threads
          if (since + ncell > every_cells) {
            consumers_sync();
            stream_flush<FLOATW, Acc>(hist, np, T, rl, tile * kStreamTile, Dc, diff, tid);
            consumers_sync();
            since = 0;
          }
          since += ncell;
        };
        switch (S.arity) {
#define WECT_ECF_AR(A)                                                                                       \
  case A: {                                                                                                  \
    constexpr int CPT = stream_unit_cells(A) / (32 * kStreamConsumers);                                     \
    int h0[CPT][A], h1[CPT][A];                                                                              \
    Acc w0[CPT], w1[CPT];                                                                                    \
    auto rd = [&](int64_t jj, int(&h)[CPT][A], Acc(&w)[CPT]) {                                              \
      const int st = (int)(jj % kStreamStages);                                                              \
      const int64_t bb = (blockIdx.x + jj * G - sustart[sg]) * uc;                                          \
      mbar_wait(&full[st], (unsigned)((jj / kStreamStages) & 1));                                           \
      ecf_read<FLOATW, A>(c1, S, bb, unit_cells(jj), (const int*)(sidx + st * kStreamIdxBytes),           \
                          sw + st * kStreamWBytes, &empty[st], tid, lane, h, w);                              \
    };                                                                                                       \
    rd(j, h0, w0);                                                                                           \
    for (; j < j1; j += 2) {                                                                                 \
      if (j + 1 < j1) rd(j + 1, h1, w1);                                                                     \
      flush_if(unit_cells(j));                                                                               \
      ecf_finish<FLOATW, A>(c1, h0, w0, lane);                                                               \
      if (j + 1 >= j1) { j += 1; break; }                                                                    \
      if (j + 2 < j1) rd(j + 2, h0, w0);                                                                     \
      flush_if(unit_cells(j + 1));                                                                           \
      ecf_finish<FLOATW, A>(c1, h1, w1, lane);                                                               \
    }                                                                                                        \
    j = j1;                                                                                                  \
  } break;
          WECT_ECF_AR(1) WECT_ECF_AR(2) WECT_ECF_AR(3)
#undef WECT_ECF_AR
        }
      }
      consumers_sync();
      stream_flush<FLOATW, Acc>(hist, np, T, rl, tile * kStreamTile, Dc, diff, tid);
      return;
    }
  }
  for (int64_t j = 0; j < my_units; ++j) {
    const int st = (int)(j % kStreamStages);
    int cells;
    int64_t b0;
    locate(blockIdx.x + j * G, sg, b0, cells);
    const Seg S = ssegs[sg];
    if (since + cells > every_cells) {  // uniform across consumer threads
      consumers_sync();
      stream_flush<FLOATW, Acc>(hist, np, T, rl, tile * kStreamTile, Dc, diff, tid);
      consumers_sync();
      since = 0;
    }
    since += cells;
    mbar_wait(&full[st], (unsigned)((j / kStreamStages) & 1));
    const int* sid = (const int*)(sidx + st * kStreamIdxBytes);
    const void* swp = sw + st * kStreamWBytes;
    switch (S.arity) {
#define WECT_AR(A)                                                                                         \
  case A:                                                                                                  \
    if (cells == stream_unit_cells(A) && S.verts && S.weights)                                             \
      stream_unit<MODE, NS, FLOATW, A, true>(c, S, b0, cells, sid, swp, &empty[st], tid, lane);            \
    else                                                                                                   \
      stream_unit<MODE, NS, FLOATW, A, false>(c, S, b0, cells, sid, swp, &empty[st], tid, lane);           \
    break;
      WECT_AR(1) WECT_AR(2) WECT_AR(3) WECT_AR(4) WECT_AR(5)
#undef WECT_AR
    }
  }
  consumers_sync();
  stream_flush<FLOATW, Acc>(hist, np, T, rl, tile * kStreamTile, Dc, diff, tid);
}

// Exact vertex bins of ONE filter (Alg. 1 line 3, VIndices = alpha(FVals)): MODE 0 the
// given values fvals[v * m + p0], MODE 1 the height <coords[v], s_p0> in the same fp32
// evaluation order as k_stream (so the same guard tau applies); near-edge vertices are
// repaired in binary64 (reading A1).  A cell's bin is then the max of its vertices' bins
// (eq. msi: alpha is monotone), so the streaming pass gathers 2-byte bins instead
// of filter values and bins nothing per cell.
template <int MODE, int N>
__device__ __forceinline__ int vbin1_one(int64_t v, const float* __restrict__ fvals, int m, int p0,
                                         const float* __restrict__ coords, const float (&s)[N > 0 ? N : 1],
                                         const GridParams& g, float h) {
  constexpr int NS = N > 0 ? N : 1;
  int b = alpha32_or_repair(h, g);
  if (b < 0) {
    double hd = (double)h;  // MODE 0: filter values are exact in binary64
    if (MODE == 1) {
      const float* x = coords + v * NS;
      hd = __dmul_rn((double)x[0], (double)s[0]);
      for (int i = 1; i < NS; ++i) hd = __dadd_rn(hd, __dmul_rn((double)x[i], (double)s[i]));
    }
    note_repair();
    b = alpha64(hd, g);
  }
  return b;
}

template <int MODE, int N>
__global__ void __launch_bounds__(256) k_vbin1(int64_t k0, const float* __restrict__ fvals, int m, int p0,
                                               const float* __restrict__ coords, const float* __restrict__ dirs,
                                               const GridParams* __restrict__ gp, uint16_t* __restrict__ vb) {
  const GridParams g = *gp;
  constexpr int NS = N > 0 ? N : 1;
  float s[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) s[i] = MODE == 1 ? dirs[(int64_t)p0 * NS + i] : 0.f;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  // 4 consecutive vertices per thread step: one 16-byte load of filter values (MODE 0, one
  // column, aligned) and one 8-byte store of their bins
  const bool vec = MODE == 0 && m == 1 && p0 == 0 && ((uintptr_t)fvals & 15) == 0 && ((uintptr_t)vb & 7) == 0;
  const int64_t n4 = vec ? k0 / 4 : 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += nt) {
    const float4 f = __ldg((const float4*)fvals + t);
    const float hv[4] = {f.x, f.y, f.z, f.w};
    uint32_t b[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] = (uint32_t)vbin1_one<MODE, N>(4 * t + k, fvals, m, p0, coords, s, g, hv[k]);
    *(uint2*)(vb + 4 * t) = make_uint2(b[0] | (b[1] << 16), b[2] | (b[3] << 16));
  }
  for (int64_t v = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < k0; v += nt) {
    float h;
    if (MODE == 0) {
      h = __ldg(fvals + v * m + p0);
    } else {
      const float* x = coords + v * NS;
      h = __ldg(x) * s[0];
#pragma unroll
      for (int i = 1; i < NS; ++i) h = fmaf(__ldg(x + i), s[i], h);
    }
    vb[v] = (uint16_t)vbin1_one<MODE, N>(v, fvals, m, p0, coords, s, g, h);
  }
}

// Host side.  Returns WECT_ENOTSUP when the streaming kernel does not apply (an arity above
// kStreamMaxAr, a misaligned list, or a histogram that does not fit); the caller then
// uses k_cells.
template <int MODE, int N>
static wect_status launch_stream_t(bool floatw, const Segs& segs, const StreamUnits& su, int64_t k0,
                                   const float* fvals, int m, const float* coords, const float* dirs, int d_begin,
                                   int Dc, int T, int rl, const GridParams* gp, const unsigned int* wmax, void* diff,
                                   cudaStream_t st, int num_sms) {
  const int tiles = (Dc + kStreamTile - 1) / kStreamTile;
  const int np = Dc < kStreamTile ? Dc : kStreamTile;
  // the gathered array, prefetched into L2 when it fits comfortably
  const char* pf = MODE == 0 ? (const char*)fvals : (const char*)coords;
  int64_t pf_bytes = k0 * (int64_t)(MODE == 0 ? m : N) * 4;
  // (the caller's fvals start at p0 = d_begin: k_stream indexes fvals + p0 itself)
  if (pf_bytes > ((int64_t)64 << 20) || ((uintptr_t)pf & 15)) pf_bytes = 0;
  const size_t smem = (size_t)kStreamStages * (kStreamIdxBytes + kStreamWBytes) + ((size_t)np * T * 4 << rl);
  int per_tile = num_sms / tiles;
  per_tile = per_tile < 1 ? 1 : per_tile;
  // one filter, cells of arity <= 3: exact vertex bins first (k_vbin1), gathered per cell
  bool small_ar = true;
  for (int i = 0; i < segs.nseg; ++i) small_ar &= segs.s[i].arity <= 3;
  AsyncScratch mem(st);
  uint16_t* vb = nullptr;
  if (Dc == 1 && small_ar && T <= 65536 && !getenv("WECT_STREAM_NO_VBIN")) {
    WECT_CUDA_TRY(mem.alloc(&vb, (size_t)(k0 > 0 ? k0 : 1) * sizeof(uint16_t)));
    const int vblocks = (int)((k0 + 255) / 256 < num_sms * 8 ? (k0 + 255) / 256 : num_sms * 8);
    k_vbin1<MODE, N><<<vblocks > 0 ? vblocks : 1, 256, 0, st>>>(k0, fvals, m, d_begin, coords, dirs, gp, vb);
    count_launch();
    WECT_CUDA_TRY(cudaGetLastError());
    pf = (const char*)vb;  // the gathered array is now the bins
    pf_bytes = k0 * 2 <= ((int64_t)64 << 20) ? ((k0 * 2) & ~(int64_t)15) : 0;
  }
  const int64_t nunits = su.ustart[segs.nseg];
  if (per_tile > nunits) per_tile = (int)(nunits > 0 ? nunits : 1);
  dim3 grid((unsigned)per_tile, (unsigned)tiles);
  MainTimer timer(st);
  if (floatw) {
    auto k = k_stream<MODE, N, true>;
    WECT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, kStreamThreads, smem, st>>>(segs, su, k0, fvals, m, coords, dirs, d_begin, Dc, gp, rl, wmax, 8192,
                                          pf, pf_bytes, vb, diff);
  } else {
    auto k = k_stream<MODE, N, false>;
    WECT_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, kStreamThreads, smem, st>>>(segs, su, k0, fvals, m, coords, dirs, d_begin, Dc, gp, rl, wmax, 8192,
                                          pf, pf_bytes, vb, diff);
  }
  count_launch();
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

wect_status launch_stream(int mode, int n, bool floatw, const Segs& segs_in, int64_t k0, const float* fvals, int m,
                          const float* coords, const float* dirs, int d_begin, int Dc, int T, const GridParams* gp,
                          const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms) {
  if (getenv("WECT_DISABLE_STREAM")) return WECT_ENOTSUP;
  if ((uint64_t)k0 * (uint64_t)(mode == 1 ? m : n) >= ((uint64_t)1 << 32)) return WECT_ENOTSUP;  // 32-bit offsets
  // process the vertex segment last: by then the cells have pulled the filter values /
  // coordinates into L2, so its loads hit (the order does not change the sums)
  Segs segs = segs_in;
  for (int i = 0; i + 1 < segs.nseg; ++i)
    if (!segs.s[i].verts) {
      const Seg v = segs.s[i];
      for (int j = i; j + 1 < segs.nseg; ++j) segs.s[j] = segs.s[j + 1];
      segs.s[segs.nseg - 1] = v;
      break;
    }
  StreamUnits su;
  su.ustart[0] = 0;
  for (int i = 0; i < segs.nseg; ++i) {
    const Seg& S = segs.s[i];
    if (S.arity < 1 || S.arity > kStreamMaxAr) return WECT_ENOTSUP;
    if (S.verts && ((uintptr_t)S.verts & 15)) return WECT_ENOTSUP;
    if (S.weights && ((uintptr_t)S.weights & 15)) return WECT_ENOTSUP;
    const int uc = stream_unit_cells(S.arity);
    su.ustart[i + 1] = su.ustart[i] + (S.count + uc - 1) / uc;
  }
  for (int i = segs.nseg + 1; i <= kMaxSegs; ++i) su.ustart[i] = su.ustart[segs.nseg];
  // histogram replicas: the largest R <= 32 with np * T * R * 4 <= 64 KB
  const int np = Dc < kStreamTile ? Dc : kStreamTile;
  if ((size_t)np * T * 4 > (size_t)kStreamHistBytes) return WECT_ENOTSUP;
  int rl = 0;
  while (rl < 5 && ((size_t)np * T * 4 << (rl + 1)) <= (size_t)kStreamHistBytes) ++rl;
  if (mode == 1)
    return launch_stream_t<0, 0>(floatw, segs, su, k0, fvals, m, nullptr, nullptr, d_begin, Dc, T, rl, gp, wmax, diff,
                                 st, num_sms);
  switch (n) {
#define WECT_CASE(NN)                                                                                          \
  case NN:                                                                                                     \
    return launch_stream_t<1, NN>(floatw, segs, su, k0, nullptr, 0, coords, dirs, d_begin, Dc, T, rl, gp, wmax, \
                                  diff, st, num_sms);
    WECT_CASE(2) WECT_CASE(3) WECT_CASE(4) WECT_CASE(5)
#undef WECT_CASE
  }
  return WECT_ENOTSUP;  // other n: k_cells
}

}  // namespace wect
