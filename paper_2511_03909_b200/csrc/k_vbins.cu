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
#include <cstdlib>
#include <cstdint>

#include "common.cuh"

namespace wect {

constexpr int kVbTile = 64;  // directions per tile: two per lane

template <int N>
struct VecN {
  float v[N];
};

// grid: blocks over vertices; lanes = direction pairs of the tile (inactive pairs of the
// last tile compute a harmless bin of direction 0 that nobody reads); each warp stages 32
// vertices' coordinates (lane-parallel), then writes one 128-byte VB row per vertex.
template <int N>
__global__ void __launch_bounds__(256, 4) k_vbins(const float* __restrict__ coords, int64_t k0,
                                               const float* __restrict__ dirs, int p0, int np,
                                               const GridParams* __restrict__ gp, uint32_t* __restrict__ vb) {
  constexpr int XS = N <= 4 ? 4 : N;  // staged floats per vertex (N <= 4: one LDS.128 per vertex)
  __shared__ __align__(16) float xs[8][32 * XS];
  const GridParams g = *gp;
  const float tau = g.fp32_only ? -1.f : g.tau;  // fp32-only: the guard never fires
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  VecN<N> sa, sb;
  const int pa = 2 * lane, pb = 2 * lane + 1;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    sa.v[i] = pa < np ? dirs[(int64_t)(p0 + pa) * N + i] : 0.f;
    sb.v[i] = pb < np ? dirs[(int64_t)(p0 + pb) * N + i] : 0.f;
  }
  float* x = xs[warp];
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t base = ((int64_t)blockIdx.x * 8 + warp) * 32; base < k0; base += nwarps * 32) {
    const int nv = (k0 - base) < 32 ? (int)(k0 - base) : 32;
    for (int t = lane; t < nv * N; t += 32) {
      const int vv = t / N;
      x[vv * XS + (t - vv * N)] = __ldg(coords + base * N + t);
    }
    __syncwarp();
    uint32_t* row = vb + base * 32 + lane;
    // fp32 bins of vertex j (both directions) and whether either lies within tau of an edge
    auto bins32 = [&](int j, int& ba, int& bb) -> uint32_t {
      float xv[XS];
      if constexpr (XS == 4) {
        const float4 q = *(const float4*)(x + j * 4);
        xv[0] = q.x; xv[1] = q.y; xv[2] = q.z; xv[3] = q.w;
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) xv[i] = x[j * XS + i];
      }
      float ha = xv[0] * sa.v[0], hb = xv[0] * sb.v[0];
#pragma unroll
      for (int i = 1; i < N; ++i) {
        ha = fmaf(xv[i], sa.v[i], ha);
        hb = fmaf(xv[i], sb.v[i], hb);
      }
      const float ua = fmaf(ha, g.A, g.B), ub = fmaf(hb, g.A, g.B);
      ba = max(0, min(__float2int_ru(ua), g.T - 1));
      bb = max(0, min(__float2int_ru(ub), g.T - 1));
      return (fabsf(ua - rintf(ua)) < tau ? 1u : 0u) | (fabsf(ub - rintf(ub)) < tau ? 2u : 0u);
    };
    // Near-edge vertices are only flagged in the loop (bit j) and repaired after it, in a
    // warp-uniform loop with the binary64 path inlined.  A divergent repair call inside the
    // loop never reconverged: the warp ran the rest of the kernel as two halves, every row
    // computed twice (ncu r02_k_vbins_cfg4: 1.5-2x the warp instructions).
    uint32_t near = 0;
    auto body = [&](int j) {
      int ba, bb;
      if (bins32(j, ba, bb)) near |= 1u << j;
      row[j * 32] = (uint32_t)ba | ((uint32_t)bb << 16);
    };
    if (nv == 32) {  // fully unrolled: immediate shared / global offsets and flag bits
#pragma unroll
      for (int j = 0; j < 32; ++j) body(j);
    } else {
#pragma unroll 2
      for (int j = 0; j < nv; ++j) body(j);
    }
    while (__any_sync(0xffffffffu, near != 0)) {
      const bool act = near != 0;
      const int j = act ? __ffs(near) - 1 : 0;
      near &= near - 1;
      int ba, bb;
      const uint32_t f = act ? bins32(j, ba, bb) : 0u;
      double ha = __dmul_rn((double)x[j * XS], (double)sa.v[0]), hb = __dmul_rn((double)x[j * XS], (double)sb.v[0]);
#pragma unroll
      for (int i = 1; i < N; ++i) {
        ha = __dadd_rn(ha, __dmul_rn((double)x[j * XS + i], (double)sa.v[i]));
        hb = __dadd_rn(hb, __dmul_rn((double)x[j * XS + i], (double)sb.v[i]));
      }
      const int ra = alpha64(ha, g), rb = alpha64(hb, g);
      const unsigned ca = __ballot_sync(0xffffffffu, f & 1u), cb = __ballot_sync(0xffffffffu, f & 2u);
      if (lane == 0 && (ca | cb)) atomicAdd(&g_repair_count, (unsigned long long)(__popc(ca) + __popc(cb)));
      if (act) row[j * 32] = (uint32_t)(f & 1u ? ra : ba) | ((uint32_t)(f & 2u ? rb : bb) << 16);
    }
    __syncwarp();
  }
}

// red.shared for int / CAS-based atomicAdd for float (fp32 shared atomics are CAS loops on sm_100)
__device__ __forceinline__ void hist_add(int* h, int w) { atomicAdd(h, w); }
__device__ __forceinline__ void hist_add(float* h, float w) { atomicAdd(h, w); }

constexpr int kVbBatch = 32;  // cells per warp batch
#ifndef WECT_VB_WARPS
#define WECT_VB_WARPS 32
#endif
#ifndef WECT_VB_U
#define WECT_VB_U 4
#endif
constexpr int kVbWarps = WECT_VB_WARPS;  // warps per CTA (one CTA per SM: MLP for the row gathers)
constexpr int kVbU = WECT_VB_U;          // cells per group: all kVbU x arity row loads in flight

// nb cells of arity AR (0: runtime `arr`) from the warp's staged ids: four cells at a
// time, all 4*AR row loads issued before the packed max and the atomics.
// red.shared.add.s32 at a 32-bit shared address (int partials, native on sm_100)
__device__ __forceinline__ void red_shared(uint32_t addr, int w) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(w) : "memory");
}

// Record stride (ints) of a staged cell: its AR ids then its signed weight, padded to a
// power of two so that one LDS.64 / LDS.128 (two for 4 <= AR <= 7) broadcasts a cell.
__host__ __device__ constexpr int rec_stride(int ar) { return ar + 1 <= 2 ? 2 : (ar + 1 <= 4 ? 4 : 8); }

template <int RS>
__device__ __forceinline__ void load_rec(const int* r, int* out) {
  if constexpr (RS == 2) {
    const int2 q = *(const int2*)r;
    out[0] = q.x; out[1] = q.y;
  } else {
#pragma unroll
    for (int i = 0; i < RS; i += 4) {
      const int4 q = *(const int4*)(r + i);
      out[i] = q.x; out[i + 1] = q.y; out[i + 2] = q.z; out[i + 3] = q.w;
    }
  }
}

// One batch of nb <= kVbBatch cells of arity AR staged as records in `rec` (ids, then
// the signed weight; dead or invalid cells carry weight 0 and ids 0): four cells at a
// time, all their 4*AR row loads issued before the packed max and the adds.
// vbl = vb + lane (the lane's column of the VB rows); hsa = shared address of hist + lane
// (int path), hl the same as a pointer (float path).  DIRECT (integer weights too large
// for int32 partials over one step): add straight into the int64 difference rows
// drow[0..T) and drow[T..2T) of the lane's two directions (aa / ab: the direction exists).
template <int AR, bool FLOATW, bool DIRECT, typename Acc>
__device__ __forceinline__ void vb_batch(const int* rec, int nb, const uint32_t* __restrict__ vbl, uint32_t hsa,
                                         Acc* hl, unsigned long long* drow, int T, bool aa, bool ab) {
  constexpr int RS = rec_stride(AR);
  for (int j = 0; j < nb; j += kVbU) {
    int r[kVbU][RS];
#pragma unroll
    for (int u = 0; u < kVbU; ++u) load_rec<RS>(rec + (j + u) * RS, r[u]);  // records past nb are zero
    uint32_t x[kVbU][AR];
#pragma unroll
    for (int u = 0; u < kVbU; ++u)
#pragma unroll
      for (int t = 0; t < AR; ++t)
#ifdef WECT_VB_NOGATHER  // A/B experiment only: bins from the id, no VB row loads (wrong results)
        x[u][t] = ((uint32_t)r[u][t] & 0x1FFu) * 0x10001u;
#else
        x[u][t] = __ldg(vbl + (int64_t)r[u][t] * 32);
#endif
#pragma unroll
    for (int u = 0; u < kVbU; ++u) {
      uint32_t m2 = x[u][0];
#pragma unroll
      for (int t = 1; t < AR; ++t) m2 = __vmaxu2(m2, x[u][t]);
      const uint32_t lo = m2 & 0xFFFFu, hi = m2 >> 16;
      const int wi = r[u][AR];
      if constexpr (DIRECT) {
        if (wi != 0) {
          if (aa) atomicAdd(drow + lo, (unsigned long long)(long long)wi);
          if (ab) atomicAdd(drow + T + hi, (unsigned long long)(long long)wi);
        }
      } else if constexpr (FLOATW) {
        const float w = __int_as_float(wi);
        hist_add(hl + lo * 64, w);
        hist_add(hl + hi * 64 + 32, w);
      } else {
#ifdef WECT_VB_NOATOM  // A/B experiment only: every load and max, no atomics (bins never 0xFFFF)
        if (m2 == 0xFFFFFFFFu) {
#else
        {
#endif
          red_shared(hsa + lo * 256u, wi);
          red_shared(hsa + hi * 256u + 128u, wi);
        }
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

// Work order (L2 locality): the cells of every segment advance together in NSTEP steps;
// step i covers cells [bnd[s][i], bnd[s][i+1]) of segment s, cut into batches of
// kVbBatch cells spread over all warps of the grid (grid-stride).  The boundaries are
// either uniform fractions of each segment or, after k_bucket_* (below), the vertex
// windows of a bucketed copy of the lists, so the VB rows gathered concurrently stay in
// a narrow window of vertices and each row comes from HBM about once per tile.  int32
// partials are flushed before a step could overflow them (a bound on the cells one CTA
// takes per step, times the device max|w|); fp32 partials every <= 32768 cells.
template <bool FLOATW>
__global__ void __launch_bounds__(kVbWarps * 32, 1) k_cells_vb(Segs segs, int64_t k0, const uint32_t* __restrict__ vb, int row0,
                                                  int np, int Dc, const GridParams* __restrict__ gp, int nstep,
                                                  const int64_t* __restrict__ bnd, const int* __restrict__ bat,
                                                  const int64_t* __restrict__ bound,
                                                  const unsigned int* __restrict__ wmax_bits,
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
  const uint32_t hsa = (uint32_t)__cvta_generic_to_shared(hist + lane);
  const uint32_t* vbl = vb + lane;
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp, W = (int64_t)gridDim.x * nwarps;
  int64_t limit;  // cells one CTA may add between flushes
  if (!FLOATW) {
    const unsigned int wm = *wmax_bits;
    limit = wm ? (int64_t)2147483647 / wm : ((int64_t)1 << 62);
  } else {
    limit = 32768;
  }
  int64_t since = 0;
  const int nseg = segs.nseg;
  __syncthreads();
  // Per-warp cursor over (step, segment, batch): the next batch's ids and weights are
  // loaded into registers (pv, pw) while the current one is processed, so the HBM
  // latency of the streamed cell lists is off the critical path.
  struct Cur {
    int step, sg, u;
  };
  auto seek = [&](int step, int sg, int u) -> Cur {  // first batch at or after (step, sg, u)
    while (step < nstep) {
      while (sg < nseg) {
        if (u < __ldg(bat + sg * nstep + step)) return Cur{step, sg, u};
        ++sg;
        u = (int)gw;
      }
      ++step;
      sg = 0;
    }
    return Cur{nstep, 0, 0};
  };
  constexpr int PF = 7;  // lane = cell of the batch: its <= 7 ids are prefetched
  int pv[PF];
  Acc pw = (Acc)0;
  int pnb = 0;
  auto fetch = [&](const Cur& c) {
    const Seg& S = ssegs[c.sg];
    const int ar = S.arity;
    const int64_t c0 = __ldg(bnd + c.sg * (int64_t)(nstep + 1) + c.step);
    const int64_t c1 = __ldg(bnd + c.sg * (int64_t)(nstep + 1) + c.step + 1);
    const int64_t b0 = c0 + (int64_t)c.u * kVbBatch;
    pnb = (c1 - b0) < kVbBatch ? (int)(c1 - b0) : kVbBatch;
    const bool live = lane < pnb;
    const int64_t b = b0 + lane;
#pragma unroll
    for (int t = 0; t < PF; ++t) pv[t] = (live && t < ar) ? (S.verts ? __ldg(S.verts + b * ar + t) : (int)b) : 0;
    pw = live ? cell_weight<FLOATW, Acc>(S, b) : (Acc)0;
  };
  Cur nxt = seek(0, 0, (int)gw);
  if (nxt.step < nstep) fetch(nxt);
  for (int step = 0; step < nstep; ++step) {
    const int64_t cta_cells = __ldg(bound + step);  // k_step_info: cells one CTA may take this step
    // a step alone could overflow the int32 partials: add straight into int64 instead
    unsigned long long* drow =
        (!FLOATW && cta_cells > limit) ? (unsigned long long*)diff + (int64_t)(row0 + 2 * lane) * T : nullptr;
    const bool aa = 2 * lane < np, ab = 2 * lane + 1 < np;
    if (since > 0 && since + cta_cells > limit) {
      __syncthreads();
      flush_tile<FLOATW, Acc>(hist, T, row0, np, diff);
      __syncthreads();
      since = 0;
    }
    since += cta_cells;
    while (nxt.step == step) {
      const Cur cur = nxt;
      const int ar = ssegs[cur.sg].arity;
      const int nb = pnb;
      const int rs = rec_stride(ar);
      // stage this lane's cell as a record: ids (validated) and signed weight
      bool bad = false;
#pragma unroll
      for (int t = 0; t < PF; ++t) bad |= t < ar && (uint64_t)(int64_t)pv[t] >= (uint64_t)k0;
      {
        int* r = ids + lane * rs;
        const int wbits = FLOATW ? __float_as_int((float)pw) : (int)pw;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (t < rs) r[t] = bad ? 0 : (t < ar ? pv[t] : (t == ar ? wbits : 0));
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&g_err_word, 1u);
      // issue the next batch's loads now; they land while this batch is processed
      nxt = seek(cur.step, cur.sg, cur.u + (int)W);
      if (nxt.step < nstep) fetch(nxt);
      __syncwarp();
      if (!FLOATW && drow) {
        switch (ar) {
          case 1: vb_batch<1, FLOATW, true>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 2: vb_batch<2, FLOATW, true>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 3: vb_batch<3, FLOATW, true>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 4: vb_batch<4, FLOATW, true>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 5: vb_batch<5, FLOATW, true>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 6: vb_batch<6, FLOATW, true>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          default: vb_batch<7, FLOATW, true>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
        }
      } else {
        switch (ar) {
          case 1: vb_batch<1, FLOATW, false>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 2: vb_batch<2, FLOATW, false>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 3: vb_batch<3, FLOATW, false>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 4: vb_batch<4, FLOATW, false>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 5: vb_batch<5, FLOATW, false>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          case 6: vb_batch<6, FLOATW, false>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
          default: vb_batch<7, FLOATW, false>(ids, nb, vbl, hsa, hl, drow, T, aa, ab); break;
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  flush_tile<FLOATW, Acc>(hist, T, row0, np, diff);
}

// ---- vertex-window bucketing of the cell lists (once per call, reused by every tile)
// key(cell) = (min vertex id) >> ws; ids outside [0, k0) get key 0 (k_cells_vb still
// reports them).  Counting sort per segment: k_bucket_count, k_bucket_scan, and
// k_bucket_scatter (CTA-aggregated reservations; order inside a bucket is not kept).
constexpr int kBucketMax = 4096;  // static smem: 4096 counters + 4096 bases = 48 KB
constexpr int kScatterChunk = 4096;

__device__ __forceinline__ int cell_key(const int32_t* verts, int64_t b, int ar, int64_t k0, int ws) {
  uint32_t mn = 0xFFFFFFFFu;
  for (int t = 0; t < ar; ++t) {
    const uint32_t v = (uint32_t)__ldg(verts + b * ar + t);
    mn = v < mn ? v : mn;
  }
  return (int64_t)mn < k0 ? (int)(mn >> ws) : 0;
}

__global__ void __launch_bounds__(512) k_bucket_count(const int32_t* __restrict__ verts, int64_t count, int ar,
                                                      int64_t k0, int ws, int nb, int* __restrict__ cnt) {
  __shared__ int h[kBucketMax];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < count; b += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[cell_key(verts, b, ar, k0, ws)], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (h[i]) atomicAdd(&cnt[i], h[i]);
}

// one CTA per segment row: bnd[i] = sum of cnt[< i] (i = 0..nb), cur = bnd[0..nb)
__global__ void __launch_bounds__(1024) k_bucket_scan(const int* __restrict__ cnt, int nb, int64_t* __restrict__ bnd,
                                                      int64_t* __restrict__ cur) {
  __shared__ int64_t part[1024];
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per, i1 = min(nb, i0 + per);
  int64_t s = 0;
  for (int i = i0; i < i1; ++i) s += cnt[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t x = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += x;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int i = i0; i < i1; ++i) {
    bnd[i] = run;
    cur[i] = run;
    run += cnt[i];
  }
  if (threadIdx.x == blockDim.x - 1) bnd[nb] = part[blockDim.x - 1];
}

__global__ void __launch_bounds__(512) k_bucket_scatter(const int32_t* __restrict__ verts,
                                                        const void* __restrict__ weights, int64_t count, int ar,
                                                        int64_t k0, int ws, int nb, unsigned long long* __restrict__ cur,
                                                        int32_t* __restrict__ overts, int32_t* __restrict__ oweights) {
  __shared__ int h[kBucketMax];
  __shared__ unsigned long long base[kBucketMax];
  constexpr int PER = kScatterChunk / 512;
  for (int64_t c0 = (int64_t)blockIdx.x * kScatterChunk; c0 < count; c0 += (int64_t)gridDim.x * kScatterChunk) {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
    __syncthreads();
    int key[PER], rank[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int64_t b = c0 + k * 512 + threadIdx.x;
      key[k] = b < count ? cell_key(verts, b, ar, k0, ws) : -1;
      rank[k] = key[k] >= 0 ? atomicAdd(&h[key[k]], 1) : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if (h[i]) base[i] = atomicAdd(&cur[i], (unsigned long long)h[i]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (key[k] < 0) continue;
      const int64_t b = c0 + k * 512 + threadIdx.x;
      const int64_t pos = (int64_t)base[key[k]] + rank[k];
      for (int t = 0; t < ar; ++t) overts[pos * ar + t] = __ldg(verts + b * ar + t);
      if (weights) oweights[pos] = __ldg((const int32_t*)weights + b);
    }
    __syncthreads();
  }
}

// per step: batches of each segment (bat[s][i]) and a bound on the cells one CTA of
// `nwarps` warps takes (grid-stride over W warps): sum_s nwarps * ceil(bat / W) * bs
__global__ void k_step_info(Segs segs, int nstep, const int64_t* __restrict__ bnd, int W, int nwarps,
                            int* __restrict__ bat, int64_t* __restrict__ bound) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nstep; i += gridDim.x * blockDim.x) {
    int64_t cells = 0;
    for (int s = 0; s < segs.nseg; ++s) {
      const int ar = segs.s[s].arity;
      const int bs = (kVbBatch * 8) / ar > kVbBatch ? kVbBatch : (kVbBatch * 8) / ar;
      const int64_t c = bnd[(int64_t)s * (nstep + 1) + i + 1] - bnd[(int64_t)s * (nstep + 1) + i];
      const int64_t u = (c + bs - 1) / bs;
      bat[s * nstep + i] = (int)u;
      cells += (int64_t)nwarps * ((u + W - 1) / W) * bs;
    }
    bound[i] = cells;
  }
}

// uniform step boundaries: bnd[s][i] = count_s * i / nstep
__global__ void k_uniform_bnd(Segs segs, int nstep, int64_t* __restrict__ bnd) {
  const int s = blockIdx.x;
  for (int i = threadIdx.x; i <= nstep; i += blockDim.x)
    bnd[(int64_t)s * (nstep + 1) + i] = (int64_t)((__int128)segs.s[s].count * i / nstep);
}

// vertex segment under bucketing: bnd[i] = min(i << ws, count)
__global__ void k_vertex_bnd(int64_t count, int ws, int nstep, int64_t* __restrict__ bnd) {
  for (int i = threadIdx.x; i <= nstep; i += blockDim.x) {
    const int64_t c = (int64_t)i << ws;
    bnd[i] = i == nstep ? count : (c < count ? c : count);
  }
}

template <int N>
static wect_status launch_vb_n(bool floatw, const Segs& segs_in, const float* coords, int64_t k0, const float* dirs,
                               int d_begin, int Dc, int T, const GridParams* gp, const unsigned int* wmax, void* diff,
                               cudaStream_t st, int num_sms) {
  Segs segs = segs_in;
  for (int i = 0; i < segs.nseg; ++i)
    if (segs.s[i].arity > 7) return WECT_ENOTSUP;  // records hold <= 7 ids: k_complex takes it
  AsyncScratch mem(st);  // freed on every return path
  uint32_t* vb = nullptr;
  WECT_CUDA_TRY(mem.alloc(&vb, (size_t)(k0 > 0 ? k0 : 1) * 32 * sizeof(uint32_t)));
  const size_t smem = (size_t)T * 64 * 4 + (size_t)kVbWarps * kVbBatch * 8 * sizeof(int);
  const int ctas = num_sms;  // one 1024-thread CTA per SM
  const int ntiles = (Dc + kVbTile - 1) / kVbTile;
  // Bucket when the VB table does not fit in L2 and there is more than one tile to reuse it
  const bool bucket = ntiles > 1 && (size_t)k0 * 128 > ((size_t)64 << 20) && !getenv("WECT_DISABLE_BUCKETS");
  int nstep;
  int ws = 0;
  if (bucket) {
    // ~8-12 windows per call: per-step overhead falls with fewer steps faster than the
    // wider window costs in L2 misses (measured on cfg4, 10M vertices: 2^16-vertex windows
    // 3.33 ms per tile, 2^18 3.20, 2^20 2.68, 2^22 2.85, one window 3.02; cfg5: 2^16 4.46,
    // 2^18 4.06, 2^20 4.01)
    ws = 16;
    while ((k0 >> ws) > 12) ++ws;
    if (const char* e = getenv("WECT_VB_WS")) ws = atoi(e);  // A/B experiments
    nstep = (int)((k0 - 1) >> ws) + 1;
  } else {
    // every warp gets ~4 batches of EVERY segment per step (balanced, narrow window)
    int64_t minU = INT64_MAX;
    for (int i = 0; i < segs.nseg; ++i) {
      if (segs.s[i].count == 0) continue;
      const int bs = (kVbBatch * 8) / segs.s[i].arity > kVbBatch ? kVbBatch : (kVbBatch * 8) / segs.s[i].arity;
      const int64_t U = (segs.s[i].count + bs - 1) / bs;
      minU = U < minU ? U : minU;
    }
    const int64_t per_step = (int64_t)ctas * kVbWarps * 4;
    nstep = minU == INT64_MAX ? 1 : (int)(minU / per_step);
    nstep = nstep < 1 ? 1 : nstep;
  }
  int64_t* bnd = nullptr;
  void* scratch = nullptr;
  WECT_CUDA_TRY(mem.alloc(&bnd, sizeof(int64_t) * kMaxSegs * (nstep + 1)));
  if (!bucket) {
    k_uniform_bnd<<<segs.nseg, 256, 0, st>>>(segs, nstep, bnd);
    count_launch();
  } else {
    // bucketed copies of every index list (and its weights) in one scratch block
    size_t bytes = 0;
    for (int i = 0; i < segs.nseg; ++i)
      if (segs.s[i].verts) bytes += (size_t)segs.s[i].count * (segs.s[i].arity + 1) * 4 + 256;
    size_t cbytes = sizeof(int) * kBucketMax + 2 * sizeof(int64_t) * (kBucketMax + 1);
    WECT_CUDA_TRY(mem.alloc(&scratch, bytes + cbytes));
    int* cnt = (int*)scratch;
    int64_t* cur = (int64_t*)((char*)scratch + sizeof(int) * kBucketMax);
    char* dst = (char*)scratch + cbytes;
    for (int i = 0; i < segs.nseg; ++i) {
      Seg& S = segs.s[i];
      int64_t* b = bnd + (int64_t)i * (nstep + 1);
      if (!S.verts) {
        k_vertex_bnd<<<1, 256, 0, st>>>(S.count, ws, nstep, b);
        count_launch();
        continue;
      }
      int32_t* ov = (int32_t*)dst;
      dst += ((size_t)S.count * S.arity * 4 + 127) & ~(size_t)127;
      int32_t* ow = S.weights ? (int32_t*)dst : nullptr;
      if (S.weights) dst += ((size_t)S.count * 4 + 127) & ~(size_t)127;
      WECT_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * kBucketMax, st));
      const int g1 = (int)((S.count + 511) / 512 < num_sms * 4 ? (S.count + 511) / 512 : num_sms * 4);
      k_bucket_count<<<g1 > 0 ? g1 : 1, 512, 0, st>>>(S.verts, S.count, S.arity, k0, ws, nstep, cnt);
      k_bucket_scan<<<1, 1024, 0, st>>>(cnt, nstep, b, cur);
      const int g2 = (int)((S.count + kScatterChunk - 1) / kScatterChunk < num_sms * 4
                               ? (S.count + kScatterChunk - 1) / kScatterChunk
                               : num_sms * 4);
      k_bucket_scatter<<<g2 > 0 ? g2 : 1, 512, 0, st>>>(S.verts, S.weights, S.count, S.arity, k0, ws, nstep,
                                                       (unsigned long long*)cur, ov, ow);
      count_launch(3);
      S.verts = ov;
      S.weights = ow;
    }
  }
  int* bat = nullptr;
  int64_t* bound = nullptr;
  WECT_CUDA_TRY(mem.alloc(&bat, sizeof(int) * kMaxSegs * nstep));
  WECT_CUDA_TRY(mem.alloc(&bound, sizeof(int64_t) * nstep));
  k_step_info<<<(nstep + 255) / 256, 256, 0, st>>>(segs, nstep, bnd, ctas * kVbWarps, kVbWarps, bat, bound);
  count_launch();
  int vblocks = (int)((k0 + 255) / 256);
  vblocks = vblocks > num_sms * 8 ? num_sms * 8 : (vblocks < 1 ? 1 : vblocks);
  wect_status s = WECT_OK;
  for (int t0 = 0; t0 < Dc && s == WECT_OK; t0 += kVbTile) {
    const int np = (Dc - t0) < kVbTile ? (Dc - t0) : kVbTile;
    k_vbins<N><<<vblocks, 256, 0, st>>>(coords, k0, dirs, d_begin + t0, np, gp, vb);
    count_launch();
    MainTimer timer(st);
    if (floatw) {
      WECT_CUDA_TRY(cudaFuncSetAttribute(k_cells_vb<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_cells_vb<true><<<ctas, kVbWarps * 32, smem, st>>>(segs, k0, vb, t0, np, Dc, gp, nstep, bnd, bat, bound, wmax, diff);
    } else {
      WECT_CUDA_TRY(cudaFuncSetAttribute(k_cells_vb<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_cells_vb<false><<<ctas, kVbWarps * 32, smem, st>>>(segs, k0, vb, t0, np, Dc, gp, nstep, bnd, bat, bound, wmax, diff);
    }
    count_launch();
    timer.stop();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) s = fail_cuda(e, "k_cells_vb", __FILE__, __LINE__);
  }
  return s;
}

// smem fits, and (integer weights) a CTA's int32 partials cannot overflow: every CTA sees at
// most total/num_sms + one step's worth of cells, checked against the host bound on max|w|
// (255 for the configs; callers with larger weights fall back to k_complex's chunked flush)
bool vb_supported(int T) { return (size_t)T * 64 * 4 + (size_t)kVbWarps * kVbBatch * 8 * sizeof(int) <= 220 * 1024; }

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

// one tile of the vertex-bin table (also used by the backward pass, k_grad.cu)
wect_status launch_vbins_tile(int n, const float* coords, int64_t k0, const float* dirs, int p0, int np,
                              const GridParams* gp, uint32_t* vb, cudaStream_t st, int num_sms) {
  int vblocks = (int)((k0 + 255) / 256);
  vblocks = vblocks > num_sms * 8 ? num_sms * 8 : (vblocks < 1 ? 1 : vblocks);
  switch (n) {
#define WECT_CASE(NN) \
  case NN: k_vbins<NN><<<vblocks, 256, 0, st>>>(coords, k0, dirs, p0, np, gp, vb); break;
    WECT_CASE(1) WECT_CASE(2) WECT_CASE(3) WECT_CASE(4) WECT_CASE(5) WECT_CASE(6) WECT_CASE(7) WECT_CASE(8)
#undef WECT_CASE
    default: return fail(WECT_EINVAL, "ambient dimension n=%d outside [1,8]", n);
  }
  count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

}  // namespace wect
