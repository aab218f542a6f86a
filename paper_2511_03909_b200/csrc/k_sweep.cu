// k_sweep.cu -- the image-batch WECT (wect_images on 2-D images of <= kSweepMaxHW pixels:
// BASELINE configs[0] and configs[1]), cubical and Freudenthal.
//
// Geometry is image-independent, so per call k_sort2d reduces it, per direction, to a
// RECORD PROGRAM: the vertices sorted by their exact binary64 bin (alpha, eq.
// left-adjoint P:637-645, reading A1), grouped per bin into 16-byte records of up to 7
// vertex rows.  Exact regrouping: for a direction s a
// cubical cell's height is that of one designated corner (upper index on every axis with
// s_k > 0), so all cells designating vertex v sum into one combined weight cw_o(v)
// (o = quadrant of s, |cw| <= 255) and land in bin(v).
//
// k_sweep2d: a persistent CTA (32 warps, one CTA per SM) takes 64 images at a time, stages
// their pixels transposed, builds the quadrant's cw table in shared memory -- one 128-byte
// row per vertex, word j = images (j, j+32) as a signed packed pair cw_j + cw_{j+32} 2^16 --
// and two warps sweep each direction (one the bins below its split upwards, one the bins
// above it downwards, emitting chi - rows above): for every bin, its records' rows are
// gathered (one LDS per row: every lane reads its own word of the same row) and summed, the
// sum is unpacked onto two int32 running totals (images lane, lane+32).  The running total
// after bin q IS the cumulative sum of the difference histogram (Alg. 1 lines 4-11,
// P:654-687): no atomics, no separate scan, exact int32.  Bins are unrolled by output chunk
// (8 int32 / 4 int64 bins = 32 bytes per image), so every bin's total lands in a register; a
// chunk goes to a per-warp 64-image x 32-byte shared stage (32B-swizzled: conflict-free
// STS.128) and out to HBM with one TMA tensor store (cp.async.bulk.tensor), which takes
// the strided [B, D, T] writes off the load/store pipe.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "async.cuh"

namespace wect {

constexpr int kRecRows = 14;     // vertex rows per 32-byte record (u16 header + 14 u16 rows + 1 spare)
constexpr int kSweepWarps = 32;   // two per direction: the bins below / above its split
constexpr int kSweepImgs = 64;   // images per CTA group: lane l owns images l, l + 32
constexpr int kPixStride = 68;   // bytes per staged pixel row (17 words: conflict-free transpose)
constexpr int kStageRow = 32;    // bytes per image row of an output chunk (8 int32 / 4 int64 bins)
constexpr int kStageBytes = kSweepImgs * kStageRow;  // per warp
constexpr int kRingRecs = 32;    // per-warp record ring: two halves of 16 records (32 B each)
constexpr int kRingBytes = kRingRecs * 32;  // 1 KB: halves at byte 0 and 512 (ro >> 9)
constexpr int kSweepMaxHW = 1024;

__host__ __device__ constexpr size_t align_up(size_t x, size_t a) { return (x + a - 1) & ~(a - 1); }
// bins per output chunk for an output element of osz bytes (32-byte image rows)
__host__ __device__ constexpr int chunk_bins(int osz) { return kStageRow / osz; }
// 32-byte records per direction: one per bin at least, + one per 15 vertices, + the prefetch pad
__host__ __device__ constexpr int sweep_rec_stride(int HW, int Tp) { return Tp + (HW + kRecRows - 1) / kRecRows + 8; }
// smem of k_sweep2d: cw table [HW][128 B] (1024-aligned) | output stages [32][2 KB] |
// record rings [32][1 KB] | ring mbarriers [32][2] | image totals [32 words][2] | pixel
// mbarrier.  The staged pixels [HW][68 B] overlay the stages: they are only read by the cw
// build, before any sweep of the phase uses its stage (the rings stay free, so every warp
// starts loading its program while the CTA stages pixels and builds cw).  The first phase
// of an image group transposes the pixels from the images and parks the staged block in
// global scratch (one bulk store, L2-resident); later phases reload it with one bulk copy.
// (row HW is all zeros: the pad row of odd-sized records)
__host__ __device__ constexpr size_t sweep_cw_bytes(int HW) { return align_up((size_t)(HW + 1) * 128, 1024); }
__host__ __device__ constexpr size_t sweep_fixed_bytes() {
  return (size_t)kSweepWarps * (kStageBytes + kRingBytes + 16) + 256 + 16;
}
__host__ __device__ constexpr size_t sweep_smem_bytes(int HW) {
  return 1024 + sweep_cw_bytes(HW) + sweep_fixed_bytes();
}
__host__ __device__ constexpr size_t sweep_pix_bytes(int HW) { return align_up((size_t)HW * kPixStride, 16); }
__host__ __device__ constexpr bool sweep_pix_fits(int HW) {
  return (size_t)HW * kPixStride <= (size_t)kSweepWarps * kStageBytes;
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

// Binary-block record layout: a record's n rows (n even: an odd record is padded with the
// all-zero row HW) occupy, for each set bit of n from the top, a block of 8 / 4 / 2 slots at
// slots 0-7 / 8-11 / 12-13, so the sweep sums them as up to three straight-line blocks of
// independent gathers (no per-row test).
__host__ __device__ __forceinline__ int rec_slot(int n, int p) {
  int base = 0;
#pragma unroll
  for (int blk = 8; blk >= 2; blk >>= 1) {
    if (n & blk) {
      if (p < blk) return base + p;
      p -= blk;
    }
    base += blk;
  }
  return 14;
}

// ---------------------------------------------------------------------------
// Per local direction (one CTA each): exact bins of all H*W vertices (binary64,
// alpha64), counting sort by bin, and the direction's record program over Tp >= T bins:
//   for bin q = 0 .. Tp-1, max(1, ceil(count_q / 15)) records of 32 bytes:
//   u16 header (bits 0-3: rows n <= 15 in this record, bit 4: another record of the same
//   bin follows), u16 slot[15] (vertex ids, any order within a bin, placed by rec_slot).
// Bins q >= T are empty (the TMA store clips them).  Also records the direction's
// quadrant / chamber in qlist, and (Freudenthal) the correction list.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sort2d(int H, int W, const float* __restrict__ dirs, int d_begin, int Dc,
                                                const GridParams* __restrict__ gp, uint4* __restrict__ recs,
                                                int rec_stride, int Tp, int* __restrict__ qlist,
                                                int* __restrict__ qcount, int4* __restrict__ split, int freud,
                                                int4* __restrict__ corr, int* __restrict__ ncorr, int corr_cap) {
  // smem: counts[Tp], rbase[Tp], totals[Tp], vbin[HW] (u16)
  extern __shared__ int sh[];
  const GridParams g = *gp;
  const int HW = H * W, dl = blockIdx.x, p = d_begin + dl;
  int* counts = sh;
  int* rbase = sh + Tp;
  int* totals = sh + 2 * Tp;
  uint16_t* vbin = (uint16_t*)(sh + 3 * Tp);
  __shared__ int sh_split, sh_nl;
  // rows in record j of a bin of c rows
  auto counts_total_rows = [&](int q, int j) {
    const int c = totals[q] - j * kRecRows;
    return c < kRecRows ? c : kRecRows;
  };
  uint4* rec = recs + (int64_t)dl * rec_stride * 2;  // 32-byte records = 2 uint4
  for (int q = threadIdx.x; q < Tp; q += blockDim.x) counts[q] = 0;
  for (int k = threadIdx.x; k < 2 * rec_stride; k += blockDim.x) rec[k] = make_uint4(0, 0, 0, 0);
  const float sx = dirs[2 * p], sy = dirs[2 * p + 1];
  const int maxd = H > W ? H : W;
  const double S = (double)(maxd - 1 > 1 ? maxd - 1 : 1);
  __syncthreads();
  for (int v = threadIdx.x; v < HW; v += blockDim.x) {
    const int r = v / W, c = v % W;
    const double h = __dadd_rn(__dmul_rn((double)axis_coord(c, W, S), (double)sx),
                               __dmul_rn((double)axis_coord(r, H, S), (double)sy));
    const int bq = alpha64(h, g);
    vbin[v] = (uint16_t)bq;
    atomicAdd(&counts[bq], 1);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // record bases: exclusive scan of max(1, ceil(count / 7)) over bins
    const int lane = threadIdx.x, per = (Tp + 31) / 32, q0 = lane * per;
    int s = 0;
    for (int q = q0; q < q0 + per && q < Tp; ++q) s += counts[q] > kRecRows ? (counts[q] + kRecRows - 1) / kRecRows : 1;
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int base = incl - s;
    for (int q = q0; q < q0 + per && q < Tp; ++q) {
      rbase[q] = base;  // ascending exclusive scan E(q) for now
      base += counts[q] > kRecRows ? (counts[q] + kRecRows - 1) / kRecRows : 1;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    // split bin (a multiple of the 8-bin output chunk): the lower warp sweeps [0, sb) upward,
    // the upper warp [sb, Tp) downward; balanced on ~3.5 instructions per row + ~22 per record.
    // Warp-parallel: a scan of the per-bin costs, each lane's chunk boundaries scored
    // |2 acc - total|, and the smallest (score, boundary) taken by one warp min-reduction.
    {
      auto cost = [&](int q) { return 7 * counts[q] + 44 * (counts[q] > kRecRows ? (counts[q] + kRecRows - 1) / kRecRows : 1); };
      int cs = 0;
      for (int q = q0; q < q0 + per && q < Tp; ++q) cs += cost(q);
      int cinc = cs;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, cinc, o);
        if (lane >= o) cinc += t;
      }
      const int wtot = __shfl_sync(0xffffffffu, cinc, 31);
      int acc = cinc - cs;
      unsigned key = lane == 31 ? ((unsigned)wtot << 10) | (unsigned)(Tp >> 3) : 0xFFFFFFFFu;  // boundary Tp
      for (int q = q0; q < q0 + per && q < Tp; ++q) {
        if ((q & 7) == 0) {
          const unsigned k = ((unsigned)abs(2 * acc - wtot) << 10) | (unsigned)(q >> 3);
          key = k < key ? k : key;
        }
        acc += cost(q);
      }
      key = __reduce_min_sync(0xffffffffu, key);
      if (lane == 0) sh_split = (int)(key & 1023u) << 3;
    }
    __syncwarp();
    if (lane == 0) {
      const int sb = sh_split;
      const int nl = sb < Tp ? rbase[sb] : tot;
      split[dl] = make_int4(nl, tot - nl, sb, 0);
      sh_nl = nl;
    }
    __syncwarp();
    // records of the upper program run from the top bin down: bin q >= sb starts at
    // nl + (records of the bins above q)
    const int sb = sh_split, nl = sh_nl;
    for (int q = q0; q < q0 + per && q < Tp; ++q)
      if (q >= sb) {
        const int nr = counts[q] > kRecRows ? (counts[q] + kRecRows - 1) / kRecRows : 1;
        rbase[q] = nl + tot - rbase[q] - nr;
      }
    if (lane == 0) {
      // cubical: quadrant (s_x > 0) | (s_y > 0) << 1; Freudenthal: chamber | (s_x + s_y > 0) << 2
      const int o = (sx > 0.f ? 1 : 0) | (sy > 0.f ? 2 : 0) | ((freud && sx + sy > 0.f) ? 4 : 0);
      const int slot = atomicAdd(&qcount[o], 1);
      qlist[o * Dc + slot] = dl;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < Tp; q += blockDim.x) {  // record headers
    const int c = counts[q];
    totals[q] = c;
    const int nrec = c > kRecRows ? (c + kRecRows - 1) / kRecRows : 1;
    for (int j = 0; j < nrec; ++j) {
      const int n = c - j * kRecRows < kRecRows ? c - j * kRecRows : kRecRows;
      const int ne = n + (n & 1);
      uint16_t* r16 = (uint16_t*)(rec + 2 * (rbase[q] + j));
      r16[0] = (uint16_t)(ne | (j + 1 < nrec ? 16 : 0));
      if (n & 1) r16[1 + rec_slot(ne, n)] = (uint16_t)HW;  // the zero row
    }
  }
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
  __syncthreads();  // headers written before the row slots of the same records
  for (int v = threadIdx.x; v < HW; v += blockDim.x) {
    const int bq = vbin[v];
    const int r = atomicAdd(&counts[bq], -1) - 1;  // position within the bin
    const int j = r / kRecRows, p = r - j * kRecRows;
    const int n = counts_total_rows(bq, j);
    ((uint16_t*)(rec + 2 * (rbase[bq] + j)))[1 + rec_slot(n + (n & 1), p)] = (uint16_t)v;
  }
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m), "r"(src),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// stage byte offset of (image row r, 16-byte chunk j): 32-byte rows, CU_TENSOR_MAP_SWIZZLE_32B
// (address bit 4 ^= bit 7); a quarter-warp writing rows r0..r0+7 hits 8 distinct 16-byte
// bank groups.
__device__ __forceinline__ uint32_t stage_off(int r, int j) { return (uint32_t)(r * kStageRow + 16 * (j ^ ((r >> 2) & 1))); }

// Freudenthal combined weight of vertex (r, c) for chamber (A, B, C): the signed weights of
// the simplices (anchored at v - delta) whose designated vertex is v (freud_des), packed
// u16x2 for images (lane, lane+32): positives (vertex, U, L) minus negatives (3 edges),
// each sum <= 765 per half.  p0 = this lane's pixel pair of vertex v in the staged rows.
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

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// shared address of cw row (u16 half of w) for this lane: base + row * 128 (LOP3/SHF + IMAD)
__device__ __forceinline__ uint32_t row_lo(uint32_t base, uint32_t w) {
  uint32_t r;
  asm("{.reg .u32 t; and.b32 t, %1, 0xFFFF; shl.b32 t, t, 7; add.u32 %0, t, %2;}" : "=r"(r) : "r"(w), "r"(base));
  return r;
}
__device__ __forceinline__ uint32_t row_hi(uint32_t base, uint32_t w) {
  uint32_t r;
  asm("{.reg .u32 t; shr.u32 t, %1, 16; shl.b32 t, t, 7; add.u32 %0, t, %2;}" : "=r"(r) : "r"(w), "r"(base));
  return r;
}

// Per-warp record ring: the direction's program streams HBM/L2 -> shared memory through
// two halves of 16 records (cp.async.bulk, one mbarrier per half), refilled 16 records
// ahead of use, so the gathers never wait on an L2 round trip.
struct Ring {
  uint8_t* buf;   // kRingBytes
  uint64_t* bar;  // [2]
  uint32_t ph;    // bit h: parity of half h's next completion
};
__device__ __forceinline__ void ring_fill(const Ring& R, int h, const uint4* prog, int first, int nrec) {
  const int n = nrec - first < 16 ? nrec - first : 16;
  if (n <= 0) return;
  mbar_arrive_expect_tx(R.bar + h, (unsigned)n * 32u);
  bulk_g2s_plain(R.buf + h * (kRingBytes / 2), prog + 2 * first, (unsigned)n * 32u, R.bar + h);
}

// One warp, one half of one direction, the CTA's 64 images: run the half's record program.
// DOWN = false: bins [q_lo, q_hi) upward, the running total is the cumulative sum of the
// rows seen (Alg. 1 line 11).  DOWN = true: bins [q_lo, q_hi) from the top down, the running
// total R sums the rows of the bins ABOVE the current one and the emitted value is
// total - R -- the same cumulative sum, since total = sum of every cw row = chi of the image
// (top bin), so neither half waits for the other.  lane_s = shared address of this lane's
// word of cw row 0 (row v at lane_s + 128 v); totals (t0, t1) of images (img0 + lane,
// img0 + lane + 32); chunk stage st (this warp's).
template <typename OutT, bool TMA, bool DOWN>
__device__ __forceinline__ void sweep_half(uint32_t lane_s, const uint4* __restrict__ prog, int nrec, Ring& R,
                                           uint8_t* __restrict__ st, const CUtensorMap* tmap, OutT* __restrict__ out,
                                           int64_t B, int64_t img0, int Dc, int dl, int T, int q_lo, int q_hi,
                                           int t0, int t1, int lane, bool prefilled) {
  constexpr int CB = chunk_bins((int)sizeof(OutT));
  constexpr int PER = 16 / (int)sizeof(OutT);  // bins per 16-byte chunk
  if (q_lo >= q_hi) return;
  if (lane == 0 && !prefilled) {
    ring_fill(R, 0, prog, 0, nrec);
    ring_fill(R, 1, prog, 16, nrec);
  }
  uint32_t ring_s;  // pinned, see st_s
  asm volatile("mov.b32 %0, %1;" : "=r"(ring_s) : "r"(smem_u32(R.buf)));
  uint32_t ro = 0;   // byte offset of the next record in the ring (32 records of 32 B)
  int fill = 32;     // first record of the next refill
  int used = 0;      // records consumed
  int B0 = 0, B1 = 0;
  // pinned (asm): otherwise the compiler re-derives the stage address from the dynamic
  // shared window (~16 uniform instructions) at every chunk store
  uint32_t st_s;
  asm volatile("mov.b32 %0, %1;" : "=r"(st_s) : "r"(smem_u32(st)));
  mbar_wait(R.bar, R.ph & 1u);  // the first half
  R.ph ^= 1u;
  // the rows of one bin: all its records, folded onto (B0, B1)
  auto take_bin = [&]() {
    uint32_t more;
    do {
      uint4 a, b;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "r"(ring_s + ro));
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "r"(ring_s + ro + 16));
      ro = (ro + 32u) & (kRingBytes - 1);
      ++used;
      if ((ro & (kRingBytes / 2 - 1)) == 0) {  // crossed into the other half (every 16 records)
        __syncwarp();
        if (lane == 0 && fill < nrec) ring_fill(R, (int)(ro >> 9) ^ 1, prog, fill, nrec);  // refill 32 ahead
        fill += 16;
        if (used < nrec) {
          const int h = (int)(ro >> 9);
          mbar_wait(R.bar + h, (R.ph >> h) & 1u);
          R.ph ^= 1u << h;
        }
      }
      // the header is the same in every lane: a warp reduction tells the compiler so (uniform
      // branches, no reconvergence barriers around the row blocks)
      const uint32_t hdr = __reduce_or_sync(0xffffffffu, a.x);
      const uint32_t n = hdr & 15u;
      more = hdr & 16u;
      uint32_t S = 0;
      if (n & 8u)
        S = lds32(row_hi(lane_s, a.x)) + lds32(row_lo(lane_s, a.y)) + lds32(row_hi(lane_s, a.y)) +
            lds32(row_lo(lane_s, a.z)) + lds32(row_hi(lane_s, a.z)) + lds32(row_lo(lane_s, a.w)) +
            lds32(row_hi(lane_s, a.w)) + lds32(row_lo(lane_s, b.x));
      if (n & 4u)
        S += lds32(row_hi(lane_s, b.x)) + lds32(row_lo(lane_s, b.y)) + lds32(row_hi(lane_s, b.y)) +
             lds32(row_lo(lane_s, b.z));
      if (n & 2u) S += lds32(row_hi(lane_s, b.z)) + lds32(row_lo(lane_s, b.w));
      // signed packed pair S = s0 + s1 2^16 (mod 2^32), |s0|, |s1| <= 14 * 765
      const int s0 = (int)(int16_t)(S & 0xFFFFu);
      B0 += s0;
      B1 += ((int)S - s0) >> 16;
    } while (more);
  };
  const int nchunk = (q_hi - q_lo) / CB;
#pragma unroll 1
  for (int ci = 0; ci < nchunk; ++ci) {
    const int q0 = DOWN ? q_hi - (ci + 1) * CB : q_lo + ci * CB;
    // one 16-byte half-row (PER bins) at a time: take its bins, store them -- only 2 PER
    // outputs live in registers; the stage is free once the previous store has read it
#pragma unroll
    for (int jj = 0; jj < CB / PER; ++jj) {
      const int j = DOWN ? CB / PER - 1 - jj : jj;
      int o0[PER], o1[PER];
      if (!DOWN) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          take_bin();
          o0[k] = B0;
          o1[k] = B1;
        }
      } else {
#pragma unroll
        for (int k = PER - 1; k >= 0; --k) {
          o0[k] = t0 - B0;  // rows of the bins above k only
          o1[k] = t1 - B1;
          take_bin();
        }
      }
      if (jj == 0) {
        // the previous chunk's TMA store has finished reading the stage
        if (TMA && lane == 0) tma_wait_read_all();
        __syncwarp();
      }
      if (sizeof(OutT) == 4) {
        *(int4*)(st + stage_off(lane, j)) = make_int4(o0[0], o0[1 % PER], o0[2 % PER], o0[3 % PER]);
        *(int4*)(st + stage_off(lane + 32, j)) = make_int4(o1[0], o1[1 % PER], o1[2 % PER], o1[3 % PER]);
      } else {
        *(longlong2*)(st + stage_off(lane, j)) = make_longlong2(o0[0], o0[1 % PER]);
        *(longlong2*)(st + stage_off(lane + 32, j)) = make_longlong2(o1[0], o1[1 % PER]);
      }
    }
    if (TMA) {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) tma_store_3d(tmap, st_s, q0, dl, (int)img0);
    } else {
      __syncwarp();
      // generic store (misaligned output / odd T): element by element with bounds
      for (int e = lane; e < kSweepImgs * CB; e += 32) {
        const int rr = e / CB, k = e - rr * CB;
        const int64_t img = img0 + rr;
        if (img < B && q0 + k < T) {
          const OutT v = *(const OutT*)(st + stage_off(rr, k / PER) + (k % PER) * sizeof(OutT));
          out[(img * Dc + dl) * (int64_t)T + q0 + k] = v;
        }
      }
      __syncwarp();
    }
  }
  // the stage and ring are reused (and overlaid by the next phase's pixels): reads done
  if (TMA && lane == 0) tma_wait_read_all();
  __syncwarp();
}

template <typename OutT, bool FREUD, bool TMA>
__global__ void __launch_bounds__(kSweepWarps * 32, 1)
    k_sweep2d(const uint8_t* __restrict__ img, int64_t B, int H, int W, const uint4* __restrict__ recs, int rec_stride,
              const int* __restrict__ qlist, const int* __restrict__ qcount, const int4* __restrict__ split, int Dc,
              int T, int Tp, OutT* __restrict__ out, uint8_t* __restrict__ pix_park,
              const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1024-aligned (the swizzle pattern of the TMA stores), kept in the shared window
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  const int HW = H * W;
  uint32_t* cwb = (uint32_t*)smem;  // [HW][32] words: images (j, j+32) signed packed
  uint8_t* stages = smem + sweep_cw_bytes(HW);
  uint8_t* rings = stages + kSweepWarps * kStageBytes;
  uint64_t* bars = (uint64_t*)(rings + kSweepWarps * kRingBytes);
  int* totals = (int*)(bars + 2 * kSweepWarps);  // [32 lanes][2]: chi of images (lane, lane + 32)
  uint8_t* pix = stages;  // [HW][kPixStride] u8, overlays the stages: byte 2j + h = image j + 32 h
  uint64_t* pbar = (uint64_t*)(totals + 2 * 32);  // pixel reload barrier
  // parked pixels (one staged block per image group) unless CTAs share groups (gridDim.y > 1)
  const bool park = pix_park != nullptr && gridDim.y == 1;
  const unsigned pbytes = (unsigned)sweep_pix_bytes(HW);
  uint32_t pph = 0;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int half = warp & 1, wpair = warp >> 1;
  uint8_t* st = stages + warp * kStageBytes;
  Ring ring{rings + warp * kRingBytes, bars + 2 * warp, 0u};
  if (threadIdx.x < 2 * kSweepWarps) mbar_init(bars + threadIdx.x, 1);
  if (threadIdx.x < 32) cwb[HW * 32 + threadIdx.x] = 0u;  // the pad row
  if (threadIdx.x == 0) mbar_init(pbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const uint32_t lane_s = (uint32_t)__cvta_generic_to_shared(cwb) + 4u * lane;
  const int64_t ngroups = (B + kSweepImgs - 1) / kSweepImgs;
  constexpr int NPH = FREUD ? 8 : 4;  // phase (quadrant / chamber) slots
  constexpr int NPAIR = kSweepWarps / 2;
  const bool phase_split = (int)gridDim.y >= NPH;
  const int ysub = phase_split ? (int)blockIdx.y / NPH : (int)blockIdx.y;
  const int nsub = phase_split ? (int)gridDim.y / NPH : (int)gridDim.y;

  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int64_t img0 = grp * kSweepImgs;
    const int nimg = (int)((B - img0) < kSweepImgs ? (B - img0) : kSweepImgs);
    bool need_tot = true, staged = false;
    uint8_t* parked = park ? pix_park + grp * (int64_t)pbytes : nullptr;
#pragma unroll 1
    for (int o = 0; o < NPH; ++o) {
      const int qco = qcount[o];
      // small batches: blockIdx.y splits the work over gridDim.y CTAs -- by phase when
      // gridDim.y >= the phase count (then by direction within the phase), else by direction
      if (phase_split && (int)blockIdx.y % NPH != o) continue;
      if (ysub >= qco) continue;
      // this warp's first half-direction of the phase: start streaming its program now, so the
      // first records arrive while the CTA stages pixels and builds cw
      const int kfirst = ysub + wpair * nsub;
      if (kfirst < qco && lane == 0) {
        const int dl0 = qlist[o * Dc + kfirst];
        const int4 sp0 = split[dl0];
        const uint4* prog0 = recs + (int64_t)dl0 * rec_stride * 2 + (half ? 2 * sp0.x : 0);
        const int nrec0 = half ? sp0.y : sp0.x;
        const bool live = half ? sp0.z < Tp : sp0.z > 0;
        if (live) {
          ring_fill(ring, 0, prog0, 0, nrec0);
          ring_fill(ring, 1, prog0, 16, nrec0);
        }
      }
      // the previous phase's generic stage accesses are ordered before the bulk copy below
      if (park && staged) fence_proxy_async();
      __syncthreads();  // previous phase's sweeps are done with cwb and the stages
      const bool reload = park && staged;
      if (reload) {
        // this group's transposed pixels, parked by its first phase (L2-resident)
        if (threadIdx.x == 0) {
          mbar_arrive_expect_tx(pbar, pbytes);
          bulk_g2s_plain(pix, parked, pbytes, pbar);
        }
        mbar_wait(pbar, pph);
        pph ^= 1u;
      } else if ((HW & 15) == 0 && ((uintptr_t)img & 15) == 0) {
        // stage the group's pixels transposed: image i -> byte 2 (i % 32) + i / 32 of pix[v]
        const int per = HW >> 4;
        for (int f = threadIdx.x; f < kSweepImgs * per; f += blockDim.x) {
          const int i = f & (kSweepImgs - 1), v = (f >> 6) << 4;
          uint4 x = make_uint4(0, 0, 0, 0);
          if (i < nimg) x = __ldg((const uint4*)(img + (img0 + i) * HW + v));
          const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
          const int pos = 2 * (i & 31) + (i >> 5);
#pragma unroll
          for (int k = 0; k < 16; ++k) pix[(v + k) * kPixStride + pos] = (uint8_t)(wv[k >> 2] >> (8 * (k & 3)));
        }
      } else {
        for (int f = threadIdx.x; f < kSweepImgs * HW; f += blockDim.x) {
          const int i = f & (kSweepImgs - 1), v = f >> 6;
          pix[v * kPixStride + 2 * (i & 31) + (i >> 5)] = i < nimg ? img[(img0 + i) * HW + v] : (uint8_t)0;
        }
      }
      const bool park_now = park && !staged;
      staged = true;
      if (park_now) fence_proxy_async();  // the STS above, before the bulk store reads them
      __syncthreads();
      if (park_now && threadIdx.x == 0) bulk_s2g(parked, pix, pbytes);
      if (FREUD) {
        int v = warp;
        int r = v / W, c = v - r * W;
        const int step_r = kSweepWarps / W, step_c = kSweepWarps - step_r * W;
        for (; v < HW; v += kSweepWarps) {
          cwb[v * 32 + lane] = freud_cw(pix + v * kPixStride + 2 * lane, r, c, H, W, o & 1, (o >> 1) & 1, (o >> 2) & 1);
          r += step_r;
          c += step_c;
          if (c >= W) { c -= W; ++r; }
        }
      } else {
        // task (row rr, m): pixel bytes 4m..4m+3 of the row's vertices = images (2m, 2m+32, 2m+1,
        // 2m+33) -> cw words 2m, 2m+1 of every vertex of the row, as signed packed pairs
        // cw_lo + cw_hi 2^16 (mod 2^32): (a + m_diag) - (m_c + m_r) per u16 half (each operand half
        // <= 510, so a negative low half borrows into the high half exactly as the packed pair
        // encodes it).  The row is walked against dc, so the column neighbour (c + dc) and its
        // row neighbour are the previous step's pixels (2 loads per vertex).  Missing
        // neighbours (grid border) drop their cells: m_c / m_r / m_diag = 0.
        const int dc = (o & 1) ? -1 : 1, dr = (o & 2) ? -1 : 1;
        for (int t = threadIdx.x; t < H * 16; t += kSweepWarps * 32) {
          const int rr = t >> 4, m = t & 15;
          const bool vr = (unsigned)(rr + dr) < (unsigned)H;
          const int orr = vr ? dr * W * kPixStride : 0;
          const int c0 = dc > 0 ? W - 1 : 0;
          const uint8_t* p0 = pix + (rr * W + c0) * kPixStride + 4 * m;
          uint32_t* q0 = cwb + (rr * W + c0) * 32 + 2 * m;
          uint32_t Cp[2] = {0u, 0u}, Dp[2] = {0u, 0u};
          for (int step = 0; step < W; ++step) {
            const uint32_t xa = *(const uint32_t*)p0, xr = *(const uint32_t*)(p0 + orr);
            uint32_t cw[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t sel = h ? 0x4342u : 0x4140u;
              const uint32_t A = __byte_perm(xa, 0, sel), R = __byte_perm(xr, 0, sel);
              const uint32_t MC = step > 0 ? __vmaxu2(A, Cp[h]) : 0u;
              const uint32_t MR = vr ? __vmaxu2(A, R) : 0u;
              const uint32_t MD = (step > 0 && vr) ? __vmaxu2(__vmaxu2(MC, MR), Dp[h]) : 0u;
              cw[h] = (A + MD) - (MC + MR);
              Cp[h] = A;
              Dp[h] = R;
            }
            *(uint2*)q0 = make_uint2(cw[0], cw[1]);
            p0 -= dc * kPixStride;
            q0 -= dc * 32;
          }
        }
      }
      if (park_now && threadIdx.x == 0) tma_wait_read_all();  // pix (= the stages) is read out
      __syncthreads();
      // totals: every cell is counted once in the cw table of ANY phase, so the sum of all cw
      // rows is the image's weighted Euler characteristic (the top bin of every direction):
      // computed in the group's first phase only
      if (need_tot) {
        need_tot = false;
        uint32_t S = 0;
        for (int v = warp; v < HW; v += kSweepWarps) S += cwb[v * 32 + lane];  // <= 32 rows: no carry
        const int s0 = (int)(int16_t)(S & 0xFFFFu);
        int* red = (int*)stages;  // [32 warps][32 lanes][2], the pixels are no longer needed
        red[(warp * 32 + lane) * 2] = s0;
        red[(warp * 32 + lane) * 2 + 1] = ((int)S - s0) >> 16;
        __syncthreads();
        if (warp == 0) {
          int a0 = 0, a1 = 0;
          for (int w2 = 0; w2 < kSweepWarps; ++w2) {
            a0 += red[(w2 * 32 + lane) * 2];
            a1 += red[(w2 * 32 + lane) * 2 + 1];
          }
          totals[2 * lane] = a0;
          totals[2 * lane + 1] = a1;
        }
        __syncthreads();
      }
      const int t0 = totals[2 * lane], t1 = totals[2 * lane + 1];
      for (int k = ysub + wpair * nsub; k < qco; k += NPAIR * nsub) {
        const int dl = __shfl_sync(0xffffffffu, qlist[o * Dc + k], 0);
        const int4 sp = split[dl];  // (records below, records above, split bin)
        const uint4* prog = recs + (int64_t)dl * rec_stride * 2;
        const bool pre = k == kfirst;
        if (half == 0)
          sweep_half<OutT, TMA, false>(lane_s, prog, sp.x, ring, st, &tmap, out, B, img0, Dc, dl, T, 0, sp.z, t0, t1,
                                       lane, pre);
        else
          sweep_half<OutT, TMA, true>(lane_s, prog + 2 * sp.x, sp.y, ring, st, &tmap, out, B, img0, Dc, dl, T, sp.z,
                                      Tp, t0, t1, lane, pre);
      }
    }
  }
  if (TMA && lane == 0) tma_wait_all();
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
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// TMA map of out [B][Dc][T] (element osz bytes), box [64 images][1][CB bins], 32B swizzle.
// false: not expressible (alignment / strides) -> the generic store path.
static bool make_out_map(CUtensorMap* m, void* out, int64_t B, int Dc, int T, int osz) {
  if (((uintptr_t)out & 15) != 0 || ((int64_t)T * osz) % 16 != 0 || B > 0xFFFFFFFFll) return false;
  PFN_cuTensorMapEncodeTiled_v12000 enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)T, (cuuint64_t)Dc, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)T * osz, (cuuint64_t)Dc * T * osz};
  const cuuint32_t box[3] = {(cuuint32_t)chunk_bins(osz), 1u, (cuuint32_t)kSweepImgs};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  const CUresult r = enc(m, osz == 4 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_INT64, 3, out, dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool sweep2d_supported(int ndim, const int64_t* dims, int T) {
  if (ndim != 2) return false;
  const int64_t HW = dims[0] * dims[1];
  return HW >= 1 && HW <= kSweepMaxHW && T <= 4096 && sweep_smem_bytes((int)HW) <= 227 * 1024 &&
         sweep_pix_fits((int)HW);
}

static int padded_bins(int T) { return (T + 7) & ~7; }  // a whole number of chunks for int32 and int64

// parked pixel blocks: only when every CTA owns whole image groups (B >= 64 * SMs-ish)
static bool sweep_parks(int64_t B, int num_sms) { return (B + kSweepImgs - 1) / kSweepImgs >= num_sms; }

size_t sweep2d_scratch_bytes(int HW, int Dc, int T, int freud, int64_t B, int num_sms) {
  return (size_t)Dc * sweep_rec_stride(HW, padded_bins(T)) * 32 + 64 + (size_t)(8 + 8 * Dc + 1) * 4 + 64 +
         (size_t)Dc * 16 + 16 + (freud ? (size_t)5 * HW * Dc * sizeof(int4) + 16 : 0) +
         (sweep_parks(B, num_sms) ? (size_t)((B + kSweepImgs - 1) / kSweepImgs) * sweep_pix_bytes(HW) + 16 : 0);
}

wect_status launch_sweep2d(const uint8_t* img, int64_t B, int H, int W, const float* dirs, int d_begin, int Dc,
                           int T, const GridParams* gp, void* scratch, void* out, wect_dtype odtype, cudaStream_t st,
                           int num_sms, int freud) {
  const int HW = H * W;
  const int Tp = padded_bins(T);
  const int rstride = sweep_rec_stride(HW, Tp);
  uint4* recs = (uint4*)align_up((uintptr_t)scratch, 16);
  int* ints = (int*)align_up((uintptr_t)(recs + (size_t)Dc * rstride * 2), 16);
  int* qcount = ints;           // 8 chamber slots (cubical uses 4)
  int* qlist = ints + 8;        // [8][Dc]
  int4* split = (int4*)align_up((uintptr_t)(qlist + 8 * Dc), 16);  // [Dc]
  int* ncorr = (int*)(split + Dc);
  int4* corr = (int4*)align_up((uintptr_t)(ncorr + 1), 16);
  const int corr_cap = freud ? 5 * HW * Dc : 0;
  uint8_t* pix_park = sweep_parks(B, num_sms) ? (uint8_t*)align_up((uintptr_t)(corr + corr_cap), 16) : nullptr;
  if (getenv("WECT_SWEEP_NOPARK")) pix_park = nullptr;
  WECT_CUDA_TRY(cudaMemsetAsync(qcount, 0, 8 * sizeof(int), st));
  WECT_CUDA_TRY(cudaMemsetAsync(ncorr, 0, sizeof(int), st));
  const size_t sort_smem = (size_t)3 * Tp * sizeof(int) + align_up((size_t)HW * 2, 16);
  if (sort_smem > 48 * 1024)
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_sort2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem));
  k_sort2d<<<Dc, 256, sort_smem, st>>>(H, W, dirs, d_begin, Dc, gp, recs, rstride, Tp, qlist, qcount, split, freud,
                                       corr, ncorr, corr_cap);
  count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  const size_t smem = sweep_smem_bytes(HW);
  const int64_t ngroups = (B + kSweepImgs - 1) / kSweepImgs;
  // fewer image groups than SMs (small batches): split every phase's directions over CTAs
  const int nph = freud ? 8 : 4;
  int ysplit = (int)(num_sms / (ngroups > 0 ? ngroups : 1));
  ysplit = ysplit < 1 ? 1 : (ysplit > (kSweepWarps / 2) * nph ? (kSweepWarps / 2) * nph : ysplit);
  if (ysplit >= nph) ysplit = (ysplit / nph) * nph;  // whole phase rows: y = phase + nph * sub
  const dim3 grid((unsigned)(ngroups < num_sms ? ngroups : num_sms), (unsigned)ysplit);
  const int osz = odtype == WECT_I32 ? 4 : 8;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  const bool tma = getenv("WECT_SWEEP_NOTMA") == nullptr && make_out_map(&tmap, out, B, Dc, T, osz);
  MainTimer timer(st);
#define WECT_SWEEP(OT, FR, TM)                                                                                      \
  do {                                                                                                              \
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_sweep2d<OT, FR, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_sweep2d<OT, FR, TM><<<grid, kSweepWarps * 32, smem, st>>>(img, B, H, W, recs, rstride, qlist, qcount, split, Dc, T, \
                                                                 Tp, (OT*)out, pix_park, tmap);                         \
    count_launch();                                                                                                 \
  } while (0)
#define WECT_SWEEP_T(OT, FR) \
  do {                       \
    if (tma) WECT_SWEEP(OT, FR, true); else WECT_SWEEP(OT, FR, false); \
  } while (0)
  if (odtype == WECT_I32) {
    if (freud) WECT_SWEEP_T(int32_t, true); else WECT_SWEEP_T(int32_t, false);
  } else {
    if (freud) WECT_SWEEP_T(long long, true); else WECT_SWEEP_T(long long, false);
  }
#undef WECT_SWEEP_T
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

}  // namespace wect
