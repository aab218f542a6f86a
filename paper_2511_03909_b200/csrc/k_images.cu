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
// Kernels here: k_grid_params (M over the grid corners, all directions) and the
// histogram path for volumes and images larger than the sweep handles: k_grid_cw writes
// the orthant-combined weights, k_grid_hist streams them with lanes = 32 directions into
// shared-memory int32 histograms [32][T+1], one int64 merge per CTA, then k_finalize's
// cumsum.  The 2-D image-batch sweep (BASELINE configs[0], configs[1]) is in k_sweep.cu.
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
    // the grid [lo, hi] holds every height of every direction (always for the paper grid):
    // the fast bin of a voxel far from a bin edge is then in [0, T-1] without clamping
    g.covers = (!g.fp32_only && !g.degenerate && g.lo <= -red[0] && g.hi >= red[0] && T < (1 << 22)) ? 1 : 0;
    *out = g;
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
constexpr int kSegVox = 128;     // voxels per staged row segment
constexpr int kSegStride = 136;  // int16 per staged octant row (68 words = 4 mod 32: conflict-free)

// Inlined and called from warp-uniform loops only: a divergent (noinline) repair call left
// warps split for the rest of the kernel (measured in k_vbins: 1.5x the instructions).
__device__ __forceinline__ int grid_repair(float cx, float cy, float cz, float s0, float s1, float s2, int nd,
                                           const GridParams* gp) {
  double h64 = __dadd_rn(__dmul_rn((double)cx, (double)s0), __dmul_rn((double)cy, (double)s1));
  if (nd == 3) h64 = __dadd_rn(h64, __dmul_rn((double)cz, (double)s2));
  return alpha64(h64, *gp);
}
// repair the voxels flagged in nm (bit h: voxel x + h of this lane's row) in a warp-uniform
// loop; out[h] = f(binary64 bin of voxel h)
template <typename F>
__device__ __forceinline__ void grid_repair_mask(uint32_t nm, const float* axc0, int x, float cy, float cz,
                                                 const float* s, int nd, const GridParams* gp, int lane, F&& set) {
  while (__any_sync(0xffffffffu, nm != 0)) {
    const bool act = nm != 0;
    const int hh = act ? __ffs(nm) - 1 : 0;
    nm &= nm - 1;
    const int r = grid_repair(axc0[x + hh], cy, cz, s[0], s[1], s[2], nd, gp);
    const unsigned c = __ballot_sync(0xffffffffu, act);
    if (lane == 0) atomicAdd(&g_repair_count, (unsigned long long)__popc(c));
    if (act) set(hh, r);
  }
}

// predicated shared-memory add (no branch, no reconvergence barrier)
__device__ __forceinline__ void red_shared_add(uint32_t addr, int w) {
  asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(w) : "memory");
}
__device__ __forceinline__ void red_shared_nz(uint32_t addr, int w) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %1, 0;\n\t@p red.shared.add.s32 [%0], %1;\n\t}" ::"r"(addr), "r"(w));
}

// The orthant-combined weights of octant o for the 4 voxels x .. x + 3 of row (y, z) of
// image im (x % 4 == 0, L0 % 4 == 0), as two int16 pairs: the signed maxima of the cells that
// designate each voxel (grid_cw_vox's rule, read from the pixels in u16x2 lanes): vertex +,
// edges -, squares +, cube -, a cell dropped when a corner falls outside the grid.
template <int ND>
__device__ __forceinline__ uint2 fused_cw4(const uint8_t* __restrict__ im, int x, int y, int z, int o, const int (&L)[3]) {
  const int ex = (o & 1) ? -1 : 1, ey = (o & 2) ? -1 : 1, ez = (o & 4) ? -1 : 1;
  const bool vy = (unsigned)(y + ey) < (unsigned)L[1];
  const bool vz = ND == 3 && (unsigned)(z + ez) < (unsigned)L[2];
  const int64_t plane = (int64_t)L[0] * L[1];
  const uint8_t* r00 = im + (int64_t)z * plane + (int64_t)y * L[0];
  const uint8_t* rows[4] = {r00, vy ? r00 + ey * L[0] : r00, vz ? r00 + ez * plane : r00,
                            (vy && vz) ? r00 + ez * plane + ey * L[0] : r00};
  uint32_t P[4][2], Cn[4][2];  // per row: the 4 voxels and their x neighbours, widened to u16x2 pairs
#pragma unroll
  for (int k = 0; k < (ND == 3 ? 4 : 2); ++k) {
    const uint32_t w = __ldg((const uint32_t*)(rows[k] + x));
    uint32_t c;
    if (ex > 0) c = __byte_perm(w, x + 4 < L[0] ? __ldg((const uint32_t*)(rows[k] + x + 4)) : 0u, 0x4321);
    else c = __byte_perm(x >= 4 ? __ldg((const uint32_t*)(rows[k] + x - 4)) : 0u, w, 0x6543);
    P[k][0] = __byte_perm(w, 0, 0x4140);
    P[k][1] = __byte_perm(w, 0, 0x4342);
    Cn[k][0] = __byte_perm(c, 0, 0x4140);
    Cn[k][1] = __byte_perm(c, 0, 0x4342);
  }
  // the voxel of the group without an x neighbour (grid border): its x-extended cells drop
  const uint32_t xm0 = (ex < 0 && x == 0) ? 0xFFFF0000u : 0xFFFFFFFFu;
  const uint32_t xm1 = (ex > 0 && x + 4 == L[0]) ? 0x0000FFFFu : 0xFFFFFFFFu;
  uint32_t res[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t xm = h ? xm1 : xm0;
    const uint32_t A = P[0][h];
    const uint32_t mx = __vmaxu2(A, Cn[0][h]) & xm;
    uint32_t my = 0u, mxy = 0u;
    if (vy) {
      my = __vmaxu2(A, P[1][h]);
      mxy = __vmaxu2(__vmaxu2(mx, P[1][h]), Cn[1][h]) & xm;
    }
    uint32_t pos = 0u, neg = 0u;
    if (ND == 2) {
      pos = A + mxy;
      neg = mx + my;
    } else {
      uint32_t mz = 0u, mxz = 0u, myz = 0u, mxyz = 0u;
      if (vz) {
        mz = __vmaxu2(A, P[2][h]);
        mxz = __vmaxu2(__vmaxu2(mx, P[2][h]), Cn[2][h]) & xm;
        if (vy) {
          myz = __vmaxu2(__vmaxu2(my, P[2][h]), P[3][h]);
          mxyz = __vmaxu2(__vmaxu2(mxy, mxz), __vmaxu2(myz, Cn[3][h])) & xm;
        }
      }
      pos = A + mxy + mxz + myz;
      neg = mx + my + mz + mxyz;
    }
    // per u16 lane pos - neg in [-1020, 1020]: offset by 2^15 so no borrow crosses lanes
    res[h] = ((pos | 0x80008000u) - neg) ^ 0x80008000u;
  }
  return make_uint2(res[0], res[1]);
}

template <int ND, bool FUSED>
__global__ void __launch_bounds__(256, 3) k_grid_hist(const int16_t* __restrict__ cwo, const uint8_t* __restrict__ img,
                                                   const int* __restrict__ perm, int64_t d0, int64_t d1, int64_t d2,
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
  // FUSED: the CTA's 32 directions are perm[blockIdx.x * 32 ..] (sorted by octant, so a tile
  // needs few octants of weights); otherwise the identity
  const int dslot = blockIdx.x * 32 + lane;
  const bool active = dslot < Dc;
  const int dl = active ? (FUSED ? perm[dslot] : dslot) : 0;
  const int p = d_begin + dl;
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
  constexpr float kMagic = 12582912.0f;  // 1.5 2^23
  const bool covers = g.covers != 0;
  const uint32_t hfast = hlane - 128u * (uint32_t)__float_as_int(kMagic);  // + 128 t = hlane + 128 bin
  // octants present in the tile; FUSED: one seg row per present octant, in octant order
  const unsigned omask = __reduce_or_sync(0xffffffffu, 1u << o);
  const int oslot = FUSED ? __popc(omask & ((1u << o) - 1u)) : o;
  const uint32_t* segw = (const uint32_t*)(seg + oslot * kSegStride);  // this lane's octant row, 2 voxels per word
  // inactive lanes (dl >= Dc) bin direction d_begin into their own column, which the flush drops
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
      if (FUSED) {
        // computed from the pixels: lane l takes voxels x0 + 4 l .. + 3 of each present octant
        const uint8_t* im = img + b * nv;
        int slot = 0;
        for (unsigned m = omask; m; m &= m - 1, ++slot) {
          const int oo = __ffs(m) - 1;
          for (int xl = 4 * lane; xl < nx; xl += 128) {
            const uint2 cw = fused_cw4<ND>(im, x0 + xl, y, z, oo, L);
            *(uint2*)(seg + slot * kSegStride + xl) = cw;
          }
        }
      } else if (((src0 | nx | nv) & 7) == 0) {
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
      // 8 voxels per step: one 16-byte load of this lane's octant row, eight fp32 bins, one
      // guard test for the group, eight red.shared adds
      if (covers) {
        // ceil without the conversion unit: t = u + 1.5 2^23 rounded up is 1.5 2^23 + ceil(u)
        // (|u| < 2^22), so t's bit pattern minus the constant's is the bin; e = ceil(u) - u
        // (exact) in [0, 1) is the distance to the bin edges: near an edge iff e < tau or
        // e > 1 - tau.  No clamp: a bin taken here is ceil(u64) in [0, T-1] (A1).
        for (int xi = 0; xi < nx; xi += 8) {
          const uint4 q = *(const uint4*)(segw + (xi >> 1));
          const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
          const float xf = (float)(x0 + xi);
          uint32_t adr[8];
          float emin = 1.f, emax = 0.f;
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const float u = fmaf(xf + (float)h, a0, U0);  // x0 + xi + h is exact in fp32
            const float t = __fadd_ru(u, kMagic);
            const float e = (t - kMagic) - u;
            emin = fminf(emin, e);
            emax = fmaxf(emax, e);
            adr[h] = hfast + 128u * (uint32_t)__float_as_int(t);
          }
          const int nvalid = nx - xi;
          if (nvalid < 8) {  // the row's zero-weight padding voxels: any in-range bin (u may be far outside)
#pragma unroll
            for (int h = 1; h < 8; ++h)
              if (h >= nvalid) adr[h] = hlane;
          }
          // warp vote: a uniform branch, no reconvergence barrier in the common case
          if (__builtin_expect(__any_sync(0xffffffffu, emin < tau || emax > 1.f - tau), 0)) {
            uint32_t nm = 0;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              const float u = fmaf(xf + (float)h, a0, U0);
              const float e = (__fadd_ru(u, kMagic) - kMagic) - u;
              nm |= ((e < tau || e > 1.f - tau) && h < nvalid ? 1u : 0u) << h;  // padding needs no repair
            }
            grid_repair_mask(nm, axc[0], x0 + xi, cy, cz, s, ND, gp, lane, [&](int hh, int r) {
#pragma unroll
              for (int h = 0; h < 8; ++h)
                if (h == hh) adr[h] = hlane + 128u * (uint32_t)r;
            });
          }
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const int w = (h & 1) ? (int)wd[h >> 1] >> 16 : (int)(int16_t)(wd[h >> 1] & 0xFFFFu);
            red_shared_add(adr[h], w);
          }
        }
      } else {
        for (int xi = 0; xi < nx; xi += 8) {
          const uint4 q = *(const uint4*)(segw + (xi >> 1));
          const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
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
          if (__builtin_expect(__any_sync(0xffffffffu, dmin < tau), 0)) {  // a voxel near a bin edge
            const int nvalid = nx - xi;  // padding voxels need no repair
            uint32_t nm = 0;
#pragma unroll
            for (int h = 0; h < 8; ++h) nm |= (dist[h] < tau && h < nvalid ? 1u : 0u) << h;
            grid_repair_mask(nm, axc[0], x0 + xi, cy, cz, s, ND, gp, lane, [&](int hh, int r) {
#pragma unroll
              for (int h = 0; h < 8; ++h)
                if (h == hh) bin[h] = r;
            });
          }
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const int w = (h & 1) ? (int)wd[h >> 1] >> 16 : (int)(int16_t)(wd[h >> 1] & 0xFFFFu);
            red_shared_add(hlane + 128u * (uint32_t)bin[h], w);
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * T; i += blockDim.x) {
    int q = i >> 5, r = i & 31;
    int val = hist[i];
    if (val != 0 && blockIdx.x * 32 + r < Dc) {
      const int dr = FUSED ? perm[blockIdx.x * 32 + r] : blockIdx.x * 32 + r;
      atomicAdd(diff + ((b_offset + b) * Dc + dr) * (int64_t)T + q, (unsigned long long)(long long)val);
    }
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

// direction order of the fused histogram path: sorted by orthant (counting sort, any order
// within an orthant), so a tile of 32 directions computes the weights of few orthants
__global__ void __launch_bounds__(256) k_dir_perm(const float* __restrict__ dirs, int nd, int d_begin, int Dc,
                                                  int* __restrict__ perm) {
  __shared__ int cnt[8], cur[8];
  if (threadIdx.x < 8) cnt[threadIdx.x] = 0;
  __syncthreads();
  auto orth = [&](int dl) {
    int o = 0;
    for (int k = 0; k < nd; ++k) o |= (dirs[(int64_t)(d_begin + dl) * nd + k] > 0.f ? 1 : 0) << k;
    return o;
  };
  for (int dl = threadIdx.x; dl < Dc; dl += blockDim.x) atomicAdd(&cnt[orth(dl)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int o = 0; o < 8; ++o) {
      cur[o] = run;
      run += cnt[o];
    }
  }
  __syncthreads();
  for (int dl = threadIdx.x; dl < Dc; dl += blockDim.x) perm[atomicAdd(&cur[orth(dl)], 1)] = dl;
}

// histogram path over a chunk of images [b0, b0 + nb): diff rows at b0.  Fused (WECT_GRID_FUSED=1,
// the x axis a multiple of 4 voxels): k_grid_hist computes the orthant weights from the pixels
// of each row segment it bins -- no weight table in HBM (cfg3: 0.018 GB of DRAM per launch
// instead of 0.278) but 21 % slower on the issue-bound binning (6.89 vs 5.70 ms),
// so the default is the table path: k_grid_cw writes the cwo table first.
bool grid_hist_fused(int ndim, const int64_t* dims, const uint8_t* img) {
  const int64_t L0 = ndim == 2 ? dims[1] : dims[2];
  const char* e = getenv("WECT_GRID_FUSED");
  return e && e[0] == '1' && (L0 % 4) == 0 && ((uintptr_t)img & 3) == 0;
}

wect_status launch_grid_hist(const uint8_t* img, int64_t b0, int64_t nb, int ndim, const int64_t* dims,
                             const float* dirs, int d_begin, int Dc, int T, const GridParams* gp, int16_t* cwo,
                             int* perm, unsigned long long* diff, cudaStream_t st, int num_sms) {
  const int64_t nv = ndim == 2 ? dims[0] * dims[1] : dims[0] * dims[1] * dims[2];
  const uint8_t* im = img + b0 * nv;
  const bool fused = grid_hist_fused(ndim, dims, img);
  if (fused) {
    k_dir_perm<<<1, 256, 0, st>>>(dirs, ndim, d_begin, Dc, perm);
    count_launch();
  } else {
    const int64_t want_x = (nv + 255) / 256;
    const int gx = (int)(want_x < (int64_t)num_sms * 16 ? want_x : (int64_t)num_sms * 16);
    int64_t gy = ((int64_t)num_sms * 16 + gx - 1) / gx;
    gy = gy < nb ? gy : nb;
    gy = gy < 65535 ? (gy < 1 ? 1 : gy) : 65535;
    dim3 gcw((unsigned)gx, (unsigned)gy);
    if (ndim == 2) k_grid_cw<2><<<gcw, 256, 0, st>>>(im, nb, dims[0], dims[1], 1, cwo);
    else k_grid_cw<3><<<gcw, 256, 0, st>>>(im, nb, dims[0], dims[1], dims[2], cwo);
    count_launch();
  }
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
#define WECT_GH(ND, FU)                                                                                          \
  do {                                                                                                           \
    WECT_CUDA_TRY(cudaFuncSetAttribute(k_grid_hist<ND, FU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_grid_hist<ND, FU><<<gridd, 256, smem, st>>>(cwo, im, perm, dims[0], dims[1], ND == 3 ? dims[2] : 1, dirs,     \
                                                  d_begin, Dc, gp, slice_rows, b0, diff);                         \
    count_launch();                                                                                              \
  } while (0)
  if (ndim == 2) {
    if (fused) WECT_GH(2, true); else WECT_GH(2, false);
  } else {
    if (fused) WECT_GH(3, true); else WECT_GH(3, false);
  }
#undef WECT_GH
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

}  // namespace wect
