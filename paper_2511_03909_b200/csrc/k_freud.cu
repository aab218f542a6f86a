// k_freud.cu -- WECT of 2-D uint8 images as weighted FREUDENTHAL complexes
// (wect_images with WECT_FREUDENTHAL).
//
// The complex: pixels are vertices (reading A3 coordinates); edges
// are the horizontal, vertical and (r,c)-(r+1,c+1) diagonal pairs; every unit square splits
// along that diagonal into U = {(r,c),(r,c+1),(r+1,c+1)} and L = {(r,c),(r+1,c),(r+1,c+1)};
// vertex weight = intensity, every other simplex's weight = max of its vertices;
// sign (-1)^dim.  The six simplices anchored at vertex (r,c) -- itself, the three edges and
// the two triangles that start there -- cover the complex once.
//
// Unlike the cubical grid, a triangle's highest vertex is not fixed by the orthant of the
// direction (the diagonal comparison depends on the sign of s_x + s_y and on rounding), so
// there is no exact designated-corner regrouping.  Instead every simplex is binned
// exactly: the bin of a simplex is the max of its vertices' exact bins (eq. msi, P:713-723;
// alpha monotone), each vertex bin from the fp32 fast path with the guard and binary64
// repair of reading A1.  Lanes = 32 directions, a warp walks an anchor row keeping the
// bins of columns x and x+1 of rows y and y+1 (two new bins per anchor), and adds the six
// signed weights (precomputed per image by k_freud_w, int16) into a lane-interleaved
// [T][32] shared histogram; int32 partials, one int64 merge per CTA, k_finalize's cumsum.
#include <cstdint>

#include "common.cuh"

namespace wect {

constexpr int kFreudCells = 6;

// per anchor (r,c) of image b: signed weights of {v, e_x, e_y, e_diag, U, L} (0 if absent)
__global__ void __launch_bounds__(256) k_freud_w(const uint8_t* __restrict__ img, int64_t nimg, int H, int W,
                                                 int16_t* __restrict__ w6) {
  const int64_t HW = (int64_t)H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nimg * HW; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / HW, v = i - b * HW;
    const int r = (int)(v / W), c = (int)(v - (int64_t)r * W);
    const uint8_t* p = img + b * HW;
    const bool hx = c + 1 < W, hy = r + 1 < H, hd = hx && hy;
    const int a = p[v];
    const int bx = hx ? p[v + 1] : 0, cy = hy ? p[v + W] : 0, d = hd ? p[v + W + 1] : 0;
    int16_t* o = w6 + b * kFreudCells * HW + v;
    o[0] = (int16_t)a;
    o[HW] = (int16_t)(hx ? -max(a, bx) : 0);
    o[2 * HW] = (int16_t)(hy ? -max(a, cy) : 0);
    o[3 * HW] = (int16_t)(hd ? -max(a, d) : 0);
    o[4 * HW] = (int16_t)(hd ? max(max(a, bx), d) : 0);
    o[5 * HW] = (int16_t)(hd ? max(max(a, cy), d) : 0);
  }
}

// binary64 height of grid vertex (x, y) in axis order, then alpha (reading A1)
__device__ __noinline__ int freud_repair(float cx, float cy, float s0, float s1, const GridParams* gp) {
  const double h = __dadd_rn(__dmul_rn((double)cx, (double)s0), __dmul_rn((double)cy, (double)s1));
  note_repair();
  return alpha64(h, *gp);
}

__device__ __forceinline__ void red_add_nz(uint32_t addr, int w) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %1, 0;\n\t@p red.shared.add.s32 [%0], %1;\n\t}" ::"r"(addr), "r"(w)
               : "memory");
}

__global__ void __launch_bounds__(256) k_freud_hist(const int16_t* __restrict__ w6, int H, int W,
                                                    const float* __restrict__ dirs, int d_begin, int Dc,
                                                    const GridParams* __restrict__ gp, int64_t slice_rows,
                                                    int64_t b_offset, unsigned long long* __restrict__ diff) {
  extern __shared__ __align__(16) int hist[];  // [T][32] lane-interleaved
  __shared__ float axc[2][1024];
  const GridParams g = *gp;
  const int T = g.T, Tm1 = T - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int maxd = H > W ? H : W;
  const double S = (double)(maxd - 1 > 1 ? maxd - 1 : 1);
  for (int i = threadIdx.x; i < W; i += blockDim.x) axc[0][i] = axis_coord(i, W, S);
  for (int i = threadIdx.x; i < H; i += blockDim.x) axc[1][i] = axis_coord(i, H, S);
  for (int i = threadIdx.x; i < 32 * T; i += blockDim.x) hist[i] = 0;
  const int dl = blockIdx.x * 32 + lane;
  const bool active = dl < Dc;
  const int p = d_begin + (active ? dl : 0);
  const float s0 = dirs[2 * p], s1 = dirs[2 * p + 1];
  const float A = g.A, Bc = g.B, tau = g.fp32_only ? -1.f : g.tau;
  const float a0 = A * s0 / (float)S;
  const float c0 = (float)((double)(W - 1) / 2.0);
  const uint32_t hlane = (uint32_t)__cvta_generic_to_shared(hist) + 4u * lane;
  const int wmask = active ? -1 : 0;
  const int64_t HW = (int64_t)H * W;
  const int64_t b = blockIdx.z;
  const int16_t* wb = w6 + b * kFreudCells * HW;
  const int r0 = (int)(blockIdx.y * slice_rows);
  const int r1 = (int)((r0 + slice_rows) < H ? (r0 + slice_rows) : H);
  __syncthreads();
  // the exact bin of grid vertex (x, y) for this lane's direction; x == W or y == H are
  // absent vertices (their simplices carry weight 0): any in-range bin will do
  auto vbin = [&](int x, int y, float U0) -> int {
    const float u = fmaf((float)x, a0, U0);
    int bq = max(0, min(__float2int_ru(u), Tm1));
    if (fabsf(u - rintf(u)) < tau && x < W && y < H) bq = freud_repair(axc[0][x], axc[1][y], s0, s1, gp);
    return bq;
  };
  auto row_u0 = [&](int y) -> float {  // the k_grid_hist evaluation order (tau covers it)
    const float C = axc[1][y < H ? y : H - 1] * s1;
    return fmaf(fmaf(-s0, c0 / (float)S, C), A, Bc);
  };
  for (int y = r0 + warp; y < r1; y += nwarps) {
    const float U0 = row_u0(y), U1 = row_u0(y + 1);
    const int16_t* wr = wb + (int64_t)y * W;
    int bv = vbin(0, y, U0), by = vbin(0, y + 1, U1);
    for (int x = 0; x < W; ++x) {
      const int bx = vbin(x + 1, y, U0), bd = vbin(x + 1, y + 1, U1);
      int w[kFreudCells];
#pragma unroll
      for (int t = 0; t < kFreudCells; ++t) w[t] = (int)__ldg(wr + t * HW + x) & wmask;
      const int cb[kFreudCells] = {bv, max(bv, bx), max(bv, by), max(bv, bd), max(max(bv, bx), bd),
                                   max(max(bv, by), bd)};
#pragma unroll
      for (int t = 0; t < kFreudCells; ++t) red_add_nz(hlane + 128u * (uint32_t)cb[t], w[t]);
      bv = bx;
      by = bd;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * T; i += blockDim.x) {
    const int q = i >> 5, r = i & 31;
    const int val = hist[i];
    if (val != 0 && blockIdx.x * 32 + r < Dc)
      atomicAdd(diff + ((b_offset + b) * Dc + blockIdx.x * 32 + r) * (int64_t)T + q, (unsigned long long)(long long)val);
  }
}

size_t freud_scratch_per_image(int H, int W) { return (size_t)kFreudCells * H * W * sizeof(int16_t); }

// images [b0, b0 + nb): weights into w6 (scratch for nb images), histogram rows at b0
wect_status launch_freud(const uint8_t* img, int64_t b0, int64_t nb, int H, int W, const float* dirs, int d_begin,
                         int Dc, int T, const GridParams* gp, int16_t* w6, unsigned long long* diff, cudaStream_t st,
                         int num_sms) {
  const int64_t HW = (int64_t)H * W;
  const int64_t total = nb * HW;
  int blocks = (int)((total + 255) / 256 < (int64_t)num_sms * 16 ? (total + 255) / 256 : (int64_t)num_sms * 16);
  k_freud_w<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(img + b0 * HW, nb, H, W, w6);
  count_launch();
  WECT_CUDA_TRY(cudaGetLastError());
  const int tiles = (Dc + 31) / 32;
  // row slices: int32 partials stay below 2^31 (<= 2^18 anchors x 6 simplices x 255 per CTA)
  int64_t rows_cap = ((int64_t)1 << 18) / W;
  if (rows_cap < 1) rows_cap = 1;
  int64_t want = ((int64_t)num_sms * 8 + tiles * nb - 1) / (tiles * nb);
  if (want < 1) want = 1;
  int64_t slice = (H + want - 1) / want;
  if (slice > rows_cap) slice = rows_cap;
  if (slice < 1) slice = 1;
  const int64_t nslices = (H + slice - 1) / slice;
  const size_t smem = (size_t)32 * T * sizeof(int);
  WECT_CUDA_TRY(cudaFuncSetAttribute(k_freud_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)tiles, (unsigned)nslices, (unsigned)nb);
  MainTimer timer(st);
  k_freud_hist<<<grid, 256, smem, st>>>(w6, H, W, dirs, d_begin, Dc, gp, slice, b0, diff);
  count_launch();
  timer.stop();
  WECT_CUDA_TRY(cudaGetLastError());
  return WECT_OK;
}

}  // namespace wect
