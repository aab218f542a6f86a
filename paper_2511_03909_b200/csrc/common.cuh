// common.cuh -- shared device helpers of libwect (the CUDA path).  Nothing here is
// shared with oracle/; the binary64 expression below is re-derived from the paper.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/wect.h"

namespace wect {

constexpr int kMaxDims = 8;     // ambient dimension n <= 8
constexpr int kMaxSegs = 10;    // vertices + up to 9 cell dimensions per call
constexpr float kEps32 = 5.9604644775390625e-08f;  // 2^-24

// Per-call grid constants, computed ON DEVICE (k_grid_params) so that no call has to
// synchronise with the host to learn M.
struct GridParams {
  double lo, hi;  // height grid [lo, hi]; paper grid: lo = -M, hi = M
  double Tm1;     // T - 1
  double M;       // maxheight
  float A, B;     // fast path: u = fmaf(h32, A, B) ~ (T-1)(h - lo)/(hi - lo)
  float tau;      // near-edge guard (A1): |u32 - rint(u32)| < tau -> binary64 repair
  int32_t T;
  int32_t degenerate;  // hi <= lo (M = 0): every value is bin 0 (reading A6)
  int32_t fp32_only;   // WECT_FP32_ONLY
  int32_t covers;      // grids: [lo, hi] holds every height (fast bins need no clamp); else 0
};

// Segments of the virtual cell index space of an explicit complex: segment 0 is the
// vertices (dimension 0), then one per cell dimension (the Complex list).
struct Seg {
  const int32_t* verts;  // nullptr: the vertex segment (cell b is vertex b)
  const void* weights;   // nullptr: unit weights
  int64_t count;
  int64_t start;  // offset in the virtual cell index space
  int32_t arity;
  int32_t sign;  // (-1)^dim
};
struct Segs {
  Seg s[kMaxSegs];
  int32_t nseg;
  int32_t pad;
  int64_t total;
};

// Backward outputs (k_grad.cu): per segment an [count] fp64 gradient, or nullptr (skip).
struct GradOut {
  double* g[kMaxSegs];
};

// Device-global diagnostics (one per device, per loaded library).
extern __device__ unsigned int g_err_word;            // bit 0: out-of-range vertex index
extern __device__ unsigned long long g_repair_count;  // binary64 near-edge repairs

// alpha(t) of eq. left-adjoint in IEEE binary64, operation for operation:
//   u = ((T-1) * (t - lo)) / (hi - lo);  bin = clamp(ceil(u), 0, T-1).
// Explicit _rn intrinsics keep nvcc from contracting or reassociating (reading A1).
__device__ __forceinline__ int alpha64(double t, const GridParams& g) {
  if (g.degenerate) return 0;
  double u = __ddiv_rn(__dmul_rn(g.Tm1, __dsub_rn(t, g.lo)), __dsub_rn(g.hi, g.lo));
  double c = ceil(u);
  if (c < 0.0) return 0;
  if (c > g.Tm1) return g.T - 1;
  return (int)c;
}

// Fast fp32 bin of an approximate height h32.  Returns -1 when h32's u lies within tau
// of an integer: the caller must then recompute the height exactly and use alpha64.
__device__ __forceinline__ int alpha32_or_repair(float h32, const GridParams& g) {
  float u = fmaf(h32, g.A, g.B);
  float r = rintf(u);
  if (!g.fp32_only && fabsf(u - r) < g.tau) return -1;
  int c = (int)ceilf(u);
  c = c < 0 ? 0 : c;
  c = c > g.T - 1 ? g.T - 1 : c;
  return c;
}

__device__ __forceinline__ void note_repair() {
  // warp-aggregated counter of repairs (reported, reading A1)
  unsigned m = __activemask();
  int leader = __ffs(m) - 1;
  if ((threadIdx.x & 31) == leader) atomicAdd(&g_repair_count, (unsigned long long)__popc(m));
}

__device__ __forceinline__ void atomic_max_u64(unsigned long long* p, unsigned long long v) {
  atomicMax(p, v);
}

// |x| of a non-negative double as monotone u64 bits
__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }

// Image embedding (reading A3): grid index g on an axis of length L ->
// (g - (L-1)/2) / S, S = max(max_dim - 1, 1), binary64 then one rounding to fp32.
__device__ __forceinline__ float axis_coord(int g, int L, double S) {
  double c = __ddiv_rn(__dsub_rn((double)g, __ddiv_rn((double)(L - 1), 2.0)), S);
  return __double2float_rn(c);
}

// ---- helpers of the shared-memory histogram kernels (k_complex.cu, k_cells.cu)
// Histogram flush into the global difference table (int64 / binary64); zeroes the rows.
template <bool FLOATW, typename Acc>
__device__ __forceinline__ void flush_hist(Acc* hist, int rows, int T, int TS, int row0, int Dc, void* diff) {
  for (int i = threadIdx.x; i < rows * T; i += blockDim.x) {
    const int r = i / T, q = i - r * T;
    const Acc val = hist[r * TS + q];
    if (val != (Acc)0 && row0 + r < Dc) {
      const int64_t o = (int64_t)(row0 + r) * T + q;
      if (FLOATW) atomicAdd((double*)diff + o, (double)val);
      else atomicAdd((unsigned long long*)diff + o, (unsigned long long)(long long)val);
    }
    hist[r * TS + q] = (Acc)0;
  }
}

// Signed weight (-1)^dim w of cell b of segment S, accumulator type.
template <bool FLOATW, typename Acc>
__device__ __forceinline__ Acc cell_weight(const Seg& S, int64_t b) {
  Acc w;
  if (FLOATW) w = S.weights ? __ldg((const float*)S.weights + b) : 1.f;
  else w = S.weights ? __ldg((const int*)S.weights + b) : 1;
  return S.sign < 0 ? -w : w;
}

__device__ __forceinline__ int64_t chunk_cells(bool floatw, int64_t float_chunk, const unsigned int* wmax_bits,
                                               int64_t span) {
  // int32 partials: chunk * max|w| < 2^31; float partials are flushed every float_chunk cells
  if (floatw) return float_chunk;
  const unsigned int wm = *wmax_bits;
  int64_t chunk = wm == 0 ? span : (int64_t)(2147483647u / wm);
  return chunk < 1 ? 1 : chunk;
}


inline static int64_t pick_slice(int64_t total, int tiles, int per_sm, int num_sms, int64_t cap) {
  int64_t want = ((int64_t)num_sms * per_sm * 2 + tiles - 1) / tiles;
  int64_t slice = (total + want - 1) / want;
  if (slice > cap) slice = cap;
  if (slice < 256) slice = 256;
  return slice;
}

}  // namespace wect

#define WECT_CUDA_TRY(expr)                                                    \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) return ::wect::fail_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)

namespace wect {
// instrumentation (api.cu): kernel launch counter and optional dominant-kernel events
void count_launch(int n = 1);
extern thread_local bool t_time_main;
struct MainTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  explicit MainTimer(cudaStream_t s);
  void stop();
};
wect_status fail_cuda(cudaError_t e, const char* what, const char* file, int line);
wect_status fail(wect_status s, const char* fmt, ...);

// Stream-ordered scratch: every block allocated through it is freed (cudaFreeAsync on the
// same stream) when the owner goes out of scope -- also on the early error returns of
// WECT_CUDA_TRY, so no path leaks pool memory.
struct AsyncScratch {
  cudaStream_t st;
  void* p[8] = {};
  int n = 0;
  explicit AsyncScratch(cudaStream_t s) : st(s) {}
  AsyncScratch(const AsyncScratch&) = delete;
  AsyncScratch& operator=(const AsyncScratch&) = delete;
  ~AsyncScratch() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], st);
  }
  template <typename Tp>
  cudaError_t alloc(Tp** out, size_t bytes) {
    *out = nullptr;
    if (n == 8) return cudaErrorMemoryAllocation;
    void* q = nullptr;
    const cudaError_t e = cudaMallocAsync(&q, bytes ? bytes : 16, st);
    if (e != cudaSuccess) return e;
    p[n++] = q;
    *out = (Tp*)q;
    return cudaSuccess;
  }
};
}  // namespace wect
