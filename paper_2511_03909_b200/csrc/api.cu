// api.cu -- the C ABI of libwect.so (include/wect.h): argument validation, host/device
// pointer staging, scratch, kernel selection.  Every step of the computation runs in
// the kernels of k_images.cu / k_complex.cu; there is no CPU fallback.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace wect {

// ---------------------------------------------------------------- errors
static thread_local char g_msg[512] = "";

wect_status fail(wect_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return s;
}

wect_status fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
  snprintf(g_msg, sizeof(g_msg), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e),
           what, file, line);
  return e == cudaErrorMemoryAllocation ? WECT_ENOMEM : WECT_ECUDA;
}

// --------------------------------------------------------- instrumentation
static std::atomic<uint64_t> g_launches{0};
thread_local bool t_time_main = false;
static std::mutex g_tmu;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timed;

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

MainTimer::MainTimer(cudaStream_t s) : st(s) {
  if (!t_time_main) return;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) { a = b = nullptr; return; }
  cudaEventRecord(a, st);
}
void MainTimer::stop() {
  if (!a) return;
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timed.emplace_back(a, b);
  a = b = nullptr;
}

// RAII: instrumentation flag for the duration of one API call
struct TimeScope {
  explicit TimeScope(uint32_t flags) { t_time_main = (flags & WECT_TIME_MAIN) != 0; }
  ~TimeScope() { t_time_main = false; }
};

// ------------------------------------------------------------- launchers
wect_status launch_grid_params(int ndim, const int64_t* dims, const float* dirs, int D, const wect_grid& grid,
                               GridParams* gp, cudaStream_t st);
bool sweep2d_supported(int ndim, const int64_t* dims, int T);
bool mma2d_supported(int ndim, const int64_t* dims, int T);
size_t mma2d_scratch_bytes(int HW, int Dc, int T);
wect_status launch_mma2d(const uint8_t* img, int64_t B, int H, int W, const float* dirs, int d_begin, int Dc, int T,
                         const GridParams* gp, void* scratch, void* out, wect_dtype odtype, cudaStream_t st,
                         int num_sms);
bool mma2_usable(void* out, int64_t B, int Dc, int T, wect_dtype odtype);
size_t mma2_scratch_bytes(int HW, int Dc, int T, int64_t B);
wect_status launch_mma2(const uint8_t* img, int64_t B, int H, int W, const float* dirs, int d_begin, int Dc, int T,
                        const GridParams* gp, void* scratch, void* out, cudaStream_t st, int num_sms);
wect_status launch_sweep2d(const uint8_t* img, int64_t B, int H, int W, const float* dirs, int d_begin, int Dc, int T,
                           const GridParams* gp, void* scratch, void* out, wect_dtype odtype, cudaStream_t st,
                           int num_sms, int freud);
size_t sweep2d_scratch_bytes(int HW, int Dc, int T, int freud, int64_t B, int num_sms);
bool grid_hist_fused(int ndim, const int64_t* dims, const uint8_t* img);
wect_status launch_grid_hist(const uint8_t* img, int64_t b0, int64_t nb, int ndim, const int64_t* dims,
                             const float* dirs, int d_begin, int Dc, int T, const GridParams* gp, int16_t* cwo, int* perm,
                             unsigned long long* diff, cudaStream_t st, int num_sms);
wect_status launch_vmax(int n, const float* coords, int64_t k0, const float* dirs, int D, float* vmax,
                        unsigned int* m32, unsigned int* r1, unsigned int* smax, unsigned long long* m64,
                        cudaStream_t st, int num_sms);
wect_status launch_complex_params(int mode, int n, const unsigned long long* m64, const unsigned int* m32,
                                  const unsigned int* r1, const unsigned int* smax, const wect_grid& grid,
                                  GridParams* gp, cudaStream_t st);
wect_status launch_absmax_f32(const float* f, int64_t n, unsigned int* bits, cudaStream_t st, int num_sms);
wect_status launch_absmax_i32(const int32_t* w, int64_t n, unsigned int* out, cudaStream_t st, int num_sms);
wect_status launch_check_indices(const int32_t* v, int64_t n, int64_t k0, unsigned int* flag, cudaStream_t st,
                                 int num_sms);
size_t ecf_images_scratch_bytes(int64_t B, int64_t nv, int T, bool per_image_M);
wect_status launch_ecf_images(const uint8_t* img, int64_t B, int ndim, const int64_t* dims, int T, int mode,
                              double lo, double hi, void* scratch, void* out, wect_dtype odtype, cudaStream_t st,
                              int num_sms);
wect_status launch_complex_grad(int mode, int n, const Segs& segs, const float* coords, int64_t k0, const float* fsrc,
                                int m_or_D, int d_begin, int Dc, int T, const GridParams* gp, const double* G,
                                const GradOut& gout, cudaStream_t st, int num_sms);
size_t freud_scratch_per_image(int H, int W);
wect_status launch_freud(const uint8_t* img, int64_t b0, int64_t nb, int H, int W, const float* dirs, int d_begin,
                         int Dc, int T, const GridParams* gp, int16_t* w6, unsigned long long* diff, cudaStream_t st,
                         int num_sms);
wect_status launch_finalize(const void* diff, bool is_float, int64_t rows, int T, void* out, wect_dtype odtype,
                            cudaStream_t st);

wect_status launch_complex(int mode, int n, bool floatw, const Segs& segs, const float* coords, int64_t k0,
                           const float* fsrc, int m_or_D, int d_begin, int Dc, int T, const GridParams* gp,
                           const unsigned int* wmax, void* diff, cudaStream_t st, int num_sms);

// --------------------------------------------------------------- helpers
static int num_sms_current() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
    // keep stream-ordered scratch cached across calls: with the default release threshold
    // (0) every synchronisation hands the pool back and the next call pays cudaMalloc
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  return cache[dev];
}

static bool is_device_ptr(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Stream-ordered scratch and host staging; everything is released stream-ordered.
struct Arena {
  cudaStream_t st;
  std::vector<void*> blocks;
  cudaError_t err = cudaSuccess;
  bool staged = false;  // some input was host memory: the call syncs before returning
  explicit Arena(cudaStream_t s) : st(s) {}
  ~Arena() {
    for (void* b : blocks) cudaFreeAsync(b, st);
  }
  void* alloc(size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, st);
    if (e != cudaSuccess) { err = e; return nullptr; }
    blocks.push_back(p);
    return p;
  }
  // device view of a caller array (copied in if it lives on the host)
  const void* in(const void* p, size_t bytes) {
    if (!p || is_device_ptr(p)) return p;
    void* d = alloc(bytes);
    if (!d) return nullptr;
    cudaError_t e = cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { err = e; return nullptr; }
    staged = true;
    return d;
  }
};

static size_t dtype_size(wect_dtype t) {
  switch (t) {
    case WECT_U8: return 1;
    case WECT_I32: return 4;
    case WECT_F32: return 4;
    case WECT_I64: return 8;
    case WECT_F64: return 8;
  }
  return 0;
}

static wect_status resolve_rows(const wect_grid* g, int D, int* d_begin, int* d_count) {
  if (g->d_begin < 0 || g->d_count < 0) return fail(WECT_EINVAL, "d_begin/d_count must be >= 0");
  int c = g->d_count == 0 ? D - g->d_begin : g->d_count;
  if (g->d_begin > D || c < 0 || (int64_t)g->d_begin + c > D)
    return fail(WECT_EINVAL, "rows [%d, %d) outside [0, %d)", g->d_begin, g->d_begin + c, D);
  *d_begin = g->d_begin;
  *d_count = c;
  return WECT_OK;
}

// output: device pointer to write, plus D2H copy on completion if the caller's is host
struct OutView {
  void* user;
  void* dev;
  size_t bytes;
};
static OutView out_view(Arena& ar, void* user, size_t bytes) {
  OutView o{user, user, bytes};
  if (user && !is_device_ptr(user)) o.dev = ar.alloc(bytes);
  return o;
}
// Host outputs are copied back; if any input or output was host memory the stream is
// synchronised, so the caller may reuse (or read) its host buffers when the call returns
// (a pinned input would otherwise still be read by an in-flight DMA).
static wect_status out_finish(const OutView& o, Arena& ar) {
  if (o.dev != o.user) WECT_CUDA_TRY(cudaMemcpyAsync(o.user, o.dev, o.bytes, cudaMemcpyDeviceToHost, ar.st));
  if (o.dev != o.user || ar.staged) WECT_CUDA_TRY(cudaStreamSynchronize(ar.st));
  return WECT_OK;
}

}  // namespace wect

using namespace wect;

extern "C" {

int32_t wect_abi_version(void) { return WECT_ABI_VERSION; }

wect_status wect_stats(uint64_t* launches, uint64_t* timed_launches, double* timed_ms, int reset) {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  {
    std::lock_guard<std::mutex> lk(g_tmu);
    ev.swap(g_timed);
  }
  double ms = 0.0;
  for (auto& e : ev) {
    float t = 0.f;
    WECT_CUDA_TRY(cudaEventSynchronize(e.second));
    WECT_CUDA_TRY(cudaEventElapsedTime(&t, e.first, e.second));
    ms += t;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  static double acc_ms = 0.0;
  static uint64_t acc_n = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  acc_ms += ms;
  acc_n += ev.size();
  if (launches) *launches = g_launches.load();
  if (timed_launches) *timed_launches = acc_n;
  if (timed_ms) *timed_ms = acc_ms;
  if (reset) {
    acc_ms = 0.0;
    acc_n = 0;
    g_launches.store(0);
  }
  return WECT_OK;
}

const char* wect_last_error(void) { return g_msg; }

wect_status wect_sync_status(void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  WECT_CUDA_TRY(cudaStreamSynchronize(st));
  unsigned int w = 0, zero = 0;
  WECT_CUDA_TRY(cudaMemcpyFromSymbol(&w, g_err_word, sizeof(w)));
  if (w) {
    WECT_CUDA_TRY(cudaMemcpyToSymbol(g_err_word, &zero, sizeof(zero)));
    return fail(WECT_ERANGE, "a vertex index outside [0, k0) was found; affected cells were skipped");
  }
  return WECT_OK;
}

wect_status wect_repair_count(uint64_t* count_host, int reset) {
  if (!count_host) return fail(WECT_EINVAL, "count_host is NULL");
  WECT_CUDA_TRY(cudaDeviceSynchronize());
  unsigned long long c = 0, zero = 0;
  WECT_CUDA_TRY(cudaMemcpyFromSymbol(&c, g_repair_count, sizeof(c)));
  if (reset) WECT_CUDA_TRY(cudaMemcpyToSymbol(g_repair_count, &zero, sizeof(zero)));
  *count_host = c;
  return WECT_OK;
}

// ------------------------------------------------------------------ images
wect_status wect_images(const uint8_t* img, int64_t B, int32_t ndim, const int64_t* dims, const float* dirs, int32_t D,
                        const wect_grid* grid, void* out, wect_dtype odtype, void* stream) {
  g_msg[0] = 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (!grid) return fail(WECT_EINVAL, "grid is NULL");
  TimeScope ts(grid->flags);
  if (ndim != 2 && ndim != 3) return fail(WECT_EINVAL, "ndim must be 2 or 3 (got %d)", ndim);
  if (!dims) return fail(WECT_EINVAL, "dims is NULL");
  if (B < 0) return fail(WECT_EINVAL, "B < 0");
  if (D < 1 || !dirs) return fail(WECT_EINVAL, "need D >= 1 directions");
  if (grid->T < 2) return fail(WECT_EINVAL, "T must be >= 2 (beta divides by T-1)");
  int64_t nv = 1, ncells = 1;
  for (int i = 0; i < ndim; ++i) {
    if (dims[i] < 1) return fail(WECT_EINVAL, "dims[%d] = %lld < 1", i, (long long)dims[i]);
    if (dims[i] > 1024) return fail(WECT_ENOTSUP, "image side %lld > 1024 not supported", (long long)dims[i]);
    nv *= dims[i];
    ncells *= 2 * dims[i] - 1;
  }
  const bool freud = (grid->flags & WECT_FREUDENTHAL) != 0;
  if (freud) {
    if (ndim != 2) return fail(WECT_ENOTSUP, "WECT_FREUDENTHAL needs 2-D images");
    // V + E + F of the Freudenthal complex: HW + [H(W-1) + W(H-1) + (H-1)(W-1)] + 2(H-1)(W-1)
    const int64_t H = dims[0], W = dims[1];
    ncells = H * W + H * (W - 1) + W * (H - 1) + 3 * (H - 1) * (W - 1);
  }
  int d_begin, Dc;
  wect_status rs = resolve_rows(grid, D, &d_begin, &Dc);
  if (rs != WECT_OK) return rs;
  if (odtype != WECT_I32 && odtype != WECT_I64) return fail(WECT_EINVAL, "image WECT output must be I32 or I64");
  if (odtype == WECT_I32 && 255.0 * (double)ncells >= 2147483648.0)
    return fail(WECT_EOVERFLOW, "int32 output cannot bound 255 * %lld cells", (long long)ncells);
  if (B > 0 && Dc > 0 && (!img || !out)) return fail(WECT_EINVAL, "img/out is NULL");
  const bool sweep = sweep2d_supported(ndim, dims, grid->T) && !(freud && getenv("WECT_FREUD_HIST"));
  if (!sweep && grid->T > 1024) return fail(WECT_ENOTSUP, "T > 1024 needs the sweep path (2D cubical, H*W <= 1024)");
  if (B == 0 || Dc == 0) return WECT_OK;
  // the tensor-core contraction (k_mma.cu, cubical 2-D): WECT_IMAGES_MMA=1 selects it
  const char* mma_env = getenv("WECT_IMAGES_MMA");
  // (its indicator operand grows with the number of directions: at most 1 GiB of scratch)
  const bool mma = !freud && mma_env && (mma_env[0] == '1' || mma_env[0] == '2') &&
                   mma2d_supported(ndim, dims, grid->T) && mma2d_scratch_bytes((int)nv, Dc, grid->T) <= ((size_t)1 << 30);
  const bool mma2 = mma && mma_env[0] == '2';

  const int nsm = num_sms_current();
  Arena ar(st);
  const uint8_t* dimg = (const uint8_t*)ar.in(img, (size_t)B * nv);
  const float* ddirs = (const float*)ar.in(dirs, (size_t)D * ndim * sizeof(float));
  const size_t obytes = (size_t)B * Dc * grid->T * dtype_size(odtype);
  OutView ov = out_view(ar, out, obytes);
  GridParams* gp = (GridParams*)ar.alloc(sizeof(GridParams));
  if (ar.err != cudaSuccess) return fail_cuda(ar.err, "staging", __FILE__, __LINE__);
  wect_status s = launch_grid_params(ndim, dims, ddirs, D, *grid, gp, st);
  if (s != WECT_OK) return s;
  if (freud && !sweep) {
    const size_t nbins = (size_t)B * Dc * grid->T;
    unsigned long long* diff = (unsigned long long*)ar.alloc(nbins * 8);
    const int64_t per_img = (int64_t)freud_scratch_per_image((int)dims[0], (int)dims[1]);
    int64_t chunk = ((int64_t)1 << 30) / per_img;
    chunk = chunk < 1 ? 1 : (chunk > 65535 ? 65535 : chunk);
    if (chunk > B) chunk = B;
    int16_t* w6 = (int16_t*)ar.alloc((size_t)chunk * per_img);
    if (ar.err != cudaSuccess) return fail_cuda(ar.err, "scratch", __FILE__, __LINE__);
    WECT_CUDA_TRY(cudaMemsetAsync(diff, 0, nbins * 8, st));
    for (int64_t b0 = 0; b0 < B && s == WECT_OK; b0 += chunk) {
      const int64_t nb = B - b0 < chunk ? B - b0 : chunk;
      s = launch_freud(dimg, b0, nb, (int)dims[0], (int)dims[1], ddirs, d_begin, Dc, grid->T, gp, w6, diff, st, nsm);
    }
    if (s == WECT_OK) s = launch_finalize(diff, false, (int64_t)B * Dc, grid->T, ov.dev, odtype, st);
  } else if (mma2 && mma2_usable(ov.dev, B, Dc, grid->T, odtype) &&
             mma2_scratch_bytes((int)nv, Dc, grid->T, B) <= ((size_t)3 << 30)) {
    // WECT_IMAGES_MMA=2: the second contraction kernel (MN-major A from transposed pixels,
    // TMA-store epilogue); =1: the first (faster of the two)
    void* scr = ar.alloc(mma2_scratch_bytes((int)nv, Dc, grid->T, B));
    if (ar.err != cudaSuccess) return fail_cuda(ar.err, "scratch", __FILE__, __LINE__);
    s = launch_mma2(dimg, B, (int)dims[0], (int)dims[1], ddirs, d_begin, Dc, grid->T, gp, scr, ov.dev, st, nsm);
  } else if (mma) {
    void* scr = ar.alloc(mma2d_scratch_bytes((int)nv, Dc, grid->T));
    if (ar.err != cudaSuccess) return fail_cuda(ar.err, "scratch", __FILE__, __LINE__);
    s = launch_mma2d(dimg, B, (int)dims[0], (int)dims[1], ddirs, d_begin, Dc, grid->T, gp, scr, ov.dev, odtype, st, nsm);
  } else if (sweep) {
    void* scr = ar.alloc(sweep2d_scratch_bytes((int)nv, Dc, grid->T, freud ? 1 : 0, B, nsm));
    if (ar.err != cudaSuccess) return fail_cuda(ar.err, "scratch", __FILE__, __LINE__);
    s = launch_sweep2d(dimg, B, (int)dims[0], (int)dims[1], ddirs, d_begin, Dc, grid->T, gp, scr, ov.dev, odtype, st,
                       nsm, freud ? 1 : 0);
  } else {
    const size_t nbins = (size_t)B * Dc * grid->T;
    unsigned long long* diff = (unsigned long long*)ar.alloc(nbins * 8);
    // orthant weights for a chunk of images: at most ~1 GiB of scratch (none when fused)
    const bool fused = grid_hist_fused(ndim, dims, dimg);
    const int64_t per_img = nv * (1 << ndim) * 2;
    int64_t chunk = fused ? B : ((int64_t)1 << 30) / per_img;
    if (chunk < 1) chunk = 1;
    if (chunk > 65535) chunk = 65535;  // k_grid_hist takes the image from gridDim.z
    if (chunk > B) chunk = B;
    int16_t* cwo = fused ? nullptr : (int16_t*)ar.alloc((size_t)chunk * per_img);
    int* perm = (int*)ar.alloc((size_t)Dc * sizeof(int));
    if (ar.err != cudaSuccess) return fail_cuda(ar.err, "scratch", __FILE__, __LINE__);
    WECT_CUDA_TRY(cudaMemsetAsync(diff, 0, nbins * 8, st));
    for (int64_t b0 = 0; b0 < B && s == WECT_OK; b0 += chunk) {
      int64_t nb = B - b0 < chunk ? B - b0 : chunk;
      s = launch_grid_hist(dimg, b0, nb, ndim, dims, ddirs, d_begin, Dc, grid->T, gp, cwo, perm, diff, st, nsm);
    }
    if (s == WECT_OK) s = launch_finalize(diff, false, (int64_t)B * Dc, grid->T, ov.dev, odtype, st);
  }
  if (s != WECT_OK) return s;
  return out_finish(ov, ar);
}

// -------------------------------------------------------------- image ECF
wect_status ecf_images(const uint8_t* img, int64_t B, int32_t ndim, const int64_t* dims, const wect_grid* grid,
                       void* out, wect_dtype odtype, void* stream) {
  g_msg[0] = 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (!grid) return fail(WECT_EINVAL, "grid is NULL");
  TimeScope ts(grid->flags);
  if (ndim != 2 && ndim != 3) return fail(WECT_EINVAL, "ndim must be 2 or 3 (got %d)", ndim);
  if (!dims) return fail(WECT_EINVAL, "dims is NULL");
  if (B < 0) return fail(WECT_EINVAL, "B < 0");
  if (grid->T < 2) return fail(WECT_EINVAL, "T must be >= 2 (beta divides by T-1)");
  if (grid->T > 65536) return fail(WECT_ENOTSUP, "T > 65536");
  if (grid->d_begin != 0 || (grid->d_count != 0 && grid->d_count != 1))
    return fail(WECT_EINVAL, "ecf_images has one filter per image: d_begin must be 0, d_count 0 or 1");
  int64_t nv = 1, ncells = 1;
  for (int i = 0; i < ndim; ++i) {
    if (dims[i] < 1) return fail(WECT_EINVAL, "dims[%d] = %lld < 1", i, (long long)dims[i]);
    if (dims[i] > 65535) return fail(WECT_ENOTSUP, "image side %lld > 65535", (long long)dims[i]);
    nv *= dims[i];
    ncells *= 2 * dims[i] - 1;
  }
  if (nv > ((int64_t)1 << 34)) return fail(WECT_ENOTSUP, "image of %lld vertices", (long long)nv);
  if (odtype != WECT_I32 && odtype != WECT_I64) return fail(WECT_EINVAL, "image ECF output must be I32 or I64");
  if (odtype == WECT_I32 && (double)ncells >= 2147483648.0)
    return fail(WECT_EOVERFLOW, "int32 output cannot bound %lld cells", (long long)ncells);
  if (B > 0 && (!img || !out)) return fail(WECT_EINVAL, "img/out is NULL");
  if (B == 0) return WECT_OK;
  if (B > 65535 && nv > 4096) return fail(WECT_ENOTSUP, "more than 65535 large images per call");
  int mode = 0;
  double lo = 0.0, hi = 0.0;
  if (grid->lo < grid->hi) { mode = 1; lo = grid->lo; hi = grid->hi; }
  else if (grid->maxheight > 0) { mode = 1; lo = -grid->maxheight; hi = grid->maxheight; }
  const int nsm = num_sms_current();
  Arena ar(st);
  const uint8_t* dimg = (const uint8_t*)ar.in(img, (size_t)B * nv);
  OutView ov = out_view(ar, out, (size_t)B * grid->T * dtype_size(odtype));
  void* scr = ar.alloc(ecf_images_scratch_bytes(B, nv, grid->T, mode == 0));
  if (ar.err != cudaSuccess) return fail_cuda(ar.err, "staging", __FILE__, __LINE__);
  wect_status s = launch_ecf_images(dimg, B, ndim, dims, grid->T, mode, lo, hi, scr, ov.dev, odtype, st, nsm);
  if (s != WECT_OK) return s;
  return out_finish(ov, ar);
}

// ----------------------------------------------------- explicit complexes
static wect_status validate_complex(const wect_complex_desc* K, bool need_coords) {
  if (!K) return fail(WECT_EINVAL, "complex descriptor is NULL");
  if (K->k0 < 0) return fail(WECT_EINVAL, "k0 < 0");
  if (K->k0 > 2147483647LL) return fail(WECT_ENOTSUP, "k0 >= 2^31");
  if (need_coords && (K->n < 1 || K->n > kMaxDims)) return fail(WECT_EINVAL, "n=%d outside [1, %d]", K->n, kMaxDims);
  if (need_coords && K->k0 > 0 && !K->coords) return fail(WECT_EINVAL, "coords is NULL");
  if (K->wdtype != WECT_I32 && K->wdtype != WECT_F32) return fail(WECT_EINVAL, "wdtype must be WECT_I32 or WECT_F32");
  if (K->ncell_dims < 0 || K->ncell_dims > kMaxSegs - 1)
    return fail(WECT_EINVAL, "ncell_dims=%d outside [0, %d]", K->ncell_dims, kMaxSegs - 1);
  if (K->ncell_dims > 0 && !K->cells) return fail(WECT_EINVAL, "cells is NULL");
  for (int i = 0; i < K->ncell_dims; ++i) {
    const wect_cells& c = K->cells[i];
    if (c.count < 0) return fail(WECT_EINVAL, "cells[%d].count < 0", i);
    if (c.arity < 1 || c.arity > 32) return fail(WECT_EINVAL, "cells[%d].arity=%d outside [1, 32]", i, c.arity);
    if (c.dim < 1) return fail(WECT_EINVAL, "cells[%d].dim=%d < 1", i, c.dim);
    if (c.count > 0 && !c.verts) return fail(WECT_EINVAL, "cells[%d].verts is NULL", i);
  }
  return WECT_OK;
}

// mode 0: WECT over coords x dirs; mode 1: ECF over fvals [k0, m]
static wect_status run_complex(int mode, const wect_complex_desc* K, const float* fsrc, int32_t D,
                               const wect_grid* grid, void* out, wect_dtype odtype, void* stream) {
  g_msg[0] = 0;
  cudaStream_t st = (cudaStream_t)stream;
  wect_status s = validate_complex(K, mode == 0);
  if (s != WECT_OK) return s;
  if (!grid) return fail(WECT_EINVAL, "grid is NULL");
  TimeScope ts(grid->flags);
  if (grid->T < 2) return fail(WECT_EINVAL, "T must be >= 2 (beta divides by T-1)");
  if (grid->T > 4096) return fail(WECT_ENOTSUP, "T > 4096 not supported");
  if (D < 1) return fail(WECT_EINVAL, mode == 0 ? "need D >= 1 directions" : "need m >= 1 filters");
  if (!fsrc && K->k0 > 0) return fail(WECT_EINVAL, mode == 0 ? "dirs is NULL" : "fvals is NULL");
  if (mode == 0 && !fsrc) return fail(WECT_EINVAL, "dirs is NULL");
  const bool floatw = K->wdtype == WECT_F32;
  if (floatw && odtype != WECT_F64) return fail(WECT_EINVAL, "float weights need WECT_F64 output");
  if (!floatw && odtype == WECT_I32) return fail(WECT_EOVERFLOW, "int32 output cannot be bounded for explicit complexes");
  if (!floatw && odtype != WECT_I64) return fail(WECT_EINVAL, "integer weights need WECT_I64 output");
  int d_begin, Dc;
  s = resolve_rows(grid, D, &d_begin, &Dc);
  if (s != WECT_OK) return s;
  if (Dc == 0) return WECT_OK;
  if (!out) return fail(WECT_EINVAL, "out is NULL");
  const int T = grid->T;
  const int n = K->n;
  const int nsm = num_sms_current();
  Arena ar(st);
  const size_t obytes = (size_t)Dc * T * 8;
  OutView ov = out_view(ar, out, obytes);
  if (ar.err != cudaSuccess) return fail_cuda(ar.err, "staging", __FILE__, __LINE__);
  if (K->k0 == 0) {  // empty complex: every WECF is 0
    WECT_CUDA_TRY(cudaMemsetAsync(ov.dev, 0, obytes, st));
    return out_finish(ov, ar);
  }
  const size_t wsz = 4;
  Segs segs;
  memset(&segs, 0, sizeof(segs));
  segs.s[0].verts = nullptr;
  segs.s[0].weights = ar.in(K->vweights, (size_t)K->k0 * wsz);
  segs.s[0].count = K->k0;
  segs.s[0].start = 0;
  segs.s[0].arity = 1;
  segs.s[0].sign = 1;
  int ns = 1;
  int64_t total = K->k0;
  for (int i = 0; i < K->ncell_dims; ++i) {
    const wect_cells& c = K->cells[i];
    if (c.count == 0) continue;
    Seg& g = segs.s[ns++];
    g.verts = (const int32_t*)ar.in(c.verts, (size_t)c.count * c.arity * 4);
    g.weights = ar.in(c.weights, (size_t)c.count * wsz);
    g.count = c.count;
    g.start = total;
    g.arity = c.arity;
    g.sign = (c.dim % 2 == 0) ? 1 : -1;
    total += c.count;
  }
  // sentinel so the segment search always terminates
  for (int i = ns; i < kMaxSegs; ++i) { segs.s[i].start = total; segs.s[i].count = (int64_t)1 << 62; }
  segs.nseg = ns;
  segs.total = total;
  const float* coords = mode == 0 ? (const float*)ar.in(K->coords, (size_t)K->k0 * n * 4) : nullptr;
  const float* dsrc = mode == 0 ? (const float*)ar.in(fsrc, (size_t)D * n * 4)
                                : (const float*)ar.in(fsrc, (size_t)K->k0 * D * 4);
  // device words: [0] m64 (u64), [1] m32, r1, smax, wmax, badidx
  unsigned long long* words = (unsigned long long*)ar.alloc(64);
  GridParams* gp = (GridParams*)ar.alloc(sizeof(GridParams));
  void* diff = ar.alloc((size_t)Dc * T * 8);
  if (ar.err != cudaSuccess) return fail_cuda(ar.err, "staging/scratch", __FILE__, __LINE__);
  unsigned long long* m64 = words;
  unsigned int* w32 = (unsigned int*)(words + 1);
  unsigned int *m32 = w32, *r1 = w32 + 1, *smax = w32 + 2, *wmax = w32 + 3, *badidx = w32 + 4;
  WECT_CUDA_TRY(cudaMemsetAsync(words, 0, 64, st));
  WECT_CUDA_TRY(cudaMemsetAsync(diff, 0, (size_t)Dc * T * 8, st));

  if (grid->flags & WECT_VALIDATE) {
    for (int i = 1; i < ns; ++i) {
      s = launch_check_indices(segs.s[i].verts, segs.s[i].count * segs.s[i].arity, K->k0, badidx, st, nsm);
      if (s != WECT_OK) return s;
    }
    unsigned int bad = 0;
    WECT_CUDA_TRY(cudaMemcpyAsync(&bad, badidx, 4, cudaMemcpyDeviceToHost, st));
    WECT_CUDA_TRY(cudaStreamSynchronize(st));
    if (bad) return fail(WECT_ERANGE, "a vertex index outside [0, %lld) (WECT_VALIDATE); nothing written", (long long)K->k0);
  }
  if (mode == 0) {
    float* vmax = (float*)ar.alloc((size_t)K->k0 * 4);
    if (ar.err != cudaSuccess) return fail_cuda(ar.err, "scratch", __FILE__, __LINE__);
    s = launch_vmax(n, coords, K->k0, dsrc, D, vmax, m32, r1, smax, m64, st, nsm);
  } else {
    s = launch_absmax_f32(dsrc, K->k0 * (int64_t)D, m32, st, nsm);
  }
  if (s != WECT_OK) return s;
  s = launch_complex_params(mode, n, m64, m32, r1, smax, *grid, gp, st);
  if (s != WECT_OK) return s;
  // (max|w| of integer weights, where a kernel needs it, is computed inside launch_complex)
  s = launch_complex(mode, n, floatw, segs, coords, K->k0, dsrc, D, d_begin, Dc, T, gp, wmax, diff, st, nsm);
  if (s != WECT_OK) return s;
  s = launch_finalize(diff, floatw, Dc, T, ov.dev, odtype, st);
  if (s != WECT_OK) return s;
  return out_finish(ov, ar);
}

// ------------------------------------------------ backward (weights gradient)

static wect_status run_complex_grad(int mode, const wect_complex_desc* K, const float* fsrc, int32_t D,
                                    const wect_grid* grid, const double* G, double* grad_vweights,
                                    double* const* grad_cells, void* stream) {
  g_msg[0] = 0;
  cudaStream_t st = (cudaStream_t)stream;
  wect_status s = validate_complex(K, mode == 0);
  if (s != WECT_OK) return s;
  if (!grid) return fail(WECT_EINVAL, "grid is NULL");
  TimeScope ts(grid->flags);
  if (grid->T < 2) return fail(WECT_EINVAL, "T must be >= 2 (beta divides by T-1)");
  if (grid->T > 4096) return fail(WECT_ENOTSUP, "T > 4096 not supported");
  if (D < 1) return fail(WECT_EINVAL, mode == 0 ? "need D >= 1 directions" : "need m >= 1 filters");
  if (!fsrc && K->k0 > 0) return fail(WECT_EINVAL, mode == 0 ? "dirs is NULL" : "fvals is NULL");
  int d_begin, Dc;
  s = resolve_rows(grid, D, &d_begin, &Dc);
  if (s != WECT_OK) return s;
  if (!G && Dc > 0 && K->k0 > 0) return fail(WECT_EINVAL, "G is NULL");
  const int T = grid->T;
  const int n = K->n;
  const int nsm = num_sms_current();
  Arena ar(st);
  // outputs (device views; host outputs are copied back at the end)
  GradOut gout;
  memset(&gout, 0, sizeof(gout));
  std::vector<OutView> views;
  Segs segs;
  memset(&segs, 0, sizeof(segs));
  segs.s[0].count = K->k0;
  segs.s[0].arity = 1;
  segs.s[0].sign = 1;
  if (grad_vweights) {
    views.push_back(out_view(ar, grad_vweights, (size_t)K->k0 * 8));
    gout.g[0] = (double*)views.back().dev;
  }
  int ns = 1;
  int64_t total = K->k0;
  for (int i = 0; i < K->ncell_dims; ++i) {
    const wect_cells& c = K->cells[i];
    if (c.count == 0) continue;
    Seg& g = segs.s[ns];
    g.verts = (const int32_t*)ar.in(c.verts, (size_t)c.count * c.arity * 4);
    g.count = c.count;
    g.start = total;
    g.arity = c.arity;
    g.sign = (c.dim % 2 == 0) ? 1 : -1;
    total += c.count;
    if (grad_cells && grad_cells[i]) {
      views.push_back(out_view(ar, grad_cells[i], (size_t)c.count * 8));
      gout.g[ns] = (double*)views.back().dev;
    }
    ++ns;
  }
  for (int i = ns; i < kMaxSegs; ++i) { segs.s[i].start = total; segs.s[i].count = (int64_t)1 << 62; }
  segs.nseg = ns;
  segs.total = total;
  if (ar.err != cudaSuccess) return fail_cuda(ar.err, "staging", __FILE__, __LINE__);
  if (K->k0 == 0) return WECT_OK;
  if (Dc == 0) {  // no rows: the gradient is 0
    for (auto& v : views) WECT_CUDA_TRY(cudaMemsetAsync(v.dev, 0, v.bytes, st));
    for (auto& v : views) { s = out_finish(v, ar); if (s != WECT_OK) return s; }
    return WECT_OK;
  }
  const float* coords = mode == 0 ? (const float*)ar.in(K->coords, (size_t)K->k0 * n * 4) : nullptr;
  const float* dsrc = mode == 0 ? (const float*)ar.in(fsrc, (size_t)D * n * 4)
                                : (const float*)ar.in(fsrc, (size_t)K->k0 * D * 4);
  const double* dG = (const double*)ar.in(G, (size_t)Dc * T * 8);
  unsigned long long* words = (unsigned long long*)ar.alloc(64);
  GridParams* gp = (GridParams*)ar.alloc(sizeof(GridParams));
  if (ar.err != cudaSuccess) return fail_cuda(ar.err, "staging/scratch", __FILE__, __LINE__);
  unsigned long long* m64 = words;
  unsigned int* w32 = (unsigned int*)(words + 1);
  unsigned int *m32 = w32, *r1 = w32 + 1, *smax = w32 + 2;
  WECT_CUDA_TRY(cudaMemsetAsync(words, 0, 64, st));
  if (mode == 0) {
    float* vmax = (float*)ar.alloc((size_t)K->k0 * 4);
    if (ar.err != cudaSuccess) return fail_cuda(ar.err, "scratch", __FILE__, __LINE__);
    s = launch_vmax(n, coords, K->k0, dsrc, D, vmax, m32, r1, smax, m64, st, nsm);
  } else {
    s = launch_absmax_f32(dsrc, K->k0 * (int64_t)D, m32, st, nsm);
  }
  if (s != WECT_OK) return s;
  s = launch_complex_params(mode, n, m64, m32, r1, smax, *grid, gp, st);
  if (s != WECT_OK) return s;
  s = launch_complex_grad(mode, n, segs, coords, K->k0, dsrc, D, d_begin, Dc, T, gp, dG, gout, st, nsm);
  if (s != WECT_OK) return s;
  for (auto& v : views) {
    s = out_finish(v, ar);
    if (s != WECT_OK) return s;
  }
  return WECT_OK;
}

wect_status wect_complex_backward(const wect_complex_desc* K, const float* dirs, int32_t D, const wect_grid* grid,
                                  const double* G, double* grad_vweights, double* const* grad_cells, void* stream) {
  return run_complex_grad(0, K, dirs, D, grid, G, grad_vweights, grad_cells, stream);
}

wect_status ecf_complex_backward(const wect_complex_desc* K, const float* fvals, int32_t m, const wect_grid* grid,
                                 const double* G, double* grad_vweights, double* const* grad_cells, void* stream) {
  return run_complex_grad(1, K, fvals, m, grid, G, grad_vweights, grad_cells, stream);
}

wect_status wect_complex(const wect_complex_desc* K, const float* dirs, int32_t D, const wect_grid* grid, void* out,
                         wect_dtype odtype, void* stream) {
  return run_complex(0, K, dirs, D, grid, out, odtype, stream);
}

wect_status ecf_complex(const wect_complex_desc* K, const float* fvals, int32_t m, const wect_grid* grid, void* out,
                        wect_dtype odtype, void* stream) {
  return run_complex(1, K, fvals, m, grid, out, odtype, stream);
}

wect_status wect_maxheight(const float* coords, int64_t k0, int32_t n, const float* dirs, int32_t D, double* M_host,
                           void* stream) {
  g_msg[0] = 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (!M_host) return fail(WECT_EINVAL, "M_host is NULL");
  if (n < 1 || n > kMaxDims) return fail(WECT_EINVAL, "n=%d outside [1, %d]", n, kMaxDims);
  if (k0 < 0 || D < 1 || !dirs || (k0 > 0 && !coords)) return fail(WECT_EINVAL, "bad coords/dirs");
  if (k0 == 0) { *M_host = 0.0; return WECT_OK; }
  const int nsm = num_sms_current();
  Arena ar(st);
  const float* dc = (const float*)ar.in(coords, (size_t)k0 * n * 4);
  const float* dd = (const float*)ar.in(dirs, (size_t)D * n * 4);
  unsigned long long* words = (unsigned long long*)ar.alloc(64);
  float* vmax = (float*)ar.alloc((size_t)k0 * 4);
  if (ar.err != cudaSuccess) return fail_cuda(ar.err, "staging/scratch", __FILE__, __LINE__);
  unsigned int* w32 = (unsigned int*)(words + 1);
  WECT_CUDA_TRY(cudaMemsetAsync(words, 0, 64, st));
  wect_status s = launch_vmax(n, dc, k0, dd, D, vmax, w32, w32 + 1, w32 + 2, words, st, nsm);
  if (s != WECT_OK) return s;
  unsigned long long bits = 0;
  WECT_CUDA_TRY(cudaMemcpyAsync(&bits, words, 8, cudaMemcpyDeviceToHost, st));
  WECT_CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(M_host, &bits, 8);
  return WECT_OK;
}

}  // extern "C"
