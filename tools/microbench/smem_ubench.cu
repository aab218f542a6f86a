// Microbenchmarks for the B200 resources the WECT kernels lean on:
// shared-memory atomics (conflict-free / random / same-address), shared loads
// of 32/64/128 bits, and a streaming HBM write. Results feed DESIGN.md's
// compute-roofline denominators (MEASURED_PEAKS.json has no smem-atomic peak).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

template <int MODE>
__global__ void __launch_bounds__(512) k_atoms(int* out, int T) {
  extern __shared__ int hist[];
  for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
  int base = warp * T;  // each warp its own row (like lanes=directions? no: warp row)
  #pragma unroll 8
  for (int it = 0; it < ITERS; ++it) {
    int addr;
    if (MODE == 0) addr = base + ((lane + it) & (T - 1));          // conflict-free
    else if (MODE == 1) { x = x * 1664525u + 1013904223u; addr = base + (x >> 20) % T; }  // random in row
    else if (MODE == 2) addr = base + (it & (T - 1));              // same address
    else { x = x * 1664525u + 1013904223u; addr = lane * (T + 1) + ((x >> 20) % T); } // lanes=rows, random bin
    atomicAdd(&hist[addr & (32 * 1024 - 1)], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = hist[0];
}

// RNG-only twin of MODE 1/3 for subtracting ALU cost
__global__ void __launch_bounds__(512) k_rng(int* out, int T) {
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x; int acc = 0;
  #pragma unroll 8
  for (int it = 0; it < ITERS; ++it) { x = x * 1664525u + 1013904223u; acc += (x >> 20) % T; }
  if (acc == 0x12345) out[0] = acc;
}

template <int VEC>
__global__ void __launch_bounds__(512) k_lds(int* out) {
  extern __shared__ int4 buf4[];
  int* buf = (int*)buf4;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) buf[i] = i;
  __syncthreads();
  int lane = threadIdx.x & 31;
  int acc = 0;
  #pragma unroll 8
  for (int it = 0; it < ITERS; ++it) {
    int row = (it * 7 + (threadIdx.x >> 5)) & 63;
    if (VEC == 1) acc += buf[row * 32 + lane];
    else if (VEC == 2) { int2 v = ((int2*)buf)[row * 32 + lane]; acc += v.x ^ v.y; }
    else { int4 v = buf4[(row & 31) * 32 + lane]; acc += v.x ^ v.y ^ v.z ^ v.w; }
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

__global__ void k_write(int4* p, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) __stcs(p + i, make_int4((int)i, 1, 2, 3));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d  L2 %d B  clock %d kHz\n", nsm, l2, clk);
  int* d; CK(cudaMalloc(&d, 1 << 20));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  const int threads = 512, blocksPerSM = 2;
  int grid = nsm * blocksPerSM;
  size_t smemA = 32 * 1024 * 4;  // 128 KB -> 1 block/SM actually
  CK(cudaFuncSetAttribute(k_atoms<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemA));
  CK(cudaFuncSetAttribute(k_atoms<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemA));
  CK(cudaFuncSetAttribute(k_atoms<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemA));
  CK(cudaFuncSetAttribute(k_atoms<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemA));
  grid = nsm;  // 1 block of 16 warps per SM
  const char* names[4] = {"conflict-free", "random-in-row(T=512)", "same-address", "lanes=rows random"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) k_atoms<0><<<grid, threads, smemA>>>(d, 512);
      if (m == 1) k_atoms<1><<<grid, threads, smemA>>>(d, 512);
      if (m == 2) k_atoms<2><<<grid, threads, smemA>>>(d, 512);
      if (m == 3) k_atoms<3><<<grid, threads, smemA>>>(d, 512);
      cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    }
    double ops = (double)grid * threads * ITERS;
    printf("ATOMS %-24s %.3f ms  %.2f Gop/s  %.2f lane-ops/clk/SM (at %d MHz)\n", names[m], ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_rng<<<grid, threads>>>(d, 512); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
  }
  printf("RNG-only                          %.3f ms\n", ms);
  size_t smemL = 48 * 1024;
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v == 0) k_lds<1><<<grid, threads, smemL>>>(d);
      if (v == 1) k_lds<2><<<grid, threads, smemL>>>(d);
      if (v == 2) k_lds<4><<<grid, threads, smemL>>>(d);
      cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    }
    double ins = (double)grid * (threads / 32) * ITERS;
    int bytes = 4 << v;
    printf("LDS.%-3d  %.3f ms  %.3f warp-instr/clk/SM  %.1f B/clk/SM\n", bytes * 8, ms,
           ins / (ms * 1e-3) / nsm / (clk * 1e3), ins * 32 * bytes / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  size_t nbytes = (size_t)2 << 30; int4* w; CK(cudaMalloc(&w, nbytes));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a); k_write<<<nsm * 8, 512>>>(w, nbytes / 16); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
  }
  printf("HBM streaming write 2 GiB: %.3f ms  %.1f GB/s\n", ms, nbytes / ms / 1e6);
  CK(cudaGetLastError());
  return 0;
}
