// Microbenchmarks for the k_sweep2d redesign (round 2): how fast can a warp gather
// 128-byte cw rows from shared memory in a direction-program order, with the program
// (row offsets) coming (a) from global memory per lane (LDG + IADD per LDS) or
// (b) from __constant__ memory through uniform registers (LDCU.64 + LDS [R+UR]);
// and how fast can 64-image x 8/16-bin output chunks be written with STG of various
// coalescing shapes vs a TMA-free baseline.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int NW = 16;        // warps per CTA
constexpr int PLEN = 1024;    // offsets per warp program
constexpr int ROWS = 785;
__constant__ uint32_t cprog[NW * PLEN];

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__global__ void __launch_bounds__(NW * 32, 1) k_gather_global(const uint32_t* __restrict__ prog, int reps, int* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < ROWS * 32; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) + 4 * lane;
  const uint4* p = (const uint4*)(prog + warp * PLEN);
  uint32_t S = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int k = 0; k < PLEN / 4; ++k) {
      uint4 w = __ldg(p + k);
      S += lds32(base + w.x) + lds32(base + w.y) + lds32(base + w.z) + lds32(base + w.w);
    }
  }
  if (S == 0x12345678u) out[0] = S;
}

__global__ void __launch_bounds__(NW * 32, 1) k_gather_const(int reps, int* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < ROWS * 32; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) + 4 * lane;
  const uint32_t* p = cprog + __shfl_sync(0xffffffffu, warp, 0) * PLEN;  // warp-uniform for ptxas
  uint32_t S = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int k = 0; k < PLEN; ++k) S += lds32(base + p[k]);
  }
  if (S == 0x12345678u) out[0] = S;
}

// const program + an "emit" every 8 gathers: extract two fields, add to bases, keep 16
// values in registers (static slots), and every 16 emits write them to a per-warp smem
// stage with STS.128 (the TMA-store design's register side).
__global__ void __launch_bounds__(NW * 32, 1) k_gather_const_emit(int reps, int* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < ROWS * 32; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) + 4 * lane;
  const uint32_t* p = cprog + __shfl_sync(0xffffffffu, warp, 0) * PLEN;  // warp-uniform for ptxas
  int4* st = (int4*)(tab + ROWS * 32) + warp * 256 + lane * 8;
  int B0 = 0, B1 = 0;
  int o0[16], o1[16];
  for (int r = 0; r < reps; ++r) {
    for (int c = 0; c < PLEN / 128; ++c) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t* q = p + c * 128 + k * 8;
        uint32_t S = lds32(base + q[0]) + lds32(base + q[1]);
        S += lds32(base + q[2]) + lds32(base + q[3]);
        S += lds32(base + q[4]) + lds32(base + q[5]);
        S += lds32(base + q[6]) + lds32(base + q[7]);
        B0 += S & 0xFFFF;
        B1 += S >> 16;
        o0[k] = B0 + (int)q[7];
        o1[k] = B1 + (int)q[7];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        st[k] = make_int4(o0[4 * k], o0[4 * k + 1], o0[4 * k + 2], o0[4 * k + 3]);
        st[4 + k] = make_int4(o1[4 * k], o1[4 * k + 1], o1[4 * k + 2], o1[4 * k + 3]);
      }
      __syncwarp();
    }
  }
  if (B0 == 0x12345678) out[0] = B0;
}

// Output-store shapes: each warp writes [64 images][CH bins] int32 chunks of a
// [B][D][T] tensor (T = 128, D = 64) -- lane-to-address maps of the candidate designs.
// SHAPE 0: 16 B per lane, 32 distinct images per instruction (no exchange)
// SHAPE 1: 2 lanes per image (32 B), 16 images per instruction (round-1 k_sweep2d)
// SHAPE 2: 4 lanes per image (64 B), 8 images per instruction (16-bin chunks)
// SHAPE 3: 8 lanes per image (128 B), 4 images per instruction (32-bin chunks)
template <int SHAPE>
__global__ void __launch_bounds__(NW * 32, 1) k_store(int* __restrict__ out, int64_t B, int D, int T) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int LPI = SHAPE == 0 ? 1 : SHAPE == 1 ? 2 : SHAPE == 2 ? 4 : 8;  // lanes per image
  constexpr int CH = 4 * LPI;                                                // bins per chunk
  const int64_t ngroups = B / 64;
  const int4 v = make_int4(lane, warp, 1, 2);
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    for (int d = warp; d < D; d += NW) {
      for (int q0 = 0; q0 < T; q0 += CH) {
#pragma unroll
        for (int r = 0; r < 64 / (32 / LPI); ++r) {
          const int64_t img = g * 64 + r * (32 / LPI) + lane / LPI;
          __stcs((int4*)(out + (img * D + d) * T + q0 + 4 * (lane % LPI)), v);
        }
      }
    }
  }
}


// P parts per warp (P = 1: LDS.32, all lanes one row; P = 2: LDS.64, half-warps read
// two rows; P = 4: LDS.128, quarter-warps read four rows).  Offsets come from global
// memory: lane reads its part's next 4 offsets with one LDG.128 (layout [group][part][4]).
template <int P, int NWARP, int UNR>
__global__ void __launch_bounds__(NWARP * 32, 1) k_gather_parts(const uint32_t* __restrict__ prog, int reps, int* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < ROWS * 32; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & (NW - 1);
  constexpr int LPP = 32 / P;  // lanes per part
  const int part = lane / LPP, sub = lane % LPP;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) + (128 / LPP) * sub;
  const uint4* p = (const uint4*)(prog + warp * PLEN) + part;
  uint32_t S0 = 0, S1 = 0, S2 = 0, S3 = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll UNR
    for (int k = 0; k < PLEN / (4 * P); ++k) {
      const uint4 w = __ldg(p + k * P);
      const uint32_t o[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (P == 1) {
          uint32_t v;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + o[j]));
          S0 += v;
        } else if (P == 2) {
          uint32_t a, b;
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(base + o[j]));
          S0 += a; S1 += b;
        } else {
          uint32_t a, b, c, d;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(base + o[j]));
          S0 += a; S1 += b; S2 += c; S3 += d;
        }
      }
    }
  }
  if ((S0 ^ S1 ^ S2 ^ S3) == 0x12345678u) out[0] = S0;
}

template <int P, int NWARP, int UNR>
int run_parts(const uint32_t* dprog, int* dout, int nsm, int clk, int reps, size_t smem, const char* name) {
  CK(cudaFuncSetAttribute(k_gather_parts<P, NWARP, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    CK(cudaEventRecord(e0));
    k_gather_parts<P, NWARP, UNR><<<nsm, NWARP * 32, smem>>>(dprog, reps, dout);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  // rows gathered per SM: NWARP warps x PLEN offsets x reps (each offset = one 128 B row)
  const double rows = (double)NWARP * PLEN * reps;
  printf("parts P=%d warps=%2d unroll=%d %-10s %.3f ms  %.3f rows/clk/SM  %.1f B/clk/SM\n", P, NWARP, UNR, name, best,
         rows / (best * 1e-3 * clk * 1e3), 128 * rows / (best * 1e-3 * clk * 1e3));
  return 0;
}


// MIO cost probes (L2-resident, not HBM-bound): each warp issues N instructions of one kind.
// KIND 0..3: STG.128 with 1/2/4/8 lanes per 16-B-contiguous run per image (16/32/64/128 B),
// rows 512 B apart, into a 4 MB buffer (L2 resident).  KIND 4: SHFL.BFLY.  KIND 5: STS.32
// conflict-free.  KIND 6: STS.128 conflict-free.  KIND 7: STS.64.
template <int KIND>
__global__ void __launch_bounds__(NW * 32, 1) k_mio(int* __restrict__ buf, int reps, int* out) {
  __shared__ int4 sm[NW * 32 * 4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int acc = lane;
  int4 v = make_int4(lane, warp, reps, 1);
  int* wb = buf + ((size_t)blockIdx.x * NW + warp) * 1024;  // 4 KB per warp
#pragma unroll 1
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (KIND <= 3) {
        constexpr int LPI = 1 << KIND;
        const int img = lane / LPI;
        __stcg((int4*)(wb + (img * 128 + 4 * (lane % LPI) + k * 4 * LPI) % 1024), v);
        v.x += 1;
      } else if (KIND == 4) {
        acc = __shfl_xor_sync(0xffffffffu, acc, 1 + (k & 15)) + k;
      } else if (KIND == 5) {
        ((int*)sm)[warp * 128 + ((lane + k * 32) & 127)] = acc + k;
      } else if (KIND == 6) {
        sm[warp * 32 + lane] = make_int4(acc, k, r, 1);
      } else {
        ((int2*)sm)[warp * 64 + ((lane + 32 * (k & 1)))] = make_int2(acc, k);
      }
    }
  }
  __syncthreads();
  if (KIND >= 5 && threadIdx.x == 0) out[blockIdx.x] = ((int*)sm)[7];
  if (acc == 0x7777777) out[0] = acc;
}

template <int KIND>
int run_mio(int* buf, int* dout, int nsm, int clk, const char* name) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 4096;
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    CK(cudaEventRecord(e0));
    k_mio<KIND><<<nsm, NW * 32>>>(buf, reps, dout);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  const double ins = (double)NW * reps * 16;  // per SM
  printf("MIO %-34s %.3f ms  %.3f cyc/instr/SM\n", name, best, best * 1e-3 * clk * 1e3 / ins);
  return 0;
}


// constant-bank programs of PL offsets per warp (total NW * PL * 4 bytes): LDCU.64 + LDS [R+UR]
template <int PL, int STR>
__global__ void __launch_bounds__(NW * 32, 1) k_gather_constN(int reps, int* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < ROWS * 32; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) + 4 * lane;
  const uint32_t* p = cprog + __shfl_sync(0xffffffffu, warp, 0) * STR;
  uint32_t S = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int k = 0; k < PL; ++k) S += lds32(base + p[k]);
  }
  if (S == 0x12345678u) out[0] = S;
}
template <int PL, int STR>
int run_constN(int* dout, int nsm, int clk, size_t smem) {
  CK(cudaFuncSetAttribute(k_gather_constN<PL, STR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 200 * 1024 / PL;
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    CK(cudaEventRecord(e0));
    k_gather_constN<PL, STR><<<nsm, NW * 32, smem>>>(reps, dout);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  const double rows = (double)NW * PL * reps;
  printf("const program %6d B per warp, stride %6d B: %.3f ms  %.3f rows/clk/SM\n", PL * 4, STR * 4, best, rows / (best * 1e-3 * clk * 1e3));
  return 0;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("SMs %d clock %d kHz\n", nsm, clk);
  // random programs: row offsets * 128
  static uint32_t h[NW * PLEN];
  uint32_t x = 12345;
  for (int i = 0; i < NW * PLEN; ++i) { x = x * 1664525u + 1013904223u; h[i] = ((x >> 8) % ROWS) * 128u; }
  uint32_t* dprog;
  int* dout;
  CK(cudaMalloc(&dprog, sizeof(h)));
  CK(cudaMalloc(&dout, 1024));
  CK(cudaMemcpy(dprog, h, sizeof(h), cudaMemcpyHostToDevice));
  CK(cudaMemcpyToSymbol(cprog, h, sizeof(h)));
  const size_t smem = ROWS * 128 + NW * 4096;
  CK(cudaFuncSetAttribute(k_gather_global, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_gather_const, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_gather_const_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 200;
  const double lds_per_sm = (double)NW * PLEN * reps;
  for (int variant = 0; variant < 3; ++variant) {
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      CK(cudaEventRecord(e0));
      if (variant == 0) k_gather_global<<<nsm, NW * 32, smem>>>(dprog, reps, dout);
      else if (variant == 1) k_gather_const<<<nsm, NW * 32, smem>>>(reps, dout);
      else k_gather_const_emit<<<nsm, NW * 32, smem>>>(reps, dout);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    const char* nm[3] = {"global offsets (LDG.128 + IADD)", "const offsets (LDCU.64, LDS [R+UR])", "const + emit/stage"};
    printf("gather %-38s %.3f ms  %.3f cyc/LDS/SM  (%.2f warp-LDS/clk/SM)\n", nm[variant], best,
           best * 1e-3 * clk * 1e3 / lds_per_sm, lds_per_sm / (best * 1e-3 * clk * 1e3));
  }
  run_constN<64, 64>(dout, nsm, clk, smem);
  run_constN<64, 80>(dout, nsm, clk, smem);
  run_constN<128, 128>(dout, nsm, clk, smem);
  run_constN<128, 144>(dout, nsm, clk, smem);
  run_constN<128, 136>(dout, nsm, clk, smem);
  run_constN<256, 272>(dout, nsm, clk, smem);
  run_constN<512, 528>(dout, nsm, clk, smem);
  run_constN<1000, 1016>(dout, nsm, clk, smem);
  run_constN<1000, 1000>(dout, nsm, clk, smem);
  run_parts<1, 16, 4>(dprog, dout, nsm, clk, reps, smem, "");
  run_parts<1, 16, 8>(dprog, dout, nsm, clk, reps, smem, "");
  run_parts<1, 32, 4>(dprog, dout, nsm, clk, reps, smem, "");
  run_parts<2, 16, 4>(dprog, dout, nsm, clk, reps, smem, "");
  run_parts<2, 32, 2>(dprog, dout, nsm, clk, reps, smem, "");
  run_parts<4, 16, 2>(dprog, dout, nsm, clk, reps, smem, "");
  run_parts<4, 16, 4>(dprog, dout, nsm, clk, reps, smem, "");
  run_parts<4, 32, 2>(dprog, dout, nsm, clk, reps, smem, "");
  {
    int* buf;
    CK(cudaMalloc(&buf, (size_t)nsm * NW * 4096));
    run_mio<0>(buf, dout, nsm, clk, "STG.128 16 B/img (32 lines/instr)");
    run_mio<1>(buf, dout, nsm, clk, "STG.128 32 B/img (16 lines/instr)");
    run_mio<2>(buf, dout, nsm, clk, "STG.128 64 B/img (8 lines/instr)");
    run_mio<3>(buf, dout, nsm, clk, "STG.128 128 B/img (4 lines/instr)");
    run_mio<4>(buf, dout, nsm, clk, "SHFL.BFLY");
    run_mio<5>(buf, dout, nsm, clk, "STS.32");
    run_mio<6>(buf, dout, nsm, clk, "STS.128");
    run_mio<7>(buf, dout, nsm, clk, "STS.64");
  }
  // stores: B = 60000, D = 64, T = 128 int32 = 1.97 GB
  const int64_t B = 60032;
  const int D = 64, T = 128;
  int* o;
  CK(cudaMalloc(&o, (size_t)B * D * T * 4));
  for (int s = 0; s < 4; ++s) {
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      CK(cudaEventRecord(e0));
      if (s == 0) k_store<0><<<nsm, NW * 32>>>(o, B, D, T);
      if (s == 1) k_store<1><<<nsm, NW * 32>>>(o, B, D, T);
      if (s == 2) k_store<2><<<nsm, NW * 32>>>(o, B, D, T);
      if (s == 3) k_store<3><<<nsm, NW * 32>>>(o, B, D, T);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    printf("store shape %d (%3d B per image per instr): %.3f ms  %.1f GB/s\n", s, 16 << s, best,
           (double)B * D * T * 4 / best / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
