// microbench.cu - measures the per-SM rates the roofline of the SMEM-resident
// Hadamard-test kernel uses (SURVEY.md §8(d) asks to confirm them on the box):
//   * FP64 pipe: independent DADD chains          -> lane-ops / clk / SM
//   * FP64 pipe: independent DFMA chains          -> lane-ops / clk / SM
//   * shared memory: conflict-free LDS.128        -> bytes / clk / SM
//   * shared memory: STS.128 + LDS.128 exchange   -> bytes / clk / SM
//   * warp shuffle SHFL.BFLY (32-bit)             -> bytes / clk / SM
//   * mixed DADD + LDS.128 (different warps)      -> do the two pipes overlap?
//   * mixed SHFL + LDS.128 (different warps)      -> do shuffles share the shared-memory data path?
// Cycles are read with clock64() per CTA (one CTA per SM, grid = #SMs), so the
// numbers are per SM clock and independent of the DVFS clock during the run.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int THREADS = 1024;

__global__ void __launch_bounds__(THREADS) k_dadd(double b, int iters, double* out, long long* cyc) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 += b; a1 += b; a2 += b; a3 += b; a4 += b; a5 += b; a6 += b; a7 += b;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * THREADS + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void __launch_bounds__(THREADS) k_dfma(double b, int iters, double* out, long long* cyc) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 1.0 + b;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, b); a1 = fma(a1, m, b); a2 = fma(a2, m, b); a3 = fma(a3, m, b);
    a4 = fma(a4, m, b); a5 = fma(a5, m, b); a6 = fma(a6, m, b); a7 = fma(a7, m, b);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * THREADS + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// each thread reads 16 B per LDS.128 from a 16 KB per-warp window, stride = lane -> conflict-free
__global__ void __launch_bounds__(THREADS) k_lds(int iters, unsigned* out, long long* cyc) {
  extern __shared__ double2 s[];
  for (int i = threadIdx.x; i < 8192; i += THREADS) s[i] = make_double2(i, -i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2* base = s + (warp & 7) * 1024;
  unsigned acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      double2 v = base[((i * 8 + r) & 31) * 32 + lane];
      acc ^= __double2loint(v.x) ^ __double2hiint(v.x) ^ __double2loint(v.y) ^ __double2hiint(v.y);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * THREADS + threadIdx.x] = acc;
}

// exchange: STS.128 32 values, syncwarp, LDS.128 32 values (transpose-like, swizzled)
__global__ void __launch_bounds__(THREADS) k_xchg(int iters, double* out, long long* cyc) {
  extern __shared__ double2 s[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // 32 warps x 4 KB (8 values/thread) = 128 KB
  double2* buf = s + warp * 256;
  double2 v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = make_double2(r + lane, r - lane);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) { int idx = (r << 5) | lane; buf[idx ^ ((idx >> 5) & 7)] = v[r]; }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 8; ++r) { int idx = ((lane & 7) << 5) | (r * 4 + (lane >> 3)); v[r] = buf[idx ^ ((idx >> 5) & 7)]; }
    __syncwarp();
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double a = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) a += v[r].x + v[r].y;
  out[blockIdx.x * THREADS + threadIdx.x] = a;
}

__global__ void __launch_bounds__(THREADS) k_shfl(int iters, unsigned* out, long long* cyc) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 * 11, a5 = a0 * 13, a6 = a0 * 17, a7 = a0 * 19;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = __shfl_xor_sync(0xffffffffu, a0, 1); a1 = __shfl_xor_sync(0xffffffffu, a1, 2);
    a2 = __shfl_xor_sync(0xffffffffu, a2, 4); a3 = __shfl_xor_sync(0xffffffffu, a3, 8);
    a4 = __shfl_xor_sync(0xffffffffu, a4, 16); a5 = __shfl_xor_sync(0xffffffffu, a5, 3);
    a6 = __shfl_xor_sync(0xffffffffu, a6, 5); a7 = __shfl_xor_sync(0xffffffffu, a7, 9);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * THREADS + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}

// half the warps do DADD, half do LDS.128: if the pipes overlap, the time is the max, not the sum
__global__ void __launch_bounds__(THREADS) k_mixed(double b, int iters_d, int iters_l, double* out, long long* cyc) {
  extern __shared__ double2 s[];
  for (int i = threadIdx.x; i < 8192; i += THREADS) s[i] = make_double2(i, -i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double r = 0;
  long long t0 = clock64();
  if (warp & 1) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters_d; ++i) {
      a0 += b; a1 += b; a2 += b; a3 += b; a4 += b; a5 += b; a6 += b; a7 += b;
    }
    r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  } else {
    const double2* base = s + (warp & 7) * 1024;
    unsigned acc = 0;
    for (int i = 0; i < iters_l; ++i) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double2 v = base[((i * 8 + q) & 31) * 32 + lane];
        acc ^= __double2loint(v.x) ^ __double2hiint(v.x) ^ __double2loint(v.y) ^ __double2hiint(v.y);
      }
    }
    r = acc;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * THREADS + threadIdx.x] = r;
}

// half the warps do SHFL.BFLY, half do LDS.128: do shuffles and shared loads share one data path?
__global__ void __launch_bounds__(THREADS) k_mixed_shfl(int iters_s, int iters_l, unsigned* out, long long* cyc) {
  extern __shared__ double2 s[];
  for (int i = threadIdx.x; i < 8192; i += THREADS) s[i] = make_double2(i, -i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned r = 0;
  long long t0 = clock64();
  if (warp & 1) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 * 11, a5 = a0 * 13, a6 = a0 * 17, a7 = a0 * 19;
    for (int i = 0; i < iters_s; ++i) {
      a0 = __shfl_xor_sync(0xffffffffu, a0, 1); a1 = __shfl_xor_sync(0xffffffffu, a1, 2);
      a2 = __shfl_xor_sync(0xffffffffu, a2, 4); a3 = __shfl_xor_sync(0xffffffffu, a3, 8);
      a4 = __shfl_xor_sync(0xffffffffu, a4, 16); a5 = __shfl_xor_sync(0xffffffffu, a5, 3);
      a6 = __shfl_xor_sync(0xffffffffu, a6, 5); a7 = __shfl_xor_sync(0xffffffffu, a7, 9);
    }
    r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  } else {
    const double2* base = s + (warp & 7) * 1024;
    unsigned acc = 0;
    for (int i = 0; i < iters_l; ++i) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double2 v = base[((i * 8 + q) & 31) * 32 + lane];
        acc ^= __double2loint(v.x) ^ __double2hiint(v.x) ^ __double2loint(v.y) ^ __double2hiint(v.y);
      }
    }
    r = acc;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * THREADS + threadIdx.x] = r;
}

// dependent-chain latencies (one warp): cycles per dependent op
__global__ void k_lat_dfma(double b, int iters, double* out, long long* cyc) {
  double a = threadIdx.x;
  const double m = 1.0 + b;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = fma(a, m, b); a = fma(a, m, b); a = fma(a, m, b); a = fma(a, m, b); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = a;
}
__global__ void k_lat_dadd(double b, int iters, double* out, long long* cyc) {
  double a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = a;
}
__global__ void k_lat_shfl(int iters, unsigned* out, long long* cyc) {
  unsigned a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a = __shfl_xor_sync(0xffffffffu, a, 1); a = __shfl_xor_sync(0xffffffffu, a, 2);
    a = __shfl_xor_sync(0xffffffffu, a, 4); a = __shfl_xor_sync(0xffffffffu, a, 8);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = a;
}
__global__ void k_lat_lds(int iters, unsigned* out, long long* cyc) {
  __shared__ unsigned s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  unsigned a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = s[a]; a = s[a]; a = s[a]; a = s[a]; }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = a;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* dout; long long* dcyc; unsigned* uout;
  CK(cudaMalloc(&dout, sizeof(double) * sms * THREADS));
  CK(cudaMalloc(&uout, sizeof(unsigned) * sms * THREADS));
  CK(cudaMalloc(&dcyc, sizeof(long long) * sms));
  std::vector<long long> cyc(sms);
  const int smem = 8192 * 16;  // 128 KB
  CK(cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_mixed_shfl, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_xchg, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 256 * 16));
  auto med = [&]() -> double { if (cudaMemcpy(cyc.data(), dcyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost) != cudaSuccess) return -1.0; std::sort(cyc.begin(), cyc.end()); return (double)cyc[sms / 2]; };
  const int it = 4096;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d", p.name, sms, p.clockRate);
  for (int rep = 0; rep < 2; ++rep) {
    k_dadd<<<sms, THREADS>>>(1e-9, it, dout, dcyc); CK(cudaDeviceSynchronize());
  }
  double c = med();
  printf(", \"dadd_lanes_per_clk_sm\": %.2f", double(THREADS) * it * 8 / c);
  k_dfma<<<sms, THREADS>>>(1e-9, it, dout, dcyc); CK(cudaDeviceSynchronize());
  c = med();
  printf(", \"dfma_lanes_per_clk_sm\": %.2f", double(THREADS) * it * 8 / c);
  k_lds<<<sms, THREADS, smem>>>(it, uout, dcyc); CK(cudaDeviceSynchronize());
  c = med();
  printf(", \"lds128_bytes_per_clk_sm\": %.2f", double(THREADS) * it * 8 * 16 / c);
  k_xchg<<<sms, THREADS, 32 * 256 * 16>>>(it / 4, dout, dcyc); CK(cudaDeviceSynchronize());
  c = med();
  printf(", \"sts_lds_exchange_bytes_per_clk_sm\": %.2f", double(THREADS) * (it / 4) * 16 * 16 / c);
  k_shfl<<<sms, THREADS>>>(it, uout, dcyc); CK(cudaDeviceSynchronize());
  c = med();
  printf(", \"shfl_bytes_per_clk_sm\": %.2f", double(THREADS) * it * 8 * 4 / c);
  // mixed: DADD warps issue 8*it_d per thread; LDS warps 8*it_l loads.  Choose equal standalone times.
  const int itd = 4096, itl = 4096;
  k_mixed<<<sms, THREADS, smem>>>(1e-9, itd, itl, dout, dcyc); CK(cudaDeviceSynchronize());
  c = med();
  const double t_d = (THREADS / 2.0) * itd * 8 / 64.0, t_l = (THREADS / 2.0) * itl * 8 * 16 / 128.0;
  printf(", \"mixed_cycles\": %.0f, \"mixed_model_sum\": %.0f, \"mixed_model_max\": %.0f", c, t_d + t_l, std::max(t_d, t_l));
  {
    // SHFL warps move 8 x 128 B per iteration, LDS warps 8 x 512 B: 4x the SHFL iterations for equal bytes
    const int its = 4 * 4096, itl2 = 4096;
    k_mixed_shfl<<<sms, THREADS, smem>>>(its, itl2, uout, dcyc); CK(cudaDeviceSynchronize());
    c = med();
    const double ts = (THREADS / 2.0) * its * 8 * 4 / 128.0, tl = (THREADS / 2.0) * itl2 * 8 * 16 / 128.0;
    printf(", \"mixed_shfl_lds_cycles\": %.0f, \"mixed_shfl_lds_model_sum\": %.0f, \"mixed_shfl_lds_model_max\": %.0f", c, ts + tl,
           std::max(ts, tl));
  }
  {
    const int li = 1024;
    k_lat_dfma<<<1, 32>>>(1e-9, li, dout, dcyc); CK(cudaDeviceSynchronize());
    long long c1; CK(cudaMemcpy(&c1, dcyc, 8, cudaMemcpyDeviceToHost));
    k_lat_dadd<<<1, 32>>>(1e-9, li, dout, dcyc); CK(cudaDeviceSynchronize());
    long long c2; CK(cudaMemcpy(&c2, dcyc, 8, cudaMemcpyDeviceToHost));
    k_lat_shfl<<<1, 32>>>(li, uout, dcyc); CK(cudaDeviceSynchronize());
    long long c3; CK(cudaMemcpy(&c3, dcyc, 8, cudaMemcpyDeviceToHost));
    k_lat_lds<<<1, 32>>>(li, uout, dcyc); CK(cudaDeviceSynchronize());
    long long c4; CK(cudaMemcpy(&c4, dcyc, 8, cudaMemcpyDeviceToHost));
    printf(", \"dfma_latency_clk\": %.1f, \"dadd_latency_clk\": %.1f, \"shfl_latency_clk\": %.1f, \"lds32_latency_clk\": %.1f",
           double(c1) / (4 * li), double(c2) / (4 * li), double(c3) / (4 * li), double(c4) / (4 * li));
  }
  printf("}\n");
  return 0;
}
