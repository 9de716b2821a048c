// gate_rate.cu - FP64 issue rate of the prefix's 2x2 complex gate pattern (4 outputs, each a
// DMUL + 3 dependent DFMA with three distinct register operands) at 256 threads / SM, against
// the plain DFMA chain rate: does the gate pattern run at the pipe's 2.2 clk per warp-instruction?
#include <cstdio>
struct d2 { double x, y; };
__device__ __forceinline__ void gate(const d2 ua, const d2 ub, d2& x0, d2& x1) {
  const d2 a = x0, b = x1;
  x0.x = fma(ua.x, a.x, fma(-ua.y, a.y, fma(-ub.x, b.x, -ub.y * b.y)));
  x0.y = fma(ua.x, a.y, fma(ua.y, a.x, fma(-ub.x, b.y, ub.y * b.x)));
  x1.x = fma(ub.x, a.x, fma(-ub.y, a.y, fma(ua.x, b.x, ua.y * b.y)));
  x1.y = fma(ub.x, a.y, fma(ub.y, a.x, fma(ua.x, b.y, -ua.y * b.x)));
}
// the same gate, coefficient-major: the four products with ua.x first (one operand shared by four
// consecutive instructions), then ua.y, ub.x, ub.y
__device__ __forceinline__ void gate_cm(const d2 ua, const d2 ub, d2& x0, d2& x1) {
  const d2 a = x0, b = x1;
  double p = ua.x * a.x, q = ua.x * a.y, r = ua.x * b.x, t = ua.x * b.y;
  p = fma(-ua.y, a.y, p); q = fma(ua.y, a.x, q); r = fma(ua.y, b.y, r); t = fma(-ua.y, b.x, t);
  p = fma(-ub.x, b.x, p); q = fma(-ub.x, b.y, q);
  double u = fma(ub.x, a.x, r), w = fma(ub.x, a.y, t);
  p = fma(-ub.y, b.y, p); q = fma(ub.y, b.x, q); u = fma(-ub.y, a.y, u); w = fma(ub.y, a.x, w);
  x0.x = p; x0.y = q; x1.x = u; x1.y = w;
}
template <int PAIRS>
__global__ void kcm(const double* __restrict__ tab, int iters, double* out, long long* cyc) {
  d2 v[2 * PAIRS];
#pragma unroll
  for (int j = 0; j < 2 * PAIRS; ++j) { v[j].x = 1e-3 * (threadIdx.x + j); v[j].y = 0.5e-3 * j; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const d2 ua = {tab[(i & 15) * 4], tab[(i & 15) * 4 + 1]}, ub = {tab[(i & 15) * 4 + 2], tab[(i & 15) * 4 + 3]};
#pragma unroll
    for (int p = 0; p < PAIRS; ++p) gate_cm(ua, ub, v[2 * p], v[2 * p + 1]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int j = 0; j < 2 * PAIRS; ++j) s += v[j].x + v[j].y;
  out[threadIdx.x] = s;
}
template <int PAIRS> void runcm(int threads, const double* t, double* o, long long* c) {
  const int it = 2048;
  kcm<PAIRS><<<1, threads>>>(t, it, o, c); cudaDeviceSynchronize();
  kcm<PAIRS><<<1, threads>>>(t, it, o, c); cudaDeviceSynchronize();
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  const double instr = double(threads / 32) / 4 * it * PAIRS * 16;
  printf("coefficient-major: threads %4d pairs/thread %d: %.2f clk per FP64 warp-instruction per SMSP\n", threads, PAIRS, cy / instr);
}
template <int PAIRS>
__global__ void k(const double* __restrict__ tab, int iters, double* out, long long* cyc) {
  d2 v[2 * PAIRS];
#pragma unroll
  for (int j = 0; j < 2 * PAIRS; ++j) { v[j].x = 1e-3 * (threadIdx.x + j); v[j].y = 0.5e-3 * j; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const d2 ua = {tab[(i & 15) * 4], tab[(i & 15) * 4 + 1]}, ub = {tab[(i & 15) * 4 + 2], tab[(i & 15) * 4 + 3]};
#pragma unroll
    for (int p = 0; p < PAIRS; ++p) gate(ua, ub, v[2 * p], v[2 * p + 1]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int j = 0; j < 2 * PAIRS; ++j) s += v[j].x + v[j].y;
  out[threadIdx.x] = s;
}
// the same gates with the coefficients as kernel parameters (constant-bank operands of the DFMAs)
template <int PAIRS>
__global__ void kc(d2 ua, d2 ub, int iters, double* out, long long* cyc) {
  d2 v[2 * PAIRS];
#pragma unroll
  for (int j = 0; j < 2 * PAIRS; ++j) { v[j].x = 1e-3 * (threadIdx.x + j); v[j].y = 0.5e-3 * j; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int p = 0; p < PAIRS; ++p) gate(ua, ub, v[2 * p], v[2 * p + 1]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int j = 0; j < 2 * PAIRS; ++j) s += v[j].x + v[j].y;
  out[threadIdx.x] = s;
}
template <int PAIRS> void runc(int threads, double* o, long long* c) {
  const int it = 2048;
  const d2 ua = {0.6, 0.1}, ub = {0.3, -0.2};
  kc<PAIRS><<<1, threads>>>(ua, ub, it, o, c); cudaDeviceSynchronize();
  kc<PAIRS><<<1, threads>>>(ua, ub, it, o, c); cudaDeviceSynchronize();
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  const double instr = double(threads / 32) / 4 * it * PAIRS * 16;
  printf("const-bank coefficients: threads %4d pairs/thread %d: %.2f clk per FP64 warp-instruction per SMSP\n", threads, PAIRS, cy / instr);
}
template <int PAIRS> void run(int threads, const double* t, double* o, long long* c) {
  const int it = 2048;
  k<PAIRS><<<1, threads>>>(t, it, o, c); cudaDeviceSynchronize();
  k<PAIRS><<<1, threads>>>(t, it, o, c); cudaDeviceSynchronize();
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  const double instr = double(threads / 32) / 4 * it * PAIRS * 16;  // FP64 warp-instructions per SMSP
  printf("threads %4d pairs/thread %d: %.2f clk per FP64 warp-instruction per SMSP\n", threads, PAIRS, cy / instr);
}
int main() {
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 0.1 + 0.01 * i;
  double *t, *o; long long* c; cudaMalloc(&t, 512); cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
  cudaMemcpy(t, h, 512, cudaMemcpyHostToDevice);
  for (int th : {128, 256, 512, 1024}) { run<1>(th, t, o, c); run<2>(th, t, o, c); run<4>(th, t, o, c); }
  for (int th : {256, 512}) { runc<1>(th, o, c); runc<2>(th, o, c); runc<4>(th, o, c); }
  for (int th : {256, 512}) { runcm<1>(th, t, o, c); runcm<2>(th, t, o, c); runcm<4>(th, t, o, c); }
  return 0;
}
