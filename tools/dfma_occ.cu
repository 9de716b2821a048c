#include <cstdio>
template <int ILP>
__global__ void k(double b, int iters, double* out, long long* cyc) {
  double a[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) a[j] = threadIdx.x + j;
  const double m = 1.0 + b;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < ILP; ++j) a[j] = fma(a[j], m, b);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += a[j];
  out[threadIdx.x] = s;
}
template <int ILP> void run(int threads, double* o, long long* c) {
  const int it = 4096;
  k<ILP><<<1, threads>>>(1e-9, it, o, c); cudaDeviceSynchronize();
  k<ILP><<<1, threads>>>(1e-9, it, o, c); cudaDeviceSynchronize();
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("threads %4d ILP %2d: %.2f lanes/clk/SM (%.2f clk per warp-DFMA per SMSP)\n", threads, ILP,
         double(threads) * it * ILP / cy, double(cy) / (double(threads / 32) / 4 * it * ILP));
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
  for (int t : {128, 256, 512, 1024}) { run<1>(t, o, c); run<2>(t, o, c); run<4>(t, o, c); run<8>(t, o, c); }
  return 0;
}
