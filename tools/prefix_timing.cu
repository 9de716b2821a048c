// prefix_timing.cu - clock64 phase stamps of prefix_quad_kernel<10> (kernels.cuh built with
// -DDVQLS_PREFIX_TS), lane 0 of every warp of CTA 0, cfg3 depth d = 10, and its back-to-back launch
// time.  Stamps (cycles from kernel entry): 1 gate + ring tables done, 2 layer 0's register and
// lane gates (positions 0..6), 3 end of layer 0 (two transposes, warp-bit gates, ring), 4 end of
// all layers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DDVQLS_PREFIX_TS -I paper_2604_14435_b200/csrc \
//        -o tools/prefix_timing tools/prefix_timing.cu
#include <cstdio>
#include <vector>
#include "kernels.cuh"
__global__ void empty_kernel(double2* x) {
  extern __shared__ double2 esm[];
  if (threadIdx.x == 0) esm[0] = x[0];
  __syncthreads();
  if (threadIdx.x == 0) x[1] = esm[0];
}
int main() {
  const int n = 10, d = 10, P = 3 * n * d, N = 1 << n;
  std::vector<double> th(P);
  for (int i = 0; i < P; ++i) th[i] = 0.37 * i - 2.0;
  double* dth;
  double2* dx;
  cudaMalloc(&dth, P * 8);
  cudaMalloc(&dx, N * 16);
  cudaMemcpy(dth, th.data(), P * 8, cudaMemcpyHostToDevice);
  const size_t smem = sizeof(double2) * (2 * N + 2 * n * d) + sizeof(int) * N;
  cudaFuncSetAttribute((const void*)&dvqls::prefix_quad_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(smem));
  for (int i = 0; i < 5; ++i) dvqls::prefix_quad_kernel<10><<<1, N / 4, smem>>>(d, 0, dth, dx);
  cudaDeviceSynchronize();
  long long ts[256];
  cudaMemcpyFromSymbol(ts, dvqls::g_prefix_ts, sizeof ts);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) dvqls::prefix_quad_kernel<10><<<1, N / 4, smem>>>(d, 0, dth, dx);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"err\": \"%s\", \"us_per_launch_back_to_back\": %.2f, \"stamps_per_warp\": [",
         cudaGetErrorString(cudaGetLastError()), ms * 10.0f);
  for (int w = 0; w < 8; ++w) {
    printf("%s[", w ? ", " : "");
    for (int k = 1; k <= 4; ++k) printf("%s%lld", k > 1 ? ", " : "", ts[w * 16 + k] - ts[w * 16]);
    printf("]");
  }
  printf("]");
  // the same kernel, stamped again once alone: %globaltimer duration of its body and the SM clock
  dvqls::prefix_quad_kernel<10><<<1, N / 4, smem>>>(d, 0, dth, dx);
  cudaDeviceSynchronize();
  unsigned long long gt[256];
  cudaMemcpyFromSymbol(ts, dvqls::g_prefix_ts, sizeof ts);
  cudaMemcpyFromSymbol(gt, dvqls::g_prefix_gt, sizeof gt);
  const double ns = double(gt[4] - gt[0]), cyc = double(ts[4] - ts[0]);
  printf(", \"body_ns_warp0\": %.0f, \"body_cycles_warp0\": %.0f, \"sm_ghz_in_body\": %.3f", ns, cyc, cyc / ns);
  // launch floor: an (almost) empty kernel with the same launch configuration, back to back
  cudaFuncSetAttribute((const void*)&empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int i = 0; i < 5; ++i) empty_kernel<<<1, N / 4, smem>>>(dx);
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) empty_kernel<<<1, N / 4, smem>>>(dx);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf(", \"empty_us_per_launch_back_to_back\": %.2f}\n", ms * 10.0f);
  return 0;
}
