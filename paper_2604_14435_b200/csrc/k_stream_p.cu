// k_stream_p.cu - n >= 13 uniform-b streaming Hadamard-test kernel (stream_plane.cuh), its planar
// copy of x, and the global-memory prefix V(theta)|0> (tile.cuh, SURVEY §8(a) a2 for n >= 13).
#include <algorithm>

#include "launch.h"
#include "stream_plane.cuh"
#include "tile.cuh"

namespace dvqls {

KernelCfg stream_plane_cfg(bool staged) {
  KernelCfg k;
  k.fn = staged ? (const void*)&streamp::stream_plane_kernel<12, true>
                : (const void*)&streamp::stream_plane_kernel<12, false>;
  k.warps = stream::TS<12>::THREADS / 32;
  k.groups = 1;
  k.smem = staged ? streamp::staged_smem<12>() : streamp::tile_smem<12>();
  return k;
}

void launch_to_planar(const double2* x, uint32_t N, uint32_t K, double* xp, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>(1184, (int64_t(K) * N + 255) / 256);
  streamp::to_planar_kernel<<<unsigned(blocks), 256, 0, st>>>(x, N, K, xp);
}

static int ngroups_host(int n) { return n <= 12 ? 1 : (n <= 21 ? 2 : 3); }

int prefix_global_launches(int n, int layers) { return 2 + layers * (ngroups_host(n) + 2); }

int launch_prefix_global(int n, int layers, int entangler, int K, const double* thetas, double2* x, double2* x2,
                         double2* gates, cudaStream_t st) {
  {
    cudaError_t e = cudaFuncSetAttribute((const void*)&tile::prefix_gate_pass,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(double2) * tile::TN));
    if (e != cudaSuccess) return int(e);
  }
  const int G = n * layers, P = 3 * n * layers, ng = ngroups_host(n);
  const uint32_t N = 1u << n;
  for (int k = 0; k < K; ++k) {
    double2* xk = x + size_t(k) * N;
    tile::prefix_gates_kernel<<<(G + 127) / 128, 128, 0, st>>>(thetas + size_t(k) * P, G, gates);
    tile::prefix_init_kernel<<<1024, 256, 0, st>>>(xk, N);
    for (int layer = 0; layer < layers; ++layer) {
      for (int gi = 0; gi < ng; ++gi)
        tile::prefix_gate_pass<<<N >> tile::TBITS, tile::THREADS, sizeof(double2) * tile::TN, st>>>(xk, gates, n, gi,
                                                                                                  layer);
      tile::prefix_ring_kernel<<<1024, 256, 0, st>>>(xk, x2, n, entangler);
      cudaError_t e = cudaMemcpyAsync(xk, x2, sizeof(double2) * N, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return int(e);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return int(e);
  }
  return 0;
}

}  // namespace dvqls
