// k_plane.cu - the n = 10 uniform-b real-plane Hadamard-test kernel (plane.cuh, the headline
// kernel), the SMEM-resident prefix kernels for n <= 12 (kernels.cuh) and the
// finalize kernel of the NCCL reduction path (a10).
#include <algorithm>

#include "kernels.cuh"
#include "launch.h"
#include "plane.cuh"
#include "plane2.cuh"
#include "prefix_cluster.cuh"

namespace dvqls {

KernelCfg plane_cfg() {
  constexpr int W = 20;  // 5 warps per SM sub-partition (<= 96 registers); measured faster than 16
  KernelCfg k;
  k.fn = (const void*)&plane::plane_kernel<W>;
  k.warps = W;
  k.groups = W / 2;
  // the x planes sit at a 16 KB-aligned shared-window address inside the allocation: size it for
  // the actual dynamic base (reserved SMEM + this kernel's static SMEM); the kernel traps if the
  // base differs
  cudaFuncAttributes fa{};
  int dev = 0, reserved = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaFuncGetAttributes(&fa, k.fn);
  const uint32_t sb = uint32_t(reserved) + ((uint32_t(fa.sharedSizeBytes) + 15u) & ~15u);
  k.smem = plane::smem_bytes<W>(sb);
  return k;
}

KernelCfg plane2_cfg() {
  KernelCfg k;
  k.fn = (const void*)&plane2::plane2_kernel;
  k.warps = plane2::WARPS;
  k.groups = plane2::NP;
  cudaFuncAttributes fa{};
  int dev = 0, reserved = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaFuncGetAttributes(&fa, k.fn);
  const uint32_t sb = uint32_t(reserved) + ((uint32_t(fa.sharedSizeBytes) + 15u) & ~15u);
  k.smem = plane2::smem_bytes(sb);
  return k;
}

PrefixCfg prefix_cfg(int n, int layers, bool cluster) {
  static const void* quads[11] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                  (const void*)&prefix_quad_kernel<7>, (const void*)&prefix_quad_kernel<8>,
                                  (const void*)&prefix_quad_kernel<9>, (const void*)&prefix_quad_kernel<10>};
  static const void* lanes[7] = {nullptr,
                                 (const void*)&prefix_lanes_kernel<1>, (const void*)&prefix_lanes_kernel<2>,
                                 (const void*)&prefix_lanes_kernel<3>, (const void*)&prefix_lanes_kernel<4>,
                                 (const void*)&prefix_lanes_kernel<5>, (const void*)&prefix_lanes_kernel<6>};
  static const void* clus[11] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                 (const void*)&pclus::prefix_cluster_kernel<7>, (const void*)&pclus::prefix_cluster_kernel<8>,
                                 (const void*)&pclus::prefix_cluster_kernel<9>, (const void*)&pclus::prefix_cluster_kernel<10>};
  static const size_t csm[11] = {0, 0, 0, 0, 0, 0, 0, sizeof(double2) * pclus::smem_doubles2<7>(1),
                                 sizeof(double2) * pclus::smem_doubles2<8>(1), sizeof(double2) * pclus::smem_doubles2<9>(1),
                                 sizeof(double2) * pclus::smem_doubles2<10>(1)};
  PrefixCfg p;
  const size_t N = size_t(1) << n;
  // cluster: 7 <= n <= 10, the state spread over 2^(n-7) CTAs joined by DSMEM (one amplitude per
  // thread), while its tables fit the SMEM of one CTA (they grow with the depth).  Measured at cfg3
  // (profiles/r2_cluster_prefix/): 20-24 us vs 21-23 us for the one-CTA kernel -- the per-layer
  // cluster barrier (~0.9 K cycles with skew) and the 8x-redundant DSMEM gather (~1-1.6 K cycles)
  // cost what the 8 SMs save -- so it is the opt-in variant (opts.prefix = 1).
  if (cluster && n >= 7 && n <= 10) {
    const size_t per_layer = csm[n] - sizeof(double2) * 3 * pclus::NL;
    const size_t bytes = sizeof(double2) * 3 * pclus::NL + per_layer * size_t(layers);
    if (bytes <= size_t(200) << 10) {
      p.fn = clus[n];
      p.threads = pclus::NL;
      p.smem = bytes;
      p.cluster = 1 << (n - pclus::LB);
      return p;
    }
  }
  if (n >= 7 && n <= 10) {  // 4 amplitudes per thread, shuffles + 2 transposes per layer
    p.fn = quads[n];
    p.threads = std::max(32, int(N / 4));
    p.smem = sizeof(double2) * (2 * N + 2 * size_t(n) * layers) + sizeof(int) * N;
  } else if (n >= 1 && n < 7) {  // one amplitude per thread
    p.fn = lanes[n];
    p.threads = std::max(32, int(N));
    p.smem = sizeof(double2) * (N + 4 * size_t(n) * layers) + sizeof(int) * N;
  } else if (n <= 12) {  // 8 amplitudes per thread, register phases (n = 11, 12)
    p.fn = (const void*)&prefix_kernel<3>;
    p.with_n = true;
    const int T = int(N >> 3);
    p.threads = std::min(512, std::max(32, (T + 31) / 32 * 32));
    p.smem = sizeof(double2) * (2 * N + 2 * size_t(n) * layers) + sizeof(int) * N;
  }
  return p;
}

// a10 after the cross-rank allreduce: (E, Psi)[K] -> (C, E, Psi)[K]
static __global__ void finalize_kernel(const double* __restrict__ ep, int K, int n, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double* e = ep + 4 * k;
  double* o = out + 5 * k;
  o[0] = cost_of_dev(e[0], e[2], n);
  o[1] = e[0]; o[2] = e[1]; o[3] = e[2]; o[4] = e[3];
}


#ifdef DVQLS_PLANE2_TS
void* plane2_ts_ptr() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, plane2::g_p2ts);
  return p;
}
#endif

void launch_finalize(const double* ep, int K, int n, double* out, cudaStream_t st) {
  finalize_kernel<<<(K + 255) / 256, 256, 0, st>>>(ep, K, n, out);
}

}  // namespace dvqls
