// k_onchip.cu - n = 11, 12 uniform-b Hadamard-test kernel (onchip_plane.cuh) and its planar,
// size-aligned copy of x.
#include <algorithm>

#include "launch.h"
#include "onchip_plane.cuh"

namespace dvqls {

KernelCfg onchip_cfg(int n) {
  KernelCfg k;
  if (n != 11 && n != 12) return k;
  k.fn = n == 11 ? (const void*)&onchip::onchip_plane_kernel<11> : (const void*)&onchip::onchip_plane_kernel<12>;
  k.warps = onchip::WARPS;
  k.groups = n == 11 ? onchip::Sh<11>::NG : onchip::Sh<12>::NG;
  k.smem = n == 11 ? onchip::smem_bytes<11>() : onchip::smem_bytes<12>();
  return k;
}

void launch_to_planar4(const double2* x, uint32_t N, uint32_t K, double* xq, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>(1184, (int64_t(K) * N + 255) / 256);
  onchip::to_planar4_kernel<<<unsigned(blocks), 256, 0, st>>>(x, N, K, xq);
}

}  // namespace dvqls
