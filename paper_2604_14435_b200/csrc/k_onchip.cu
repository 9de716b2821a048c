// k_onchip.cu - n = 11, 12 uniform-b Hadamard-test kernel (onchip_plane.cuh) and its planar,
// size-aligned copy of x.
#include <algorithm>

#include "launch.h"
#include "onchip_plane.cuh"

namespace dvqls {

template <int NQ, bool XS>
static KernelCfg cfg_of() {
  KernelCfg k;
  k.fn = (const void*)&onchip::onchip_plane_kernel<NQ, XS>;
  k.warps = onchip::Sh<NQ, XS>::W;
  k.groups = onchip::Sh<NQ, XS>::NG;
  k.smem = onchip::smem_bytes<NQ, XS>();
  return k;
}

KernelCfg onchip_cfg(int n, bool x_in_smem) {
  if (n == 11) return x_in_smem ? cfg_of<11, true>() : cfg_of<11, false>();
  if (n == 12) return x_in_smem ? cfg_of<12, true>() : cfg_of<12, false>();
  return KernelCfg{};
}

void launch_to_planar4(const double2* x, uint32_t N, uint32_t K, double* xq, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>(1184, (int64_t(K) * N + 255) / 256);
  onchip::to_planar4_kernel<<<unsigned(blocks), 256, 0, st>>>(x, N, K, xq);
}

}  // namespace dvqls
