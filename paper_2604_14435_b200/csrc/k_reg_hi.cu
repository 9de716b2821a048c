// k_reg_hi.cu - complex register-path Hadamard-test kernels, n = 7..10 (kernels.cuh; for n = 10
// only Householder b: uniform b at n = 10 runs the real-plane kernel, k_plane.cu).
#include "k_reg.inc"

namespace dvqls {
KernelCfg reg_cfg_hi(int n, bool hh) {
  switch (n) {
    case 7: return cfg_n<7>(hh);
    case 8: return cfg_n<8>(hh);
    case 9: return cfg_n<9>(hh);
    case 10: return hh ? pick_cfg<10, true>() : KernelCfg{};
    default: return KernelCfg{};
  }
}
}  // namespace dvqls
