// k_reg_lo.cu - complex register-path Hadamard-test kernels, n = 1..6 (kernels.cuh).
#include "k_reg.inc"

namespace dvqls {
KernelCfg reg_cfg_lo(int n, bool hh) {
  switch (n) {
    case 1: return cfg_n<1>(hh);
    case 2: return cfg_n<2>(hh);
    case 3: return cfg_n<3>(hh);
    case 4: return cfg_n<4>(hh);
    case 5: return cfg_n<5>(hh);
    case 6: return cfg_n<6>(hh);
    default: return KernelCfg{};
  }
}
}  // namespace dvqls
