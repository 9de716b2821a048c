// k_stream_c.cu - complex streaming Hadamard-test kernels for Householder U_b, n = 11..24
// (stream.cuh): n = 11, 12 one SMEM tile per circuit, n >= 13 three read-only sweeps.
#include "launch.h"
#include "stream.cuh"

namespace dvqls {

KernelCfg stream_hh_cfg(int n) {
  KernelCfg k;
  k.groups = 1;
  if (n == 11) {
    k.fn = (const void*)&stream::stream_hadamard_kernel<11, true>;
    k.warps = stream::TS<11>::THREADS / 32;
    k.smem = sizeof(double2) * stream::TS<11>::TN;
  } else if (n == 12) {
    k.fn = (const void*)&stream::stream_hadamard_kernel<12, true>;
    k.warps = stream::TS<12>::THREADS / 32;
    k.smem = sizeof(double2) * stream::TS<12>::TN;
  } else if (n >= 13 && n <= 24) {
    k.fn = (const void*)&stream::stream_hh_kernel<12>;
    k.warps = stream::TS<12>::THREADS / 32;
    k.smem = 0;
  }
  return k;
}

}  // namespace dvqls
