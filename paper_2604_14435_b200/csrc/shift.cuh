// shift.cuh - parameter-shift gradient of the local cost (NEXT-1 with 2P shift points; P:13
// "parameter-shift gradients" as the multi-circuit workload; SURVEY §8(c) reading 23).
//
// Every parameter of V(theta) enters through exactly one exp(-i theta sigma / 2) (reading 7), so
// every Hadamard-test value f, hence Re E and Re Psi (fixed linear combinations of them), obeys
//     df/dtheta_p = [f(theta + pi/2 e_p) - f(theta - pi/2 e_p)] / 2           (exact)
// and C = 1/2 - Re E / (2 n Re Psi) (Alg. 1 Step 4c) by the quotient rule:
//     dC/dtheta_p = -(dReE_p Re Psi - Re E dRePsi_p) / (2 n Re Psi^2).
// The 2P shifted thetas and theta itself are evaluated as one batch of the circuit path.
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace shift {

// rows 2p (+pi/2 on parameter p), 2p + 1 (-pi/2), row 2P: theta unshifted
__global__ void shift_thetas_kernel(const double* __restrict__ theta, int P, double* __restrict__ out) {
  const int64_t total = int64_t(2 * P + 1) * P;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int row = int(i / P), col = int(i - int64_t(row) * P);
    double v = theta[col];
    if (row < 2 * P && (row >> 1) == col) v += (row & 1) ? -1.5707963267948966 : 1.5707963267948966;
    out[i] = v;
  }
}

// res5: 2P + 1 rows of (C, Re E, Im E, Re Psi, Im Psi);  out: C, dC/dtheta[P], (E, Psi) at theta
__global__ void shift_grad_kernel(const double* __restrict__ res5, int P, int n, double* __restrict__ out) {
  const double* r0 = res5 + size_t(2 * P) * 5;
  const double E0 = r0[1], Psi0 = r0[3];
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) {
    const double* rp = res5 + size_t(2 * p) * 5;
    const double* rm = rp + 5;
    const double dE = 0.5 * (rp[1] - rm[1]), dPsi = 0.5 * (rp[3] - rm[3]);
    out[1 + p] = Psi0 <= 1e-12 ? nan_dev() : -(dE * Psi0 - E0 * dPsi) / (2.0 * double(n) * Psi0 * Psi0);
  }
  if (p == 0) {
    out[0] = r0[0];
    out[1 + P + 0] = r0[1];
    out[1 + P + 1] = r0[2];
    out[1 + P + 2] = r0[3];
    out[1 + P + 3] = r0[4];
  }
}

}  // namespace shift
}  // namespace dvqls
