// global.cuh - NEXT-3: the global VQLS cost (Eq. 1)
//     C_G = 1 - |<b|A|x>|^2 / <x|A^+A|x>,   <b|A|x> = sum_l c_l beta_l,
//     beta_l = <0| U_b^+ A_l V(theta) |0> = <b| A_l |x>
// from the L overlap Hadamard tests (Re and Im circuits of each l) and the local cost's
// denominator sum Re Psi = <x|A^+A|x> (Alg. 1 Step 4b) of the same call.
//
// Overlap circuit l (ancilla-|1> branch only, as in kernels.cuh): the |0> branch stays |0^n>
// and the |1> branch is U_b^+ A_l x, so <Z_anc> = Re(kappa <0^n| U_b^+ A_l x>) = Re(kappa
// <b| A_l x>) with kappa = 1 (Re) or -i (Im).  The amplitude <0^n|U_b^+|phi> is read
// directly as the dot product b^+ phi (U_b|0> = b for both U_b constructions, reading 5),
// so one circuit is one signed gather of x (c-A_l) and one reduction of 2^n terms.
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace glob {

constexpr int THREADS = 256;

// grid (L, K): CTA (l, k) computes beta_l of theta k; the last CTA of theta k (ticket)
// combines them in fixed l order with Re Psi from cost5[k] into C_G.
// b == NULL: uniform b (b_i = 2^{-n/2}).
// out6[k] = (C_L, Re E, Im E, Re Psi, Im Psi, C_G) (cost5[k] copied through).
__global__ void __launch_bounds__(THREADS)
overlap_kernel(const double2* __restrict__ x_all, int n, const PauliTerm* __restrict__ tab,
               const double2* __restrict__ coef, const double2* __restrict__ b, int L,
               const double* __restrict__ cost5, double* __restrict__ beta, double* __restrict__ out6,
               unsigned* __restrict__ counter) {
  __shared__ double red[2][THREADS / 32];
  __shared__ unsigned s_last;
  const int l = blockIdx.x, kth = blockIdx.y;
  const uint32_t N = 1u << n;
  const double2* __restrict__ x = x_all + (size_t)kth * N;
  const PauliTerm T = tab[l];
  // sum_j conj(b_{j ^ m}) (-1)^{popcount(j & z)} x_j, then the i^{n_Y} phase
  double re = 0.0, im = 0.0;
  for (uint32_t j = threadIdx.x; j < N; j += THREADS) {
    const double2 xv = x[j];
    const double2 bv = b ? b[j ^ T.xm] : make_double2(1.0, 0.0);
    const uint32_t f = (uint32_t(__popc(j & T.zm)) & 1u) << 31;
    re += flip(fma(bv.x, xv.x, bv.y * xv.y), f);
    im += flip(fma(bv.x, xv.y, -bv.y * xv.x), f);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, off);
    im += __shfl_xor_sync(0xffffffffu, im, off);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = re; red[1][w] = im; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0, i = 0.0;
    for (int q = 0; q < THREADS / 32; ++q) { r += red[0][q]; i += red[1][q]; }
    if (!b) {
      const double s = rsqrt(double(N));  // 2^{-n/2}: exact for even n, correctly rounded otherwise
      r *= s; i *= s;
    }
    // i^{n_Y}
    const int q = T.ny & 3;
    const double br = q == 0 ? r : q == 1 ? -i : q == 2 ? -r : i;
    const double bi = q == 0 ? i : q == 1 ? r : q == 2 ? -i : -r;
    double* o = beta + ((size_t)kth * L + l) * 2;
    o[0] = br;
    o[1] = bi;
    __threadfence();
    s_last = (atomicAdd(counter + kth, 1u) == unsigned(L) - 1u) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  double sr = 0.0, si = 0.0;
  for (int ll = 0; ll < L; ++ll) {  // fixed order
    const double2 c = coef[ll];
    const double br = __ldcg(beta + ((size_t)kth * L + ll) * 2), bi = __ldcg(beta + ((size_t)kth * L + ll) * 2 + 1);
    sr += c.x * br - c.y * bi;
    si += c.x * bi + c.y * br;
  }
  const double* c5 = cost5 + (size_t)kth * 5;
  double* o = out6 + (size_t)kth * 6;
  for (int q = 0; q < 5; ++q) o[q] = c5[q];
  const double RePsi = c5[3];
  o[5] = RePsi <= 1e-12 ? __longlong_as_double(0x7ff8000000000000ll) : 1.0 - (sr * sr + si * si) / RePsi;
  counter[kth] = 0u;
}

}  // namespace glob
}  // namespace dvqls
