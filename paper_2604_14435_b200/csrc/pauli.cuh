// pauli.cuh - NEXT-2: the algebraic fast path, FLAGGED and reported
// separately from the circuit path (it is never the headline circuits/s).
//
// For uniform b, U_b Z_j U_b^+ = H^n Z_j H^n = X_j, so every Hadamard-test term of Eq. 4
// is the expectation of ONE Pauli string up to a phase:
//     <x| A_l X_j A_k |x>  (numerator),   <x| A_l A_k |x>  (denominator)
//     = i^q * e(m, z),  e(m, z) = sum_i conj(x_{i ^ m}) (-1)^{popcount(i & z)} x_i
// The host (dvqls_create) multiplies the Pauli strings symbolically, deduplicates the
// resulting (m, z) over all (n+1)L^2 tasks and folds c_l^* c_k i^q into two complex weights
// per distinct observable (W^E, W^Psi).  Per theta the device then evaluates each distinct
// e(m, z) once (O(2^n) each) and E = sum_P W^E_P e_P, Psi = sum_P W^Psi_P e_P.  Re/Im of one
// task come from the same complex e.  This is exactly the "cancelling gates across the
// U_b ... U_b^+ sandwich, deduplicating equal Pauli observables, sharing one branch between
// Re and Im" that SURVEY §8(d) excludes from the headline.
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace pauli {

// struct Obs (x-mask, z-mask of one distinct observable): types.h

constexpr int WARPS = 8;

// One warp per observable, observables [d0, d1) split contiguously over the CTAs (x staged
// in SMEM when it fits, else read through L1/L2).  Per theta (blockIdx.y): e_d -> out_e
// (when out_e != NULL) and the CTA's fixed-order partial (Re E, Im E, Re Psi, Im Psi).
__global__ void __launch_bounds__(WARPS * 32)
pauli_expect_kernel(const double2* __restrict__ x_all, int n, const Obs* __restrict__ obs,
                    const double2* __restrict__ wE, const double2* __restrict__ wP, int64_t d0, int64_t d1,
                    int64_t D, double2* __restrict__ out_e, double* __restrict__ partials, int with_cost,
                    double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p, int stage_x) {
  extern __shared__ double2 xs_dyn[];
  __shared__ double wsum[WARPS][4];
  const int kth = blockIdx.y;
  const uint32_t N = 1u << n;
  const double2* __restrict__ xg = x_all + (size_t)kth * N;
  if (stage_x) {
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) xs_dyn[i] = xg[i];
    __syncthreads();
  }
  const double2* __restrict__ x = stage_x ? xs_dyn : xg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x, R = d1 - d0;
  const int64_t cb = d0 + (int64_t)blockIdx.x * R / G, ce = d0 + ((int64_t)blockIdx.x + 1) * R / G;
  double sE0 = 0.0, sE1 = 0.0, sP0 = 0.0, sP1 = 0.0;
  for (int64_t d = cb + warp; d < ce; d += WARPS) {
    const Obs o = obs[d];
    double re = 0.0, im = 0.0;
    for (uint32_t i = lane; i < N; i += 32) {
      const double2 a = x[i ^ o.m], b = x[i];
      const uint32_t f = (uint32_t(__popc(i & o.z)) & 1u) << 31;
      // conj(a) b (-1)^{i.z}
      re += flip(fma(a.x, b.x, a.y * b.y), f);
      im += flip(fma(a.x, b.y, -a.y * b.x), f);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, off);
      im += __shfl_xor_sync(0xffffffffu, im, off);
    }
    if (lane == 0) {
      if (out_e) out_e[(size_t)kth * D + d] = make_double2(re, im);
      const double2 we = wE[d], wp = wP[d];
      sE0 += we.x * re - we.y * im; sE1 += we.x * im + we.y * re;
      sP0 += wp.x * re - wp.y * im; sP1 += wp.x * im + wp.y * re;
    }
  }
  if (lane == 0) { wsum[warp][0] = sE0; wsum[warp][1] = sE1; wsum[warp][2] = sP0; wsum[warp][3] = sP1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int w = 0; w < WARPS; ++w) { a0 += wsum[w][0]; a1 += wsum[w][1]; a2 += wsum[w][2]; a3 += wsum[w][3]; }
    double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
    o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3;
  }
  if (red_out) finish_partials(partials, G, kth, n, with_cost, red_out, counter, p2p.world > 1 ? &p2p : nullptr);
}

// terms of circuits [c0, c0 + C): task t = c / 2 -> (observable, phase q) packed as
// (d << 2) | q; value Re(i^q e_d) (part 0) or Im(i^q e_d) (part 1)
__global__ void pauli_scatter_kernel(const double2* __restrict__ e, const uint32_t* __restrict__ task, int64_t c0,
                                     int64_t C, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = c0 + i;
    const uint32_t tq = task[c >> 1];
    const double2 v = e[tq >> 2];
    const int q = int(tq & 3u);
    // i^q v: q=0 (re, im), 1 (-im, re), 2 (-re, -im), 3 (im, -re)
    const double r = q == 0 ? v.x : q == 1 ? -v.y : q == 2 ? -v.x : v.y;
    const double m = q == 0 ? v.y : q == 1 ? v.x : q == 2 ? -v.y : -v.x;
    out[i] = (c & 1) ? m : r;
  }
}

}  // namespace pauli
}  // namespace dvqls
