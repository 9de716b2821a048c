// launch.h - host-side interface between dvqls_api.cu (the C ABI) and the kernel translation
// units.  Each k_*.cu instantiates its kernel templates once and exports, through the functions
// below, either the kernel's launch description (KernelCfg: address, block, dynamic SMEM; the
// API launches it with cudaLaunchKernel / cudaLaunchKernelExC) or a small launcher.  No device
// code is visible from here, so the TUs compile in parallel (build.py).
#pragma once

#include "types.h"

namespace dvqls {

// ---- k_reg_lo.cu (n = 1..6) / k_reg_hi.cu (n = 7..10): complex register-path kernel
// hadamard_kernel<n, W, HH> (kernels.cuh), one circuit per thread group, x in SMEM
KernelCfg reg_cfg_lo(int n, bool householder);
KernelCfg reg_cfg_hi(int n, bool householder);

// ---- k_plane.cu: the n = 10 uniform-b real-plane kernel (plane.cuh) and the SMEM prefixes
KernelCfg plane_cfg();   // plane_kernel<20>; SMEM sized for this device's dynamic-SMEM base
KernelCfg plane2_cfg();  // plane2_kernel: two circuits in flight per warp (plane2.cuh)
// prefix x = V(theta)|0> for n <= 12, one CTA per theta (a2): args (layers, entangler, thetas, x)
// when !with_n, else (n, layers, entangler, thetas, x)
struct PrefixCfg {
  const void* fn = nullptr;
  int threads = 0;
  size_t smem = 0;
  bool with_n = false;
  int cluster = 0;  // > 0: thread-block-cluster prefix (prefix_cluster.cuh), grid (cluster, K) with
                    // cluster dims (cluster, 1, 1), args (layers, entangler, thetas, x)
};
PrefixCfg prefix_cfg(int n, int layers, bool cluster = true);
void launch_finalize(const double* ep, int K, int n, double* out, cudaStream_t st);

// ---- k_onchip.cu: n = 11, 12 uniform b (onchip_plane.cuh) + its planar copy of x
KernelCfg onchip_cfg(int n, bool x_in_smem = false);
void launch_to_planar4(const double2* x, uint32_t N, uint32_t K, double* xq, cudaStream_t st);

// ---- k_stream_c.cu: complex streaming kernels for Householder U_b, n = 11..24 (stream.cuh):
// n <= 12 one SMEM tile (stream_hadamard_kernel), n >= 13 scratch-free three-sweep kernel
// (stream_hh_kernel); grid (G, K)
KernelCfg stream_hh_cfg(int n);

// ---- k_stream_p.cu: n >= 13 uniform b (stream_plane.cuh), global-memory prefix (tile.cuh)
KernelCfg stream_plane_cfg(bool staged);
void launch_to_planar(const double2* x, uint32_t N, uint32_t K, double* xp, cudaStream_t st);
// V(theta_k)|0> for k < K in global memory (x: K x 2^n), ping-pong buffer x2 (2^n), gate table
// gates (2 n layers); returns a cudaError_t
int launch_prefix_global(int n, int layers, int entangler, int K, const double* thetas, double2* x, double2* x2,
                         double2* gates, cudaStream_t st);
int prefix_global_launches(int n, int layers);

// ---- k_aux.cu: NEXT-2 (pauli.cuh), NEXT-3 (global.cuh), parameter-shift helpers (shift.cuh)
const void* pauli_expect_fn();
int pauli_warps();
void launch_pauli_scatter(const double2* e, const uint32_t* task, int64_t c0, int64_t C, double* out,
                          cudaStream_t st);
void launch_overlap(dim3 grid, const double2* x, int n, const PauliTerm* tab, const double2* coef, const double2* b,
                    int L, const double* cost5, double* beta, double* out6, unsigned* counter, cudaStream_t st);
// theta_out[(2p + s) * P + i] = theta[i] + (i == p ? (s ? -pi/2 : +pi/2) : 0) for p < P, then the
// unshifted theta as row 2P (Alg. 1 Step 4c's cost at theta itself)
void launch_shift_thetas(const double* theta, int P, double* theta_out, cudaStream_t st);
// parameter-shift gradient of C = 1/2 - Re E / (2 n Re Psi) from the 2P + 1 rows (C, E, Psi)
// of res5: out[0] = C(theta), out[1 + p] = dC/dtheta_p, out[1 + P + 0..3] = (E, Psi)(theta)
void launch_shift_grad(const double* res5, int P, int n, double* out, cudaStream_t st);

}  // namespace dvqls
