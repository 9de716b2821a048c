// k_aux.cu - NEXT-2 Pauli fast path (pauli.cuh), NEXT-3 global-cost overlaps (global.cuh) and the
// parameter-shift gradient helpers (shift.cuh).
#include <algorithm>

#include "global.cuh"
#include "launch.h"
#include "pauli.cuh"
#include "shift.cuh"

namespace dvqls {

const void* pauli_expect_fn() { return (const void*)&pauli::pauli_expect_kernel; }
int pauli_warps() { return pauli::WARPS; }

void launch_pauli_scatter(const double2* e, const uint32_t* task, int64_t c0, int64_t C, double* out,
                          cudaStream_t st) {
  pauli::pauli_scatter_kernel<<<296, 256, 0, st>>>(e, task, c0, C, out);
}

void launch_overlap(dim3 grid, const double2* x, int n, const PauliTerm* tab, const double2* coef, const double2* b,
                    int L, const double* cost5, double* beta, double* out6, unsigned* counter, cudaStream_t st) {
  glob::overlap_kernel<<<grid, glob::THREADS, 0, st>>>(x, n, tab, coef, b, L, cost5, beta, out6, counter);
}

void launch_shift_thetas(const double* theta, int P, double* theta_out, cudaStream_t st) {
  const int64_t total = int64_t(2 * P + 1) * P;
  shift::shift_thetas_kernel<<<unsigned(std::min<int64_t>(296, (total + 255) / 256)), 256, 0, st>>>(theta, P,
                                                                                                     theta_out);
}

void launch_shift_grad(const double* res5, int P, int n, double* out, cudaStream_t st) {
  shift::shift_grad_kernel<<<(P + 255) / 256, 256, 0, st>>>(res5, P, n, out);
}

}  // namespace dvqls
