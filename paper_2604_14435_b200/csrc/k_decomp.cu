// k_decomp.cu - NEXT-4: Pauli decomposition + pruning of a dense A on the GPU
// (Alg. 1 Steps 1-2; FWHT decomposition P:379; pruning P:490).  Host driver of the
// decomp.cuh kernels and the C-ABI entry points dvqls_decompose / dvqls_pauli_coefficients
// (declared in include/dvqls.h).  Context-free: allocates its own device buffers per call.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "../../include/dvqls.h"
#include "decomp.cuh"

using namespace dvqls;

// ---- NEXT-4: Pauli decomposition + pruning (decomp.cuh) ---------------------------------------
namespace {
struct DecompBufs {
  uint64_t* kq = nullptr;  // global-sort keys (more than SORT_MAX candidates)
  uint64_t* kl = nullptr;
  uint32_t* ki = nullptr;
  unsigned long long* kept = nullptr;
  double2* A = nullptr;
  double2* C = nullptr;
  double* sq = nullptr;
  double* norm = nullptr;
  double* thr0 = nullptr;
  double* fro = nullptr;
  unsigned long long* count = nullptr;
  unsigned long long* outL = nullptr;
  uint64_t* idx = nullptr;
  double2* oc = nullptr;
  char* os = nullptr;
  cudaStream_t st = nullptr;
  size_t nfro = 0;
  ~DecompBufs() {
    cudaFree(A); cudaFree(C); cudaFree(sq); cudaFree(norm); cudaFree(count); cudaFree(idx); cudaFree(oc); cudaFree(os);
    cudaFree(thr0); cudaFree(fro); cudaFree(outL); cudaFree(kq); cudaFree(kl); cudaFree(ki); cudaFree(kept);
    if (st) cudaStreamDestroy(st);
  }
};
thread_local std::string g_decomp_err;

int decomp_fail(int code, const char* msg) {
  g_decomp_err = msg;
  return code;
}

// NEXT-4 device pass over the XOR diagonals of A (decomp.cuh).
// MODE 0: all coefficients into C;  MODE 1: candidates + per-row |c|^2.
template <int NB, int MODE>
int launch_rows_reg(DecompBufs& b, uint64_t cap) {
  const void* fn = (const void*)&decomp::fwht_rows_reg_kernel<NB, MODE>;
  const int smem = int(sizeof(double2) << NB);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
    return decomp_fail(DVQLS_E_CUDA, "fwht_rows_reg_kernel smem");
  decomp::fwht_rows_reg_kernel<NB, MODE><<<1u << NB, 1u << (NB - 4), smem, b.st>>>(b.A, b.C, b.sq, b.thr0, cap,
                                                                                  b.count, b.idx);
  return DVQLS_OK;
}
template <int MODE>
int launch_rows(DecompBufs& b, int n, uint64_t cap) {
  switch (n) {
    case 9: return launch_rows_reg<9, MODE>(b, cap);
    case 10: return launch_rows_reg<10, MODE>(b, cap);
    case 11: return launch_rows_reg<11, MODE>(b, cap);
    case 12: return launch_rows_reg<12, MODE>(b, cap);
    case 13: return launch_rows_reg<13, MODE>(b, cap);
    default: break;
  }
  const unsigned N = 1u << n;
  if (cudaFuncSetAttribute((const void*)&decomp::fwht_rows_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(sizeof(double2) << n)))
    return decomp_fail(DVQLS_E_CUDA, "fwht_rows_kernel smem");
  decomp::fwht_rows_kernel<MODE><<<N, decomp::THREADS, sizeof(double2) * N, b.st>>>(b.A, n, b.C, b.sq, b.thr0, cap,
                                                                                  b.count, b.idx);
  return DVQLS_OK;
}

// A -> device in row chunks, |A|^2 of each chunk summed as it lands (pruning only); write_c: every
// coefficient into C, else: Parseval candidate bound, one candidate pass over the XOR diagonals,
// exact norm in the sort (decomp.cuh).  *ev0 is recorded after the upload.
int decomp_transform(DecompBufs& b, int n, const double* A_host, int device, bool write_c, double eps = 0.0,
                     cudaEvent_t* ev0 = nullptr) {
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return decomp_fail(DVQLS_E_CUDA, "cudaSetDevice");
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10)
    return decomp_fail(DVQLS_E_CUDA, "libdvqls is built for sm_100a only");
  const size_t N = size_t(1) << n, NN = N * N;
  const uint32_t fro_rows = uint32_t(std::min<size_t>(N, 8));  // rows per |A|^2 partial
  const size_t nfro = N / fro_rows;
  const uint64_t cap = decomp::SORT_MAX;
  if (cudaStreamCreateWithFlags(&b.st, cudaStreamNonBlocking) || cudaMalloc((void**)&b.A, sizeof(double2) * NN) ||
      cudaMalloc((void**)&b.C, sizeof(double2) * (write_c ? NN : size_t(cap))) ||
      cudaMalloc((void**)&b.sq, sizeof(double) * N) || cudaMalloc((void**)&b.norm, sizeof(double)) ||
      cudaMalloc((void**)&b.thr0, sizeof(double)) || cudaMalloc((void**)&b.fro, sizeof(double) * nfro) ||
      cudaMalloc((void**)&b.count, sizeof(unsigned long long)) ||
      cudaMalloc((void**)&b.outL, sizeof(unsigned long long)))
    return decomp_fail(DVQLS_E_CUDA, "cudaMalloc failed (decomposition)");
  if (!write_c && (cudaMalloc((void**)&b.idx, sizeof(uint64_t) * cap) ||
                   cudaMalloc((void**)&b.oc, sizeof(double2) * cap) || cudaMalloc((void**)&b.os, size_t(cap) * n)))
    return decomp_fail(DVQLS_E_CUDA, "cudaMalloc failed (pruning)");
  // upload in chunks of ~32 MB of whole row blocks; after each chunk its |A|^2 partials
  const size_t chunk_rows = std::max<size_t>(fro_rows, ((size_t(32) << 20) / (16 * N)) / fro_rows * fro_rows);
  const double2* Ah = reinterpret_cast<const double2*>(A_host);
  for (size_t r0 = 0; r0 < N; r0 += chunk_rows) {
    const size_t rows = std::min(chunk_rows, N - r0);
    if (cudaMemcpyAsync(b.A + r0 * N, Ah + r0 * N, sizeof(double2) * rows * N, cudaMemcpyHostToDevice, b.st))
      return decomp_fail(DVQLS_E_CUDA, "copy of A failed");
    if (!write_c)
      decomp::fro_rows_kernel<<<unsigned(rows / fro_rows), 256, 0, b.st>>>(b.A, uint32_t(N), uint32_t(r0), fro_rows,
                                                                           b.fro);
  }
  if (ev0 && (cudaEventCreate(ev0) || cudaEventRecord(*ev0, b.st))) return decomp_fail(DVQLS_E_CUDA, "event");
  int rc;
  if (write_c) {
    rc = launch_rows<0>(b, n, 0);
  } else {
    decomp::prenorm_kernel<<<1, 256, 0, b.st>>>(b.fro, uint32_t(nfro), uint32_t(N), eps, b.thr0, b.count);
    rc = launch_rows<1>(b, n, cap);  // the exact norm is formed inside sort_emit_kernel
    b.nfro = nfro;
  }
  if (rc) return rc;
  if (cudaGetLastError()) return decomp_fail(DVQLS_E_CUDA, "decomposition kernel launch failed");
  return DVQLS_OK;
}
}  // namespace

extern "C" {

int dvqls_pauli_coefficients(int n, const double* A, double* out_coeffs, int device) {
  g_decomp_err.clear();
  if (n < 1 || n > 13 || !A || !out_coeffs) return decomp_fail(DVQLS_E_ARG, "n must be in [1, 13], non-NULL buffers");
  DecompBufs b;
  int rc = decomp_transform(b, n, A, device, true);
  if (rc) return rc;
  const size_t NN = (size_t(1) << n) * (size_t(1) << n);
  if (cudaMemcpyAsync(out_coeffs, b.C, sizeof(double2) * NN, cudaMemcpyDeviceToHost, b.st) ||
      cudaStreamSynchronize(b.st))
    return decomp_fail(DVQLS_E_CUDA, "decomposition failed");
  return DVQLS_OK;
}

int dvqls_decompose(int n, const double* A, double eps, int64_t max_terms, char* out_paulis, double* out_coeffs,
                    int64_t* out_L, double* out_norm, int device, float* out_ms) {
  g_decomp_err.clear();
  if (n < 1 || n > 13 || !A || !out_L || (max_terms > 0 && (!out_paulis || !out_coeffs)) || max_terms < 0 ||
      !(eps >= 0.0 && eps < 1.0))
    return decomp_fail(DVQLS_E_ARG, "n in [1, 13], 0 <= eps < 1, non-NULL outputs");
  DecompBufs b;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = decomp_transform(b, n, A, device, false, eps, out_ms ? &e0 : nullptr);
  if (rc) return rc;
  if (cudaFuncSetAttribute((const void*)&decomp::sort_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(decomp::SORT_SMEM)))
    return decomp_fail(DVQLS_E_CUDA, "sort kernel smem");
  decomp::sort_emit_kernel<<<1, decomp::THREADS, decomp::SORT_SMEM, b.st>>>(b.C, n, b.idx, b.count, b.sq, b.norm,
                                                                             eps, b.oc, b.os, b.outL);
  if (out_ms && (cudaEventCreate(&e1) || cudaEventRecord(e1, b.st)))
    return decomp_fail(DVQLS_E_CUDA, "event");
  unsigned long long cand = 0, L = 0;
  double norm = 0.0;
  if (cudaGetLastError() || cudaMemcpyAsync(&cand, b.count, sizeof cand, cudaMemcpyDeviceToHost, b.st) ||
      cudaMemcpyAsync(&L, b.outL, sizeof L, cudaMemcpyDeviceToHost, b.st) ||
      cudaMemcpyAsync(&norm, b.norm, sizeof norm, cudaMemcpyDeviceToHost, b.st) || cudaStreamSynchronize(b.st))
    return decomp_fail(DVQLS_E_CUDA, "pruning failed");
  if (out_norm) *out_norm = norm;
  if (cand > decomp::SORT_MAX) {
    // more candidates than the one-CTA sort holds: compact them all (second candidate pass with
    // buffers of the counted size) and sort globally (bitonic network, the same total order)
    const size_t N = size_t(1) << n;
    uint64_t P = 1;
    while (P < cand) P <<= 1;
    cudaFree(b.C); cudaFree(b.idx); cudaFree(b.oc); cudaFree(b.os);
    b.C = nullptr; b.idx = nullptr; b.oc = nullptr; b.os = nullptr;
    if (cudaMalloc((void**)&b.C, sizeof(double2) * cand) || cudaMalloc((void**)&b.idx, sizeof(uint64_t) * cand) ||
        cudaMalloc((void**)&b.oc, sizeof(double2) * cand) || cudaMalloc((void**)&b.os, size_t(cand) * n) ||
        cudaMalloc((void**)&b.kq, sizeof(uint64_t) * P) || cudaMalloc((void**)&b.kl, sizeof(uint64_t) * P) ||
        cudaMalloc((void**)&b.ki, sizeof(uint32_t) * P) || cudaMalloc((void**)&b.kept, sizeof(unsigned long long)))
      return decomp_fail(DVQLS_E_CUDA, "cudaMalloc failed (large candidate set)");
    decomp::prenorm_kernel<<<1, 256, 0, b.st>>>(b.fro, uint32_t(b.nfro), uint32_t(N), eps, b.thr0, b.count);
    if ((rc = launch_rows<1>(b, n, cand))) return rc;
    decomp::norm_kernel<<<1, decomp::THREADS, 0, b.st>>>(b.sq, n, b.norm);
    cudaMemsetAsync(b.kept, 0, sizeof(unsigned long long), b.st);
    const unsigned grid = unsigned(std::min<uint64_t>(4096, (P + 255) / 256));
    decomp::keys_kernel<<<grid, 256, 0, b.st>>>(b.C, b.idx, cand, P, n, b.norm, eps, b.kq, b.kl, b.ki, b.kept);
    for (uint64_t k = 2; k <= P; k <<= 1)
      for (uint64_t j = k >> 1; j > 0; j >>= 1)
        decomp::bitonic_step_kernel<<<grid, 256, 0, b.st>>>(b.kq, b.kl, b.ki, P, k, j);
    decomp::emit_kernel<<<grid, 256, 0, b.st>>>(b.C, b.idx, b.ki, b.kept, n, b.oc, b.os, b.outL);
    if (out_ms && (cudaEventRecord(e1, b.st))) return decomp_fail(DVQLS_E_CUDA, "event");
    if (cudaGetLastError() || cudaMemcpyAsync(&L, b.outL, sizeof L, cudaMemcpyDeviceToHost, b.st) ||
        cudaMemcpyAsync(&norm, b.norm, sizeof norm, cudaMemcpyDeviceToHost, b.st) || cudaStreamSynchronize(b.st))
      return decomp_fail(DVQLS_E_CUDA, "global sort failed");
    if (out_norm) *out_norm = norm;
  }
  *out_L = int64_t(L);
  if (int64_t(L) > max_terms) return decomp_fail(DVQLS_E_ARG, "max_terms too small (*out_L holds the count)");
  if (L > 0 && (cudaMemcpyAsync(out_coeffs, b.oc, sizeof(double2) * L, cudaMemcpyDeviceToHost, b.st) ||
                cudaMemcpyAsync(out_paulis, b.os, size_t(L) * n, cudaMemcpyDeviceToHost, b.st) ||
                cudaStreamSynchronize(b.st)))
    return decomp_fail(DVQLS_E_CUDA, "sort/emit failed");
  if (out_ms) {  // device time from after the H2D copy of A to the end of sort/emit
    cudaEventElapsedTime(out_ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return DVQLS_OK;
}

const char* dvqls_decompose_error(void) { return g_decomp_err.c_str(); }

}  // extern "C"
