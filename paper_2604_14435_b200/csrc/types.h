// types.h - plain structs shared by the host side (dvqls_api.cu) and the sm_100a kernels.
//
// No device code here: dvqls_api.cu includes only this file and launch.h, so the kernel
// templates are instantiated once, in their own translation units (k_*.cu), which nvcc
// compiles in parallel.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace dvqls {

// A Pauli string as an operator on basis states:
//   P|j> = i^{ny} (-1)^{popcount(j & zm)} |j ^ xm>,  big-endian masks (reading 9)
struct PauliTerm {
  uint32_t xm, zm;
  int32_t ny;
  uint32_t wpar;  // bit r = popcount(r & (zm >> TB)) & 1: register-part sign word (host-built)
};

// Fused cross-rank reduction over NVLink peer memory (a10, Alg. 1 Step 4c P:461-463).
// Every rank owns a symmetric buffer, IPC-mapped into all peers:
//   double   slot[2][world][KB][4]   (E, Psi) written by rank r for theta slot k
//   uint64_t flag[2][world][KB]      epoch of that write
// epochs[k] (device memory, one per theta slot) is advanced by the CTA that reduces slot k, so
// the launch parameters are identical from call to call (CUDA-graph replayable) and all ranks,
// making the same calls, agree on it.  A peer that has not published within timeout_ns sets
// *err (sticky; the host maps it to DVQLS_E_NCCL) and the slot's cost becomes NaN.
struct P2PArgs {
  int world, rank, KB;
  unsigned long long* epochs;  // KB per-slot epoch counters (device)
  char* const* peers;          // world device pointers (peers[rank] = own buffer)
  unsigned long long timeout_ns;
  unsigned* err;               // sticky error word (device)
};

namespace pauli {
struct Obs {
  uint32_t m, z;  // x-mask, z-mask (big-endian index bits)
};
}  // namespace pauli

// Launch description of a Hadamard-test kernel (host side).
struct KernelCfg {
  const void* fn = nullptr;
  int warps = 0;      // threads per CTA / 32
  size_t smem = 0;    // dynamic shared memory per CTA
  int groups = 0;     // circuit groups per CTA (flat-grid kernels)
};

}  // namespace dvqls
