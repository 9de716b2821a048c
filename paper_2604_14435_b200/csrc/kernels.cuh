// kernels.cuh - sm_100a kernels of the D-VQLS hot path (arXiv 2604.14435).
//
//   prefix_kernel    SURVEY §8(a) a2: x = V(theta)|0^n> once per theta
//   hadamard_kernel  a3-a9: every Hadamard-test circuit of the rank's block,
//                    one circuit per thread group, state in registers, x in SMEM,
//                    coefficient-weighted partial sums fused in (Alg. 1 4a-4b)
//
// Only the ancilla-|1> branch of each Hadamard test is simulated: every gate
// after the first ancilla H is controlled on the ancilla (or is U_b / U_b^+
// applied controlled), so the |0> branch stays x/sqrt2 and
//     <Z_anc> = Re( kappa <x| A_l U_b Z_j U_b^+ A_k |x> ),  kappa = 1 (Re), -i (Im, S^+)
// (P:367).  Gates are fused within a circuit: the controlled Pauli
// strings become signed gathers, U_b = H^{(x)n} becomes an unnormalised
// in-register FWHT (2 n N DADD), Z_j a sign flip, and the ancilla
// normalisations and i^{n_Y} phases are folded into one final scale.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "types.h"

namespace dvqls {

// Dynamic shared memory of the Hadamard-test kernel.  Accesses are written as
// byte offsets from this symbol so the compiler folds the base into the
// LDS/STS immediate and the per-access address work is a single XOR.
extern __shared__ double2 dvqls_smem[];

// Programmatic dependent launch (sm_90+): the prefix lets the Hadamard kernel be scheduled while
// it runs, and the Hadamard kernel waits for the prefix's completion (and memory flush) before it
// touches anything.  Both are no-ops when the launch does not carry the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ double2 lds2(uint32_t off) {
  return *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(dvqls_smem) + off);
}
__device__ __forceinline__ void sts2(uint32_t off, double2 v) {
  *reinterpret_cast<double2*>(reinterpret_cast<char*>(dvqls_smem) + off) = v;
}

// sign flip of a double by XOR of the IEEE sign bit (m = 0 or 0x80000000):
// one ALU LOP3 on the high word, no FP64-pipe instruction.
__device__ __forceinline__ double flip(double v, uint32_t m) {
  return __hiloint2double(__double2hiint(v) ^ int(m), __double2loint(v));
}

// ---------------------------------------------------------------------------
// a2: shared ansatz prefix.  One CTA per theta; state in SMEM (n <= 12).
// Each layer applies n fused single-qubit unitaries U_q = Ry(t2) Rz(t1) Ry(t0)
// (within-circuit fusion of the three rotations on one qubit; U_q is in SU(2),
// U = [[a, -conj(b)], [b, conj(a)]], so a gate is two complex numbers), RB
// qubits at a time: every thread holds 2^RB amplitudes in registers (the RB
// index bits of the current qubit group), so a layer is ceil(n/RB) phases of
// load -> RB gates -> store into the other SMEM buffer -> one barrier.  The
// entangling ring is one index permutation (CNOT ring) or one diagonal sign
// (CZ ring), folded into the first load of the next layer (and the final
// write-out) through a precomputed table.
// ---------------------------------------------------------------------------
// SMEM slot of state index i in the prefix: XOR-swizzle of the low 3 bits with bits 3..5,
// so every register-group phase hits 8 distinct 16-byte bank groups per quarter warp
// (without it the phase whose qubits are the low index bits is 2^RB-way conflicted).
__device__ __forceinline__ int pswz(int i) { return i ^ ((i >> 3) & 7); }

template <int RB>
__global__ void __launch_bounds__(512)
prefix_kernel(int n, int layers, int entangler, const double* __restrict__ thetas, double2* __restrict__ x_all) {
  pdl_trigger();
  constexpr int RA = 1 << RB;
  extern __shared__ double2 psm[];
  const int N = 1 << n;
  const int P = 3 * n * layers;
  const int G = n * layers;
  const int T = N >> RB;  // active threads
  double2* bufA = psm;
  double2* bufB = psm + N;
  double2* U = psm + 2 * N;                       // (a, b) per fused gate
  int* perm = reinterpret_cast<int*>(U + 2 * G);  // ring permutation (| sign << 31 for CZ)
  const double* th = thetas + (size_t)blockIdx.x * P;
  const int tid = threadIdx.x;

  for (int g = tid; g < G; g += blockDim.x) {
    double s0, c0, s1, c1, s2, c2;
    sincos(0.5 * th[3 * g + 0], &s0, &c0);
    sincos(0.5 * th[3 * g + 1], &s1, &c1);
    sincos(0.5 * th[3 * g + 2], &s2, &c2);
    // Rz(t1) Ry(t0) = [[e0 c0, -e0 s0], [e1 s0, e1 c0]], e0 = e^{-i t1/2}, e1 = e^{+i t1/2};
    // U = Ry(t2) Rz(t1) Ry(t0): a = U00 = c2 e0 c0 - s2 e1 s0, b = U10 = s2 e0 c0 + c2 e1 s0
    U[2 * g + 0] = make_double2(c1 * (c2 * c0 - s2 * s0), -s1 * (c2 * c0 + s2 * s0));
    U[2 * g + 1] = make_double2(c1 * (s2 * c0 + c2 * s0), s1 * (c2 * s0 - s2 * c0));
  }
  for (int i = tid; i < N; i += blockDim.x) {
    int e = i;
    if (n >= 2) {
      if (entangler == 0) {
        // CNOT ring C_{n-1} ... C_0 (C_q: control q -> target (q+1) mod n, C_0 applied first):
        // new[i] = old[c_0(c_1(...c_{n-1}(i)))]
        int j = i;
        for (int q = n - 1; q >= 0; --q) {
          const int pc = n - 1 - q, pt = n - 1 - ((q + 1) % n);
          if ((j >> pc) & 1) j ^= 1 << pt;
        }
        e = j;
      } else {
        // CZ ring: diagonal (-1)^{sum_q b_q b_{q+1 mod n}}
        int par = 0;
        for (int q = 0; q < n; ++q) par ^= ((i >> (n - 1 - q)) & (i >> (n - 1 - (q + 1) % n))) & 1;
        e = int(unsigned(i) | (unsigned(par) << 31));
      }
    }
    perm[i] = e;
    bufA[pswz(i)] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();

  double2* src = bufA;
  double2* dst = bufB;
  const int phases = (n + RB - 1) / RB;
  for (int layer = 0; layer < layers; ++layer) {
    for (int ph = 0; ph < phases; ++ph) {
      const int b0 = min(RB * ph, n - RB);  // register bits b0 .. b0+RB-1
      if (tid < T) {
        const int base = ((tid >> b0) << (b0 + RB)) | (tid & ((1 << b0) - 1));
        double2 v[RA];
#pragma unroll
        for (int r = 0; r < RA; ++r) {
          const int idx = base | (r << b0);
          if (ph == 0 && layer > 0) {  // previous layer's entangling ring
            const int e = perm[idx];
            double2 a = src[pswz(e & 0x7fffffff)];
            if (e < 0) a = make_double2(-a.x, -a.y);
            v[r] = a;
          } else {
            v[r] = src[pswz(idx)];
          }
        }
#pragma unroll
        for (int rbit = 0; rbit < RB; ++rbit) {
          const int pos = b0 + rbit;
          if (pos >= RB * ph) {  // qubit not yet rotated in this layer
            const int g = layer * n + (n - 1 - pos);
            const double2 ua = U[2 * g + 0], ub = U[2 * g + 1];
#pragma unroll
            for (int r = 0; r < RA; ++r) {
              if (!(r & (1 << rbit))) {
                const double2 x0 = v[r], x1 = v[r | (1 << rbit)];
                // y0 = a x0 - conj(b) x1 ; y1 = b x0 + conj(a) x1
                v[r] = make_double2(fma(ua.x, x0.x, fma(-ua.y, x0.y, fma(-ub.x, x1.x, -ub.y * x1.y))),
                                    fma(ua.x, x0.y, fma(ua.y, x0.x, fma(-ub.x, x1.y, ub.y * x1.x))));
                v[r | (1 << rbit)] = make_double2(fma(ub.x, x0.x, fma(-ub.y, x0.y, fma(ua.x, x1.x, ua.y * x1.y))),
                                                  fma(ub.x, x0.y, fma(ub.y, x0.x, fma(ua.x, x1.y, -ua.y * x1.x))));
              }
            }
          }
        }
#pragma unroll
        for (int r = 0; r < RA; ++r) dst[pswz(base | (r << b0))] = v[r];
      }
      __syncthreads();
      double2* tmp = src; src = dst; dst = tmp;
    }
  }
  double2* x = x_all + (size_t)blockIdx.x * N;
  for (int i = tid; i < N; i += blockDim.x) {
    double2 a;
    if (n >= 2) {
      const int e = perm[i];
      a = src[pswz(e & 0x7fffffff)];
      if (e < 0) a = make_double2(-a.x, -a.y);
    } else {
      a = src[pswz(i)];
    }
    x[i] = a;
  }
}

// ---------------------------------------------------------------------------
// a2 for n <= 10: one amplitude per thread (2^n threads, up to 32 warps).
// Index i is split into LB = min(5, n) lane bits and WB = n - LB warp bits.
//   layout X: i = (w << LB) | l   -> gates on positions [0, LB) are lane bits
//   layout Y: i = (l << WB) | w   -> gates on positions [LB, n) are lane bits
// A gate on a lane bit is one shuffle of the partner amplitude and one complex
// 2-term dot (8 FP64 ops per amplitude, no redundant work); the row of U a thread
// needs (c_self, c_other) is read from a per-gate table by the thread's bit.
// A layer is X-gates, transpose X->Y, Y-gates, transpose Y->X with the
// entangling ring folded into the read, i.e. two barriers per layer.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int tswz(int i) { return i ^ ((i >> 5) & 7); }

template <int NQ>
__global__ void __launch_bounds__(1024)
prefix_lanes_kernel(int layers, int entangler, const double* __restrict__ thetas, double2* __restrict__ x_all) {
  pdl_trigger();
  constexpr int n = NQ;
  constexpr int N = 1 << n;
  constexpr int LB = n < 5 ? n : 5, WB = n - LB;
  extern __shared__ double2 qsm[];
  const int P = 3 * n * layers;
  const int G = n * layers;
  double2* sbuf = qsm;                            // N amplitudes (transposes)
  double2* tabU = qsm + N;                        // 4 per gate: [bit0: c_self, c_other, bit1: ...]
  int* perm = reinterpret_cast<int*>(tabU + 4 * G);
  const double* th = thetas + (size_t)blockIdx.x * P;
  const int tid = threadIdx.x;
  const int l = tid & 31, w = tid >> 5;
  const unsigned full = 0xffffffffu;

  for (int g = tid; g < G; g += blockDim.x) {
    double s0, c0, s1, c1, s2, c2;
    sincos(0.5 * th[3 * g + 0], &s0, &c0);
    sincos(0.5 * th[3 * g + 1], &s1, &c1);
    sincos(0.5 * th[3 * g + 2], &s2, &c2);
    // U = Ry(t2) Rz(t1) Ry(t0) = [[a, -conj(b)], [b, conj(a)]]
    const double2 a = make_double2(c1 * (c2 * c0 - s2 * s0), -s1 * (c2 * c0 + s2 * s0));
    const double2 b = make_double2(c1 * (s2 * c0 + c2 * s0), s1 * (c2 * s0 - s2 * c0));
    tabU[4 * g + 0] = a;                             // bit 0: self  = U00
    tabU[4 * g + 1] = make_double2(-b.x, b.y);       // bit 0: other = U01 = -conj(b)
    tabU[4 * g + 2] = make_double2(a.x, -a.y);       // bit 1: self  = U11 = conj(a)
    tabU[4 * g + 3] = b;                             // bit 1: other = U10 = b
  }
  for (int i = tid; i < N; i += blockDim.x) {
    int e = i;
    if (n >= 2) {
      if (entangler == 0) {
        int j = i;  // new[i] = old[c_0(c_1(...c_{n-1}(i)))]
#pragma unroll
        for (int q = n - 1; q >= 0; --q) {
          const int pc = n - 1 - q, pt = n - 1 - ((q + 1) % n);
          if ((j >> pc) & 1) j ^= 1 << pt;
        }
        e = j;
      } else {
        int par = 0;
#pragma unroll
        for (int q = 0; q < n; ++q) par ^= ((i >> (n - 1 - q)) & (i >> (n - 1 - (q + 1) % n))) & 1;
        e = int(unsigned(i) | (unsigned(par) << 31));
      }
    }
    perm[i] = e;
  }
  __syncthreads();

  const bool active = tid < N;
  const int ixX = (w << LB) | l, ixY = (l << WB) | w;
  const int sX = tswz(ixX), sY = tswz(ixY);
  const int eperm = (active && n >= 2) ? perm[ixX] : ixX;
  const int sP = tswz(eperm & 0x7fffffff);
  const bool pneg = eperm < 0;
  double2 v = make_double2(tid == 0 ? 1.0 : 0.0, 0.0);  // layout X, |0...0>
  for (int layer = 0; layer < layers; ++layer) {
    // gate table of this layer: qubit q = n - 1 - pos at tabU + 4 (layer n + q) + 2 mybit
    const double2* tl = tabU + 4 * (layer * n) + 2 * 0;
#pragma unroll
    for (int pos = 0; pos < n; ++pos) {
      if (pos == LB && WB > 0) {  // X -> Y transpose
        if (active) sbuf[sX] = v;
        __syncthreads();
        if (active) v = sbuf[sY];
        __syncthreads();
      }
      const int lbit = pos < LB ? pos : pos - WB;  // lane bit carrying this position
      const int mybit = (l >> lbit) & 1;
      const double2* u = tl + 4 * (n - 1 - pos) + 2 * mybit;
      const double2 cs = u[0], co = u[1];
      const double2 pp = make_double2(__shfl_xor_sync(full, v.x, 1 << lbit), __shfl_xor_sync(full, v.y, 1 << lbit));
      v = make_double2(fma(cs.x, v.x, fma(-cs.y, v.y, fma(co.x, pp.x, -co.y * pp.y))),
                       fma(cs.x, v.y, fma(cs.y, v.x, fma(co.x, pp.y, co.y * pp.x))));
    }
    // back to layout X with the entangling ring folded into the read
    if (active) sbuf[WB > 0 ? sY : sX] = v;
    __syncthreads();
    if (active) {
      const double2 a = sbuf[sP];
      v = pneg ? make_double2(-a.x, -a.y) : a;
    }
    __syncthreads();
  }
  if (active) x_all[(size_t)blockIdx.x * N + ixX] = v;
}

// ---------------------------------------------------------------------------
// a2 for 7 <= n <= 10: four amplitudes per thread (2^(n-2) threads, <= 8 warps).
//   layout X: i = (w << 7) | (l << 2) | r     r: 2 register bits, l: 5 lane bits, w: W = n-7 bits
//   layout Y: warp bits <-> lane bits 0..W-1 swapped: positions 7..n-1 become lane bits 0..W-1
// Register-bit gates are in-thread 2x2 complex matvecs; lane-bit gates are one shuffle per
// amplitude + a 2-term complex dot.  The gate coefficients are loaded once per warp and gate
// and reused for the thread's 4 independent amplitudes (4x fewer SMEM wavefronts per
// amplitude than one amplitude per thread; measured SMEM-bound otherwise).
// ---------------------------------------------------------------------------
// phase timestamps for tools/prefix_timing.cu (compiled with -DDVQLS_PREFIX_TS; no code otherwise)
#ifdef DVQLS_PREFIX_TS
__device__ long long g_prefix_ts[256];
__device__ unsigned long long g_prefix_gt[256];  // %globaltimer (ns) at the same stamps
#define PREFIX_TS(k) do { if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) { \
    unsigned long long gt_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_)); \
    g_prefix_ts[(threadIdx.x >> 5) * 16 + (k)] = clock64(); g_prefix_gt[(threadIdx.x >> 5) * 16 + (k)] = gt_; } } while (0)
#else
#define PREFIX_TS(k) do { } while (0)
#endif
__device__ __forceinline__ int qswz(int i) { return i ^ ((i >> 2) & 7) ^ ((i >> 7) & 7); }

template <int NQ>
__global__ void __launch_bounds__(256)
prefix_quad_kernel(int layers, int entangler, const double* __restrict__ thetas, double2* __restrict__ x_all) {
  PREFIX_TS(0);
  pdl_trigger();
  constexpr int n = NQ;
  constexpr int N = 1 << n;
  constexpr int W = n - 7;
  extern __shared__ double2 qsm[];
  const int P = 3 * n * layers;
  const int G = n * layers;
  double2* sbuf0 = qsm;                           // 2 x N amplitudes: the two transposes of a
  double2* sbuf1 = qsm + N;                       // layer use different buffers (1 barrier each)
  double2* tabU = qsm + 2 * N;                    // 2 per gate: a, b of U = [[a, -b*], [b, a*]]
  int* perm = reinterpret_cast<int*>(tabU + 2 * G);
  const double* th = thetas + (size_t)blockIdx.x * P;
  const int tid = threadIdx.x;
  const int l = tid & 31, w = tid >> 5;
  const unsigned full = 0xffffffffu;

  for (int g = tid; g < G; g += blockDim.x) {
    double s0, c0, s1, c1, s2, c2;
    sincos(0.5 * th[3 * g + 0], &s0, &c0);
    sincos(0.5 * th[3 * g + 1], &s1, &c1);
    sincos(0.5 * th[3 * g + 2], &s2, &c2);
    tabU[2 * g + 0] = make_double2(c1 * (c2 * c0 - s2 * s0), -s1 * (c2 * c0 + s2 * s0));
    tabU[2 * g + 1] = make_double2(c1 * (s2 * c0 + c2 * s0), s1 * (c2 * s0 - s2 * c0));
  }
  for (int i = tid; i < N; i += blockDim.x) {
    int e = i;
    if (entangler == 0) {
      int j = i;  // new[i] = old[c_0(c_1(...c_{n-1}(i)))]
#pragma unroll
      for (int q = n - 1; q >= 0; --q) {
        const int pc = n - 1 - q, pt = n - 1 - ((q + 1) % n);
        if ((j >> pc) & 1) j ^= 1 << pt;
      }
      e = j;
    } else {
      int par = 0;
#pragma unroll
      for (int q = 0; q < n; ++q) par ^= ((i >> (n - 1 - q)) & (i >> (n - 1 - (q + 1) % n))) & 1;
      e = int(unsigned(i) | (unsigned(par) << 31));
    }
    perm[i] = e;
  }
  __syncthreads();

  // element indices of this thread's 4 amplitudes in both layouts
  const int iX0 = (w << 7) | (l << 2);
  const int iY0 = ((l >> W) << (2 + W)) | (w << 2) | ((l & ((1 << W) - 1)) << 7);
  int pX[4];
  bool nX[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = perm[iX0 | r];
    pX[r] = qswz(e & 0x7fffffff);
    nX[r] = e < 0;
  }
  double2 v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) v[r] = make_double2((iX0 | r) == 0 ? 1.0 : 0.0, 0.0);

  // 2x2 gate on register bit RBIT (positions 0, 1)
  auto reg_gate = [&](int g, int rbit) {
    const double2 ua = tabU[2 * g], ub = tabU[2 * g + 1];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (!(r & (1 << rbit))) {
        const double2 x0 = v[r], x1 = v[r | (1 << rbit)];
        v[r] = make_double2(fma(ua.x, x0.x, fma(-ua.y, x0.y, fma(-ub.x, x1.x, -ub.y * x1.y))),
                            fma(ua.x, x0.y, fma(ua.y, x0.x, fma(-ub.x, x1.y, ub.y * x1.x))));
        v[r | (1 << rbit)] = make_double2(fma(ub.x, x0.x, fma(-ub.y, x0.y, fma(ua.x, x1.x, ua.y * x1.y))),
                                          fma(ub.x, x0.y, fma(ub.y, x0.x, fma(ua.x, x1.y, -ua.y * x1.x))));
      }
  };
  // gate on lane bit LBIT: row of U selected by the thread's bit; partner amplitude by shuffle
  auto lane_gate = [&](int g, int lbit) {
    const double2 ua = tabU[2 * g], ub = tabU[2 * g + 1];
    const bool bit = (l >> lbit) & 1;
    // bit 0: self = a, other = -conj(b);  bit 1: self = conj(a), other = b
    const double2 cs = make_double2(ua.x, bit ? -ua.y : ua.y);
    const double2 co = make_double2(bit ? ub.x : -ub.x, ub.y);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double2 pp =
          make_double2(__shfl_xor_sync(full, v[r].x, 1 << lbit), __shfl_xor_sync(full, v[r].y, 1 << lbit));
      // self part first (overlaps the shuffle latency), then two FMAs on the partner:
      // 4 FP64 ops per component (DMUL + 3 DFMA), 2 of them after the shuffle
      const double sr = fma(cs.x, v[r].x, -cs.y * v[r].y), si = fma(cs.x, v[r].y, cs.y * v[r].x);
      v[r] = make_double2(fma(co.x, pp.x, fma(-co.y, pp.y, sr)), fma(co.x, pp.y, fma(co.y, pp.x, si)));
    }
  };

  PREFIX_TS(1);
  for (int layer = 0; layer < layers; ++layer) {
    const int gl = layer * n;  // gate of qubit q is gl + q, qubit q <-> position n - 1 - q
    reg_gate(gl + (n - 1 - 0), 0);
    reg_gate(gl + (n - 1 - 1), 1);
#pragma unroll
    for (int pos = 2; pos < 7; ++pos) lane_gate(gl + (n - 1 - pos), pos - 2);
    if (layer == 0) PREFIX_TS(2);
    // Buffer discipline: a buffer is rewritten only after a barrier that follows every read of
    // it (the reads of sbuf0 precede the barrier of sbuf1 and vice versa), so each transpose
    // needs a single barrier.  W = 0 (no warp bits): alternate the one transpose per layer.
    double2* ring = sbuf1;
    if (W > 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) sbuf0[qswz(iX0 | r)] = v[r];
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 4; ++r) v[r] = sbuf0[qswz(iY0 | r)];
#pragma unroll
      for (int pos = 7; pos < n; ++pos) lane_gate(gl + (n - 1 - pos), pos - 7);
#pragma unroll
      for (int r = 0; r < 4; ++r) sbuf1[qswz(iY0 | r)] = v[r];
    } else {
      ring = (layer & 1) ? sbuf1 : sbuf0;
#pragma unroll
      for (int r = 0; r < 4; ++r) ring[qswz(iX0 | r)] = v[r];
    }
    __syncthreads();
    // entangling ring folded into the read back to layout X
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double2 a = ring[pX[r]];
      v[r] = nX[r] ? make_double2(-a.x, -a.y) : a;
    }
    if (layer == 0) PREFIX_TS(3);
  }
  PREFIX_TS(4);
  double2* x = x_all + (size_t)blockIdx.x * N;
#pragma unroll
  for (int r = 0; r < 4; ++r) x[iX0 | r] = v[r];
}

// ---------------------------------------------------------------------------
// a9/a10 fused into the Hadamard kernels: the last CTA of a theta to finish (ticket
// counter) sums the NG partial quadruples in a fixed order and writes (C, E, Psi) or
// (E, Psi) for the cross-rank allreduce.
// ---------------------------------------------------------------------------
// Fused cross-rank reduction over NVLink peer memory (replaces ncclAllReduce + finalize on the
// cost path; layout and protocol in types.h P2PArgs).  The buffer half is chosen by epoch
// parity; a rank can be at most one call ahead of any peer (it cannot finish call e+1 before
// every peer has published call e+1), so two halves suffice.  The wait is bounded by
// timeout_ns of %globaltimer (wall clock, independent of the SM clock): on expiry the sticky
// error word is set (the host returns DVQLS_E_NCCL and refuses further cost calls on the
// context) and the slot's cost is NaN.
__device__ __forceinline__ double* p2p_slot(char* base, const P2PArgs& a, int par, int r, int k) {
  return reinterpret_cast<double*>(base) + ((size_t(par) * a.world + r) * a.KB + k) * 4;
}
__device__ __forceinline__ unsigned long long* p2p_flag(char* base, const P2PArgs& a, int par, int r, int k) {
  return reinterpret_cast<unsigned long long*>(base + size_t(2) * a.world * a.KB * 32) +
         (size_t(par) * a.world + r) * a.KB + k;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double nan_dev() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ __forceinline__ double cost_of_dev(double ReE, double RePsi, int n) {
  return RePsi <= 1e-12 ? nan_dev() : 0.5 - 0.5 * ReE / (double(n) * RePsi);
}

static __device__ void p2p_allreduce(const P2PArgs& a, int kth, int n, double e0, double e1, double e2, double e3,
                              double* __restrict__ out) {
  const unsigned long long epoch = a.epochs[kth] + 1ull;
  a.epochs[kth] = epoch;  // only this thread reduces slot kth in this launch
  const int par = int(epoch & 1ull);
  for (int q = 0; q < a.world; ++q) {
    volatile double* d = p2p_slot(a.peers[q], a, par, a.rank, kth);
    d[0] = e0; d[1] = e1; d[2] = e2; d[3] = e3;
  }
  __threadfence_system();
  for (int q = 0; q < a.world; ++q) *reinterpret_cast<volatile unsigned long long*>(
      p2p_flag(a.peers[q], a, par, a.rank, kth)) = epoch;
  char* mine = a.peers[a.rank];
  bool ok = true;
  const unsigned long long t0 = globaltimer_ns();
  for (int q = 0; q < a.world && ok; ++q) {
    volatile unsigned long long* f = p2p_flag(mine, a, par, q, kth);
    while (*f != epoch) {
      if (globaltimer_ns() - t0 > a.timeout_ns) { ok = false; break; }
    }
  }
  __threadfence_system();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int q = 0; q < a.world; ++q) {  // fixed rank order: identical sums on every rank
    volatile double* d = p2p_slot(mine, a, par, q, kth);
    s0 += d[0]; s1 += d[1]; s2 += d[2]; s3 += d[3];
  }
  double* o = out + (size_t)kth * 5;
  if (!ok) {
    atomicOr(a.err, 1u);
    s0 = s1 = s2 = s3 = nan_dev();
  }
  o[0] = ok ? cost_of_dev(s0, s2, n) : nan_dev();
  o[1] = s0; o[2] = s1; o[3] = s2; o[4] = s3;
}

static __device__ void finish_partials(const double* __restrict__ partials, int64_t NG, int kth, int n, int with_cost,
                                double* __restrict__ out, unsigned* __restrict__ counter,
                                const P2PArgs* p2p = nullptr) {
  __shared__ unsigned s_last;
  __shared__ double sred[4][32];
  __threadfence();  // partials of this CTA visible device-wide before the ticket
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter + kth, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double* p = partials + (size_t)kth * NG * 4;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int64_t i = threadIdx.x; i < NG; i += blockDim.x) {
    a0 += __ldcg(p + 4 * i + 0); a1 += __ldcg(p + 4 * i + 1);
    a2 += __ldcg(p + 4 * i + 2); a3 += __ldcg(p + 4 * i + 3);
  }
  for (int off = 16; off >= 1; off >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, off); a1 += __shfl_xor_sync(0xffffffffu, a1, off);
    a2 += __shfl_xor_sync(0xffffffffu, a2, off); a3 += __shfl_xor_sync(0xffffffffu, a3, off);
  }
  const int wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) { sred[0][wid] = a0; sred[1][wid] = a1; sred[2][wid] = a2; sred[3][wid] = a3; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
    for (int w = 0; w < nw; ++w) { e0 += sred[0][w]; e1 += sred[1][w]; e2 += sred[2][w]; e3 += sred[3][w]; }
    if (p2p) {
      p2p_allreduce(*p2p, kth, n, e0, e1, e2, e3, out);
    } else if (with_cost) {  // 2: partial sums of a virtual rank (no cost)
      double* o = out + (size_t)kth * 5;
      o[0] = with_cost == 2 ? nan_dev() : cost_of_dev(e0, e2, n); o[1] = e0; o[2] = e1; o[3] = e2; o[4] = e3;
    } else {
      double* o = out + (size_t)kth * 4;
      o[0] = e0; o[1] = e1; o[2] = e2; o[3] = e3;
    }
    counter[kth] = 0u;  // ready for the next call (stream-ordered)
  }
}

// a9/a10 for kernels whose CTAs cover (theta, circuit) ranges flattened over a batch of K
// thetas: partials[k][G][4] holds one fixed-order quadruple per CTA and theta (zero where the CTA
// did not touch theta).  The last CTA of the grid (ticket) sums each theta's G quadruples in CTA
// order and writes (C, E, Psi) / (E, Psi), or runs the NVLink allreduce per theta.
static __device__ void finish_all(const double* __restrict__ partials, int G, int K, int n, int with_cost,
                           double* __restrict__ out, unsigned* __restrict__ counter, const P2PArgs& p2p) {
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp w reduces thetas w, w + nwarps, ...: lanes stride the CTAs, then a fixed shuffle tree
  for (int k = warp; k < K; k += int(blockDim.x >> 5)) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int b = lane; b < G; b += 32) {
      const double* p = partials + (size_t(k) * G + b) * 4;
      a0 += __ldcg(p + 0); a1 += __ldcg(p + 1); a2 += __ldcg(p + 2); a3 += __ldcg(p + 3);
    }
    for (int off = 16; off >= 1; off >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, off); a1 += __shfl_xor_sync(0xffffffffu, a1, off);
      a2 += __shfl_xor_sync(0xffffffffu, a2, off); a3 += __shfl_xor_sync(0xffffffffu, a3, off);
    }
    if (lane == 0) {
      if (p2p.world > 1) {
        p2p_allreduce(p2p, k, n, a0, a1, a2, a3, out);
      } else if (with_cost) {  // 2: partial sums of a virtual rank (no cost)
        double* o = out + size_t(k) * 5;
        o[0] = with_cost == 2 ? nan_dev() : cost_of_dev(a0, a2, n); o[1] = a0; o[2] = a1; o[3] = a2; o[4] = a3;
      } else {
        double* o = out + size_t(k) * 4;
        o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *counter = 0u;  // ready for the next launch (stream-ordered)
}

// ---------------------------------------------------------------------------
// a3-a9: batched Hadamard-test kernel for n = NQ system qubits.
//
// A circuit is owned by a group of GT = 2^TB threads, each holding R = 2^RB
// complex128 amplitudes of the ancilla-|1> branch in registers (TB = NQ/2,
// RB = NQ - TB; n = 10: one warp, 32 amplitudes per thread).
//   layout A: thread t, register r  <->  index i = (r << TB) | t
//   layout B: thread t, register r  <->  index i = (t << RB) | r
// One U_b^+ = H^{(x)n} is: butterflies on the RB register bits in layout A,
// one SMEM exchange A->B, butterflies on the remaining TB bits in layout B.
// The second FWHT runs B then A, so a numerator circuit costs two exchanges.
// Exchange buffers are XOR-swizzled so both layouts hit 8 distinct 16-byte
// bank groups per quarter-warp (conflict-free LDS.128/STS.128).
// ---------------------------------------------------------------------------
template <int NQ>
struct Shape {
  static constexpr int TB = NQ / 2;
  static constexpr int RB = NQ - TB;
  static constexpr int GT = 1 << TB;  // threads per circuit
  static constexpr int R = 1 << RB;   // amplitudes per thread
  static constexpr int N = 1 << NQ;
  static constexpr int GPW = 32 / GT; // circuit groups per warp
};

template <int NQ>
__device__ __forceinline__ int swz(int i) {
  if constexpr (NQ >= 6)
    return i ^ ((i >> Shape<NQ>::RB) & 7);
  else
    return i;
}

// butterflies (a, b) -> (a + b, a - b) on register bits [B0, B1)
template <int R, int B0, int B1>
__device__ __forceinline__ void fwht_regs(double2 (&v)[R]) {
#pragma unroll
  for (int bb = B0; bb < B1; ++bb) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!(r & (1 << bb))) {
        const double2 p = v[r], q = v[r | (1 << bb)];
        v[r] = make_double2(p.x + q.x, p.y + q.y);
        v[r | (1 << bb)] = make_double2(p.x - q.x, p.y - q.y);
      }
    }
  }
}

// A value the compiler cannot see through: stops it from keeping 32 exchange addresses
// alive between the two exchanges of a circuit (they are one LOP3 each to recompute).
// (a shuffle with offset 0: ptxas cannot prove the result equal to its input)
__device__ __forceinline__ uint32_t opaque(uint32_t v, unsigned gmask) {
  return __shfl_xor_sync(gmask, v, 0);
}

__host__ __device__ constexpr int ctz_c(int k) {
  return (k & 1) ? 0 : (k & 2) ? 1 : (k & 4) ? 2 : (k & 8) ? 3 : (k & 16) ? 4 : (k & 32) ? 5 : 6;
}

// Registers are visited in Gray-code order r_k = k ^ (k >> 1): every index map used here
// (XOR masks, sign bit, swizzle) is GF(2)-linear in r, so the next address is the
// previous one XOR one column -- one LOP3 and one live address register per access.
//
// Exchange A -> B (A_TO_B) or B -> A through the group's SMEM buffer.  Slot of index i
// is swz(i); swz is linear, so slot((r << TB) | t) = swz(t) ^ swz(r << TB) and
// slot((t << RB) | r) = swz(t << RB) ^ r.
template <int NQ, bool A_TO_B>
__device__ __forceinline__ void exchange(double2 (&v)[Shape<NQ>::R], uint32_t buf_off, int t, unsigned gmask) {
  using S = Shape<NQ>;
  // buf_off is a multiple of the buffer size (a power of two >= every slot offset),
  // so buf_off + slot == buf_off ^ slot and the whole address is one XOR chain.
  const uint32_t to = opaque(uint32_t(t), gmask);
  const uint32_t slotA0 = buf_off ^ (uint32_t(swz<NQ>(int(to))) * 16u);           // layout A, r = 0
  const uint32_t slotB0 = buf_off ^ (uint32_t(swz<NQ>(int(to) << S::RB)) * 16u);  // layout B, r = 0
  __syncwarp(gmask);  // previous readers of buf are done
  {
    uint32_t a = A_TO_B ? slotA0 : slotB0;
#pragma unroll
    for (int k = 0; k < S::R; ++k) {
      const int r = k ^ (k >> 1);
      if (k) {
        const int bb = ctz_c(k);
        a ^= A_TO_B ? uint32_t(swz<NQ>(1 << (S::TB + bb))) * 16u : (16u << bb);
      }
      sts2(a, v[r]);
    }
  }
  __syncwarp(gmask);
  {
    uint32_t a = A_TO_B ? slotB0 : slotA0;
#pragma unroll
    for (int k = 0; k < S::R; ++k) {
      const int r = k ^ (k >> 1);
      if (k) {
        const int bb = ctz_c(k);
        a ^= A_TO_B ? (16u << bb) : uint32_t(swz<NQ>(1 << (S::TB + bb))) * 16u;
      }
      v[r] = lds2(a);
    }
  }
}

// Signed, XOR-permuted read of [x, -x] in layout A (Gray-code addressing):
//   register r <- (-1)^{sgn0 ^ parity(r & zh)} x[((r ^ mh) << TB) | tl]
// (SMEM holds x at [0, N) and -x at [N, 2N): the sign is index bit NQ).
template <int NQ>
__device__ __forceinline__ void signed_gather(double2 (&v)[Shape<NQ>::R], uint32_t mh, uint32_t tl, uint32_t zh,
                                              uint32_t sgn0) {
  using S = Shape<NQ>;
  uint32_t a = (((mh << S::TB) | tl) | (sgn0 << NQ)) * 16u;
#pragma unroll
  for (int k = 0; k < S::R; ++k) {
    const int r = k ^ (k >> 1);
    if (k) {
      const int bb = ctz_c(k);
      a ^= ((1u << (S::TB + bb)) | (((zh >> bb) & 1u) << NQ)) * 16u;
    }
    v[r] = lds2(a);
  }
}

// Readout sum over registers of conj(x'_r) phi_r, x' from the same signed gather.
// IM = false: sum Re(conj(x') phi) = xr phr + xi phi;  IM = true: sum Im = xr phi - xi phr.
template <int NQ, bool IM>
__device__ __forceinline__ double signed_dot(const double2 (&v)[Shape<NQ>::R], uint32_t mh, uint32_t tl,
                                             uint32_t zh, uint32_t sgn0) {
  using S = Shape<NQ>;
  uint32_t a = (((mh << S::TB) | tl) | (sgn0 << NQ)) * 16u;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < S::R; ++k) {
    const int r = k ^ (k >> 1);
    if (k) {
      const int bb = ctz_c(k);
      a ^= ((1u << (S::TB + bb)) | (((zh >> bb) & 1u) << NQ)) * 16u;
    }
    // at most 8 x loads in flight: keeps the live set at 128 branch registers + 32
    if (k && !(k & 7)) asm volatile("" ::: "memory");
    const double2 x = lds2(a);
    if (IM) {
      acc[k & 3] = fma(x.x, v[r].y, acc[k & 3]);
      acc[k & 3] = fma(-x.y, v[r].x, acc[k & 3]);
    } else {
      acc[k & 3] = fma(x.x, v[r].x, acc[k & 3]);
      acc[k & 3] = fma(x.y, v[r].y, acc[k & 3]);
    }
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

template <int GT>
__device__ __forceinline__ double group_sum(double v, unsigned gmask) {
#pragma unroll
  for (int off = GT / 2; off >= 1; off >>= 1) v += __shfl_xor_sync(gmask, v, off);
  return v;
}

// phi <- H_v phi = phi - (2 / v^+v) (v^+ phi) v  (layout A), Householder U_b up to the
// phase w, which cancels between U_b^+ and U_b.
template <int NQ>
__device__ __forceinline__ void householder(double2 (&v)[Shape<NQ>::R], const double2* shv, double hv_scale,
                                            int t, unsigned gmask) {
  using S = Shape<NQ>;
  double dr = 0.0, di = 0.0;
#pragma unroll
  for (int r = 0; r < S::R; ++r) {
    const double2 h = shv[(r << S::TB) | t];
    dr = fma(h.x, v[r].x, fma(h.y, v[r].y, dr));
    di = fma(h.x, v[r].y, fma(-h.y, v[r].x, di));
  }
  dr = group_sum<S::GT>(dr, gmask) * hv_scale;
  di = group_sum<S::GT>(di, gmask) * hv_scale;
#pragma unroll
  for (int r = 0; r < S::R; ++r) {
    const double2 h = shv[(r << S::TB) | t];
    v[r].x -= dr * h.x - di * h.y;
    v[r].y -= dr * h.y + di * h.x;
  }
}

// sign flip of every amplitude whose register index has bit B set (compile-time B)
template <int R, int B>
__device__ __forceinline__ void zflip_reg(double2 (&v)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r & (1 << B)) v[r] = make_double2(flip(v[r].x, 0x80000000u), flip(v[r].y, 0x80000000u));
}

template <int R, int B = 0>
__device__ __forceinline__ void zflip_reg_rt(double2 (&v)[R], int bit) {
  if constexpr ((1 << B) < R) {
    if (bit == B) zflip_reg<R, B>(v);
    else zflip_reg_rt<R, B + 1>(v, bit);
  }
}

// register cap per thread: the whole 64K-entry register file split over WARPS warps,
// rounded down to the allocation granularity of 8
template <int WARPS>
constexpr int reg_cap() { return (65536 / (WARPS * 32)) / 8 * 8 > 255 ? 255 : (65536 / (WARPS * 32)) / 8 * 8; }

// Cost-weighted static split of circuits [c0, c0 + C) over NG groups: in canonical order every
// period of 2(n+1) circuits holds 2 denominator circuits (weight 1: gather + readout) and 2n
// numerator circuits (weight WNUM: + two FWHTs and exchanges; ~3x the SMEM wavefronts).
// Equal-count ranges leave whole numerator circuits of imbalance per group at small per-GPU
// work (6 circuits per group at 8 GPUs); equal-weight ranges halve it.  Closed form, no search.
constexpr int64_t WNUM = 3;
__device__ __forceinline__ int64_t wcum(int64_t c, int n) {  // weight of circuits [0, c)
  const int64_t P = 2 * int64_t(n + 1), per = 2 + 2 * int64_t(n) * WNUM;
  const int64_t q = c / P, r = c - q * P;
  return q * per + (r < 2 ? r : 2 + (r - 2) * WNUM);
}
__device__ __forceinline__ int64_t winv(int64_t w, int n) {  // smallest c with wcum(c) >= w
  const int64_t P = 2 * int64_t(n + 1), per = 2 + 2 * int64_t(n) * WNUM;
  const int64_t q = w / per, rem = w - q * per;
  return q * P + (rem <= 2 ? rem : 2 + (rem - 2 + WNUM - 1) / WNUM);
}
__device__ __forceinline__ void weighted_range(int64_t c0, int64_t C, int64_t g, int64_t NG, int n, int64_t* b,
                                               int64_t* e) {
  const int64_t w0 = wcum(c0, n), tot = wcum(c0 + C, n) - w0;
  const int64_t lo = winv(w0 + tot * g / NG, n), hi = winv(w0 + tot * (g + 1) / NG, n);
  *b = min(max(lo - c0, int64_t(0)), C);
  *e = g + 1 == NG ? C : min(max(hi - c0, int64_t(0)), C);
}

template <int NQ, int WARPS, bool HH>
__global__ void __launch_bounds__(WARPS * 32) __maxnreg__(reg_cap<WARPS>())
hadamard_kernel(const double2* __restrict__ x_all, const PauliTerm* __restrict__ tab,
                const double2* __restrict__ coef, const double2* __restrict__ hv, double hv_scale, int L,
                int64_t c0, int64_t C, int K, double* __restrict__ out_terms, double* __restrict__ partials,
                int with_cost, double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {
  pdl_wait();
  using S = Shape<NQ>;
  constexpr int TB = S::TB, RB = S::RB, GT = S::GT, R = S::R, N = S::N, GPW = S::GPW;
  double2* smem = dvqls_smem;
  double2* sx = smem;              // [x, -x]: 2N
  double2* shv = smem + 2 * N;     // Householder vector (HH only)
  double2* sbuf = smem + (HH ? 3 : 2) * N;
  double* sacc = reinterpret_cast<double*>(sbuf + (size_t)WARPS * GPW * N);  // 4 per group

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane / GT, t = lane % GT;
  const unsigned gmask = (GT == 32) ? 0xffffffffu : (((1u << GT) - 1u) << (gw * GT));
  double2* buf = sbuf + (size_t)(warp * GPW + gw) * N;
  // byte offset of this group's exchange buffer; a multiple of 16 N when HH is false
  const uint32_t buf_off = uint32_t(reinterpret_cast<char*>(buf) - reinterpret_cast<char*>(smem));
  constexpr int NGC = WARPS * GPW;  // circuit groups per CTA
  const int gi = warp * GPW + gw;
  const int n1 = NQ + 1;
  double* acc4 = sacc + 4 * gi;  // per-group running sums (Re E, Im E, Re Psi, Im Psi)
  if (HH)
    for (int i = threadIdx.x; i < N; i += blockDim.x) shv[i] = hv[i];

  // ---- a3: this CTA's cost-weighted slice of the K x C (theta, circuit) work, flattened so
  // that a batch of K thetas balances across all CTAs of one persistent grid ----
  const int64_t G = gridDim.x;
  const int64_t w0 = wcum(c0, NQ), Wt = wcum(c0 + C, NQ) - w0, Wall = Wt * K;
  auto flat_of = [&](int64_t w) -> int64_t {  // first flattened circuit at weight >= w
    if (w >= Wall) return int64_t(K) * C;
    const int64_t th = w / Wt, rem = w - th * Wt;
    const int64_t c = min(max(winv(w0 + rem, NQ) - c0, int64_t(0)), C);
    return th * C + c;
  };
  const int64_t Fb = Wall > 0 ? flat_of(Wall * (int64_t)blockIdx.x / G) : 0;
  const int64_t Fe = Wall <= 0 ? 0 : blockIdx.x + 1 == G ? int64_t(K) * C : flat_of(Wall * ((int64_t)blockIdx.x + 1) / G);
  const int th_first = C > 0 ? int(Fb / C) : 0, th_last = Fe > Fb ? int((Fe - 1) / C) : th_first - 1;
  for (int k = threadIdx.x; k < K; k += blockDim.x)  // thetas this CTA does not touch contribute 0
    if (k < th_first || k > th_last)
      for (int q = 0; q < 4; ++q) partials[(size_t(k) * G + blockIdx.x) * 4 + q] = 0.0;

  for (int kth = th_first; kth <= th_last; ++kth) {
  // ---- one phase per theta: stage [x, -x] of this theta, split its circuits over the groups ----
  const int64_t pa = max(Fb, int64_t(kth) * C) - int64_t(kth) * C;
  const int64_t pb = min(Fe, int64_t(kth + 1) * C) - int64_t(kth) * C;
  const double2* x = x_all + (size_t)kth * N;
  __syncthreads();  // previous phase's readers of sx are done
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double2 a = x[i];
    sx[i] = a;
    sx[N + i] = make_double2(-a.x, -a.y);
  }
  __syncthreads();
  int cb, ce;  // this group's circuits [cb, ce) of theta kth (local index), cost-weighted
  {
    int64_t b, e;
    weighted_range(c0 + pa, pb - pa, gi, NGC, NQ, &b, &e);
    cb = int(pa + b);
    ce = int(pa + e);
  }
  if (t == 0) acc4[0] = acc4[1] = acc4[2] = acc4[3] = 0.0;
  // canonical decode c -> (l, k, s, part) once per phase, then advanced per circuit without
  // divisions (64-bit division by the run-time L costs ~100 instructions per circuit)
  int part_, s_, k_, l_;
  {
    const int64_t c = c0 + cb, tk = c >> 1, lk = tk / n1;
    part_ = int(c & 1);
    s_ = int(tk % n1);
    k_ = int(lk % L);
    l_ = int(lk / L);
  }
  for (int cl = cb; cl < ce; ++cl) {
    const int part = part_, s = s_, k = k_, l = l_;
    if (++part_ == 2) {
      part_ = 0;
      if (++s_ == n1) {
        s_ = 0;
        if (++k_ == L) { k_ = 0; ++l_; }
      }
    }
    const PauliTerm Tk = tab[k];

    // ---- a4: branch init + c-A_k: phi_i = sgn_k(i ^ m_k) x[i ^ m_k]  (layout A) ----
    // (the i^{n_Y} and kappa phases are folded into q below)
    double2 v[R];
    {
      const uint32_t mh = Tk.xm >> TB, tl = uint32_t(t) ^ (Tk.xm & (GT - 1)), zh = Tk.zm >> TB;
      const uint32_t sg0 = (__popc(tl & Tk.zm & (GT - 1)) ^ __popc(mh & zh)) & 1u;
      signed_gather<NQ>(v, mh, tl, zh, sg0);
    }
    double scale = 1.0;
    if (s > 0) {
      const int p = NQ - 1 - (s - 1);  // bit position of Z_j, j = s - 1
      if (!HH) {
        // ---- a5: c-U_b^+ = unnormalised FWHT (layout A bits TB..NQ-1, layout B bits 0..TB-1)
        fwht_regs<R, 0, RB>(v);
        exchange<NQ, true>(v, buf_off, t, gmask);
        fwht_regs<R, 0, TB>(v);
        // ---- a6: c-Z_j (layout B: register bit p, or thread bit p - RB) --------------
        if (p < RB) {
          zflip_reg_rt<R>(v, p);
        } else {
          const uint32_t m = uint32_t((t >> (p - RB)) & 1) << 31;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = make_double2(flip(v[r].x, m), flip(v[r].y, m));
        }
        // ---- a7: c-U_b ------------------------------------------------------------------
        fwht_regs<R, 0, TB>(v);
        exchange<NQ, false>(v, buf_off, t, gmask);
        fwht_regs<R, 0, RB>(v);
        scale = 1.0 / double(N);
      } else {
        householder<NQ>(v, shv, hv_scale, t, gmask);
        if (p >= TB) {
          zflip_reg_rt<R>(v, p - TB);
        } else {
          const uint32_t m = uint32_t((t >> p) & 1) << 31;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = make_double2(flip(v[r].x, m), flip(v[r].y, m));
        }
        householder<NQ>(v, shv, hv_scale, t, gmask);
      }
    }
    // ---- a8: c-A_l + ancilla readout: Re(i^q S), S = sum_j conj(sgn_l(j) x_{j ^ m_l}) phi_j
    const PauliTerm Tl = tab[l];  // loaded late: not live across the FWHTs
    const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
    double val;
    {
      const uint32_t mh = Tl.xm >> TB, tl = uint32_t(t) ^ (Tl.xm & (GT - 1)), zh = Tl.zm >> TB;
      const uint32_t sg0 = __popc(uint32_t(t) & Tl.zm & (GT - 1)) & 1u;
      val = (q & 1) ? signed_dot<NQ, true>(v, mh, tl, zh, sg0) : signed_dot<NQ, false>(v, mh, tl, zh, sg0);
    }
    val = group_sum<GT>(val, gmask);
    val *= (q == 1 || q == 2) ? -scale : scale;

    // ---- a9 (fused): write the term, accumulate c_l^* c_k (Re + i Im) -----
    if (t == 0) {
      out_terms[(size_t)kth * C + cl] = val;
      const double2 cl_ = coef[l], ck = coef[k];
      const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
      const double cr = part == 0 ? wr * val : -wi * val;
      const double ci = part == 0 ? wi * val : wr * val;
      double* d = acc4 + (s == 0 ? 2 : 0);
      d[0] += cr;
      d[1] += ci;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // fixed group order
    double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
    for (int q = 0; q < NGC; ++q) { e0 += sacc[4 * q]; e1 += sacc[4 * q + 1]; e2 += sacc[4 * q + 2]; e3 += sacc[4 * q + 3]; }
    double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
    o[0] = e0; o[1] = e1; o[2] = e2; o[3] = e3;
  }
  }  // theta phases
  if (red_out) finish_all(partials, int(G), K, NQ, with_cost, red_out, counter, p2p);
}

}  // namespace dvqls
