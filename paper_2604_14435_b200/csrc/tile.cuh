// tile.cuh - V(theta)|0> for n >= 13 (SURVEY §8(a) a2 on the streaming path): the state
// lives in global memory and every layer is a few tile passes over it.
//
// A tile pass maps the TN = 4096 tile elements onto global index bits:
//     tile bits [0, c)   = global bits [0, c)         ("passengers": coalescing only)
//     tile bits [c, tb)  = global bits [b, b + tb - c) (the active bits of the pass)
// and applies the layer's fused single-qubit gates Ry Rz Ry on the active bits in rounds
// of 4 tile bits (16 amplitudes per thread in registers).  Bit groups:
//     g0 = [0, min(n,12)),  g1 = [12, 12 + min(n-12, 9)),  g2 = [21, n)
// The entangling ring is one gather pass (prefix_ring_kernel).  The Hadamard-test circuits
// of the n >= 11 path are in stream.cuh.
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace tile {

constexpr int TBITS = 12;
constexpr int TN = 1 << TBITS;
constexpr int THREADS = 256;
constexpr int RB = 4;          // register bits per round
constexpr int RR = 1 << RB;    // amplitudes per thread per round

struct Geo {
  int c, b, tb;  // passengers, first active global bit, tile bits
  __device__ __forceinline__ int a() const { return tb - c; }
  // global index of tile element e in tile number `tile`
  __device__ __forceinline__ uint32_t gidx(uint32_t tile, uint32_t e) const {
    const uint32_t lowp = e & ((1u << c) - 1u);
    const uint32_t act = e >> c;
    const uint32_t mid = tile & ((1u << (b - c)) - 1u);  // global bits [c, b)
    const uint32_t hi = tile >> (b - c);                  // global bits [b + a, n)
    return lowp | (mid << c) | (act << b) | (hi << (b + a()));
  }
};

__device__ __forceinline__ int ngroups(int n) { return n <= 12 ? 1 : (n <= 21 ? 2 : 3); }

__device__ __forceinline__ Geo group(int n, int gi) {
  Geo g;
  if (gi == 0) {
    g.c = 0; g.b = 0; g.tb = n < TBITS ? n : TBITS;
  } else if (gi == 1) {
    const int a = (n - 12) < 9 ? (n - 12) : 9;
    g.tb = TBITS; g.c = TBITS - a; g.b = 12;
  } else {
    const int a = n - 21;
    g.tb = TBITS; g.c = TBITS - a; g.b = 21;
  }
  return g;
}

// SMEM slot of tile element e: low 3 bits XOR bits 4..6 -> every round is conflict-free
__device__ __forceinline__ int tslot(int e) { return e ^ ((e >> 4) & 7); }

// element handled by (thread t, register r) in the round covering tile bits [4 rho, 4 rho + 4)
__device__ __forceinline__ int relem(int t, int r, int rho) {
  const int s = RB * rho;
  return ((t >> s) << (s + RB)) | (r << s) | (t & ((1 << s) - 1));
}

// ---------------------------------------------------------------------------
// Prefix for n >= 13 (state in global memory), one kernel per pass:
//   prefix_gates_kernel: SU(2) parameters (a, b) of every fused gate Ry Rz Ry
//   prefix_gate_pass:    one tile per CTA, the layer's gates on the group's bits
//   prefix_ring_kernel:  CNOT ring as a gather into the other buffer / CZ ring sign
// ---------------------------------------------------------------------------
__global__ void prefix_gates_kernel(const double* __restrict__ theta, int G, double2* __restrict__ gates) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  double s0, c0, s1, c1, s2, c2;
  sincos(0.5 * theta[3 * g + 0], &s0, &c0);
  sincos(0.5 * theta[3 * g + 1], &s1, &c1);
  sincos(0.5 * theta[3 * g + 2], &s2, &c2);
  gates[2 * g + 0] = make_double2(c1 * (c2 * c0 - s2 * s0), -s1 * (c2 * c0 + s2 * s0));
  gates[2 * g + 1] = make_double2(c1 * (s2 * c0 + c2 * s0), s1 * (c2 * s0 - s2 * c0));
}

__global__ void prefix_init_kernel(double2* __restrict__ x, uint32_t N) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
    x[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
}

__global__ void __launch_bounds__(THREADS)
prefix_gate_pass(double2* __restrict__ x, const double2* __restrict__ gates, int n, int gi, int layer) {
  double2* s = dvqls_smem;
  const Geo geo = group(n, gi);
  const uint32_t tile = blockIdx.x;
  const int t = threadIdx.x;
  for (int e = t; e < (1 << geo.tb); e += THREADS) s[tslot(e)] = x[geo.gidx(tile, e)];
  __syncthreads();
  for (int rho = 0; rho < TBITS / RB; ++rho) {
    double2 v[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) v[r] = s[tslot(relem(t, r, rho))];
#pragma unroll
    for (int bb = 0; bb < RB; ++bb) {
      const int q = RB * rho + bb;
      if (q >= geo.c && q < geo.tb) {
        const int pos = geo.b + (q - geo.c);
        const int g = layer * n + (n - 1 - pos);
        const double2 ua = gates[2 * g], ub = gates[2 * g + 1];
#pragma unroll
        for (int r = 0; r < RR; ++r)
          if (!(r & (1 << bb))) {
            const double2 x0 = v[r], x1 = v[r | (1 << bb)];
            v[r] = make_double2(fma(ua.x, x0.x, fma(-ua.y, x0.y, fma(-ub.x, x1.x, -ub.y * x1.y))),
                                fma(ua.x, x0.y, fma(ua.y, x0.x, fma(-ub.x, x1.y, ub.y * x1.x))));
            v[r | (1 << bb)] = make_double2(fma(ub.x, x0.x, fma(-ub.y, x0.y, fma(ua.x, x1.x, ua.y * x1.y))),
                                            fma(ub.x, x0.y, fma(ub.y, x0.x, fma(ua.x, x1.y, -ua.y * x1.x))));
          }
      }
    }
#pragma unroll
    for (int r = 0; r < RR; ++r) s[tslot(relem(t, r, rho))] = v[r];
    __syncthreads();
  }
  for (int e = t; e < (1 << geo.tb); e += THREADS) x[geo.gidx(tile, e)] = s[tslot(e)];
}

__global__ void prefix_ring_kernel(const double2* __restrict__ src, double2* __restrict__ dst, int n, int entangler) {
  const uint32_t N = 1u << n;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (entangler == 0) {
      uint32_t j = i;  // new[i] = old[c_0(c_1(...c_{n-1}(i)))]
      for (int q = n - 1; q >= 0; --q) {
        const int pc = n - 1 - q, pt = n - 1 - ((q + 1) % n);
        if ((j >> pc) & 1u) j ^= 1u << pt;
      }
      dst[i] = src[j];
    } else {
      int par = 0;
      for (int q = 0; q < n; ++q) par ^= int((i >> (n - 1 - q)) & (i >> (n - 1 - (q + 1) % n))) & 1;
      const double2 a = src[i];
      dst[i] = par ? make_double2(-a.x, -a.y) : a;
    }
  }
}

}  // namespace tile
}  // namespace dvqls
