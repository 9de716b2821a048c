// prefix_cluster.cuh - a2 for 7 <= n <= 10 on a thread-block CLUSTER: x = V(theta)|0^n> spread
// over CS = 2^(n-7) CTAs whose shared memories are joined through DSMEM (
// SURVEY §8(c) readings 6-9).
//
// One theta's 2^n amplitudes used to live in ONE CTA (prefix_quad_kernel): a latency-bound
// 20 us chain on a single SM that every cost call pays before any circuit can start (the K = 1
// fixed cost).  Here the state is split over the cluster, one amplitude per thread:
//   global index i = (rank << 7) | tid,  tid = (warp << 5) | lane,
//   positions 0..4 = lane bits, 5..6 = warp bits, 7..n-1 = cluster bits (the CTA rank).
// A layer (per qubit Ry Rz Ry fused into one SU(2) gate U_q, then the entangling ring) is
//   1. lane-bit gates: one shuffle of the partner amplitude + a 2-term complex dot each;
//   2. warp-bit gates (positions 5, 6) together: amplitudes through the CTA's SMEM, one barrier,
//      new value = sum over the 4 partners of (U_5 (x) U_6)[row, col] * partner;
//   3. cluster-bit gates (positions >= 7) AND the ring together: every CTA publishes its 128
//      amplitudes, one cluster barrier, then thread i reads, from all CS CTAs over DSMEM, the
//      amplitudes at local index j(p) of p = ring(i) and forms
//          x'[i] = sign(i) * sum_c' (U_{7} (x) ... (x) U_{n-1})[c(p), c'] * S_c'[j(p)]
//      (new[i] = old[ring(i)] for the CNOT ring, old[i] (-1)^{...} for the CZ ring).
// The Kronecker tables of steps 2 and 3 are built once per call from the gate table.  One CTA
// barrier and one cluster barrier per layer; the CS SMs share the FP64 work of the layer.
// Exchange buffers are double-buffered by layer parity, so a CTA may publish layer l+1 while a
// peer still reads layer l; a final cluster barrier keeps every CTA's SMEM alive until its peers
// have read the last layer.
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace pclus {

constexpr int LB = 7;          // local bits per CTA (lane 0..4, warp 5..6)
constexpr int NL = 1 << LB;    // amplitudes (= threads) per CTA

template <int NQ>
struct PC {
  static constexpr int CB = NQ - LB;  // cluster bits
  static constexpr int CS = 1 << CB;  // CTAs per cluster
};

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ double2 ld_dsmem(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmac(double2 a, double2 b, double2 acc) {  // acc + a b
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// entry (row, col) of U = [[a, -conj(b)], [b, conj(a)]] (gate table: a, b per gate)
__device__ __forceinline__ double2 uent(const double2* U, int g, int row, int col) {
  const double2 a = U[2 * g], b = U[2 * g + 1];
  if (row == 0) return col == 0 ? a : make_double2(-b.x, b.y);
  return col == 0 ? b : make_double2(a.x, -a.y);
}

// dynamic SMEM (double2 units): gates 2G | warp tables 16 per layer | cluster tables CS^2 per layer
// | warp-bit exchange 128 | published amplitudes 2 x 128
template <int NQ>
__host__ __device__ constexpr size_t smem_doubles2(int layers) {
  return size_t(2) * NQ * layers + size_t(16) * layers + size_t(PC<NQ>::CS) * PC<NQ>::CS * layers + 3 * NL;
}

template <int NQ>
__global__ void __launch_bounds__(NL)
prefix_cluster_kernel(int layers, int entangler, const double* __restrict__ thetas, double2* __restrict__ x_all) {
  pdl_trigger();
  constexpr int n = NQ, CB = PC<NQ>::CB, CS = PC<NQ>::CS;
  extern __shared__ double2 pcsm[];
  const int G = n * layers;
  double2* U = pcsm;                      // 2 per gate: a, b
  double2* W4 = U + 2 * G;                // [layer][x6 x5][y6 y5]
  double2* GC = W4 + 16 * layers;         // [layer][c][c']
  double2* sbuf = GC + CS * CS * layers;  // 128 (warp-bit step)
  double2* pub = sbuf + NL;               // [2][128] published amplitudes (cluster step)
  const double* th = thetas + (size_t)blockIdx.y * 3 * G;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t rank = CS > 1 ? cta_rank() : 0u;

  // ---- gate table (every CTA computes the whole table; 1 gate per thread for d <= 12) ----
  for (int g = tid; g < G; g += NL) {
    double s0, c0, s1, c1, s2, c2;
    sincos(0.5 * th[3 * g + 0], &s0, &c0);
    sincos(0.5 * th[3 * g + 1], &s1, &c1);
    sincos(0.5 * th[3 * g + 2], &s2, &c2);
    // U = Ry(t2) Rz(t1) Ry(t0) = [[a, -conj(b)], [b, conj(a)]]
    U[2 * g + 0] = make_double2(c1 * (c2 * c0 - s2 * s0), -s1 * (c2 * c0 + s2 * s0));
    U[2 * g + 1] = make_double2(c1 * (s2 * c0 + c2 * s0), s1 * (c2 * s0 - s2 * c0));
  }
  __syncthreads();
  // ---- Kronecker tables: positions 5, 6 (qubits n-6, n-7) and the cluster positions 7.. ----
  for (int e = tid; e < 16 * layers; e += NL) {
    const int layer = e >> 4, r = e & 15;
    const int x5 = (r >> 2) & 1, x6 = (r >> 3) & 1, y5 = r & 1, y6 = (r >> 1) & 1;
    const int gl = layer * n;
    W4[e] = cmul(uent(U, gl + (n - 1 - 5), x5, y5), uent(U, gl + (n - 1 - 6), x6, y6));
  }
  for (int e = tid; e < CS * CS * layers; e += NL) {
    const int layer = e / (CS * CS), rc = e % (CS * CS), c = rc / CS, cp = rc % CS;
    double2 f = make_double2(1.0, 0.0);
    for (int b = 0; b < CB; ++b)  // cluster bit b = position 7 + b = qubit n - 8 - b
      f = cmul(f, uent(U, layer * n + (n - 1 - (LB + b)), (c >> b) & 1, (cp >> b) & 1));
    GC[e] = f;
  }
  // ---- this thread's ring source p = ring(i): CTA c(p), local j(p), CZ sign ----
  const uint32_t i = (rank << LB) | uint32_t(tid);
  uint32_t p = i;
  bool neg = false;
  if (entangler == 0) {  // new[i] = old[c_0(c_1(...c_{n-1}(i)))], C_q: control q -> target q+1 mod n
#pragma unroll
    for (int q = n - 1; q >= 0; --q) {
      const int pc = n - 1 - q, pt = n - 1 - ((q + 1) % n);
      if ((p >> pc) & 1u) p ^= 1u << pt;
    }
  } else {  // CZ ring: diagonal (-1)^{sum_q b_q b_{q+1 mod n}}
    int par = 0;
#pragma unroll
    for (int q = 0; q < n; ++q) par ^= int((i >> (n - 1 - q)) & (i >> (n - 1 - (q + 1) % n))) & 1;
    neg = par;
  }
  const uint32_t pc = p >> LB, pj = p & uint32_t(NL - 1);
  const uint32_t pub_base = uint32_t(__cvta_generic_to_shared(pub));
  uint32_t remote[CS];
#pragma unroll
  for (int c = 0; c < CS; ++c) remote[c] = (CS > 1 ? mapa(pub_base, uint32_t(c)) : pub_base) + pj * 16u;
  __syncthreads();  // tables ready

  double2 v = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
  const unsigned full = 0xffffffffu;
  for (int layer = 0; layer < layers; ++layer) {
    const int gl = layer * n;
    // 1. lane bits (positions 0..4): the thread's row of U, partner by shuffle
#pragma unroll
    for (int pos = 0; pos < 5; ++pos) {
      const int g = gl + (n - 1 - pos);
      const int bit = (lane >> pos) & 1;
      const double2 cs = uent(U, g, bit, bit), co = uent(U, g, bit, bit ^ 1);
      const double2 pp = make_double2(__shfl_xor_sync(full, v.x, 1 << pos), __shfl_xor_sync(full, v.y, 1 << pos));
      v = cmac(co, pp, cmul(cs, v));
    }
    // 2. warp bits (positions 5, 6): U_5 (x) U_6 over the 4 partners through SMEM
    sbuf[tid] = v;
    __syncthreads();
    {
      const int x = (tid >> 5) & 3;  // (x6 x5)
      const double2* w = W4 + 16 * layer + 4 * x;
      const double2 a0 = cmac(w[1], sbuf[(tid & 31) | (1 << 5)], cmul(w[0], sbuf[tid & 31]));
      const double2 a1 = cmac(w[3], sbuf[(tid & 31) | (3 << 5)], cmul(w[2], sbuf[(tid & 31) | (2 << 5)]));
      v = make_double2(a0.x + a1.x, a0.y + a1.y);
    }
    // 3. cluster bits + ring: publish, cluster barrier, gather over DSMEM
    const uint32_t par = uint32_t(layer & 1) * (NL * 16u);
    pub[(layer & 1) * NL + tid] = v;
    if (CS > 1) cluster_barrier(); else __syncthreads();
    {
      const double2* gc = GC + CS * CS * layer + CS * pc;
      double2 r[CS];
#pragma unroll
      for (int c = 0; c < CS; ++c) r[c] = ld_dsmem(remote[c] + par);  // all loads in flight first
      // independent partial sums (the 2-DFMA dependency of one complex MAC is the latency unit)
      double2 acc[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                        make_double2(0.0, 0.0)};
#pragma unroll
      for (int c = 0; c < CS; ++c) acc[c & 3] = cmac(gc[c], r[c], acc[c & 3]);
      const double2 s = make_double2((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x),
                                     (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
      v = neg ? make_double2(-s.x, -s.y) : s;
    }
  }
  x_all[(size_t)blockIdx.y * (1u << n) + i] = v;
  if (CS > 1) cluster_barrier();  // peers may still read this CTA's last published layer
}

}  // namespace pclus
}  // namespace dvqls
