// pclus_timing.cu - clock64 timestamps of the phases of the cluster prefix (prefix_cluster.cuh),
// thread 0 of CTA 0, n = 10, d = 10: tables, then per layer lane gates / warp step / cluster barrier
// / DSMEM gather.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_14435_b200/csrc -o tools/pclus_timing tools/pclus_timing.cu
#include <cstdio>
#include <vector>
#include "prefix_cluster.cuh"
namespace dvqls { namespace pclus {
template <int NQ>
__global__ void __launch_bounds__(NL)
prefix_cluster_timed(int layers, int entangler, const double* __restrict__ thetas, double2* __restrict__ x_all, long long* ts) {
  int tsi = 0;
#define TS_() do { if (threadIdx.x == 0 && blockIdx.x == 0) ts[tsi] = clock64(); ++tsi; } while (0)
  TS_();
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
  TS_();

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
    TS_();
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
    TS_();
    // 3. cluster bits + ring: publish, cluster barrier, gather over DSMEM
    const uint32_t par = uint32_t(layer & 1) * (NL * 16u);
    pub[(layer & 1) * NL + tid] = v;
    if (CS > 1) cluster_barrier(); else __syncthreads();
    TS_();
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
    TS_();
  }
  x_all[(size_t)blockIdx.y * (1u << n) + i] = v;
  if (CS > 1) cluster_barrier();  // peers may still read this CTA's last published layer
  TS_();
}

}}  // namespace dvqls::pclus
using namespace dvqls::pclus;
int main() {
  const int n = 10, layers = 10, P = 3 * n * layers;
  std::vector<double> th(P);
  for (int i = 0; i < P; ++i) th[i] = 0.37 * i - 3.0;
  double* dth; double2* dx; long long* dts;
  cudaMalloc(&dth, P * 8); cudaMalloc(&dx, 16 << n); cudaMalloc(&dts, 4096 * 8);
  cudaMemcpy(dth, th.data(), P * 8, cudaMemcpyHostToDevice);
  const size_t smem = sizeof(double2) * (3 * NL) + (sizeof(double2) * smem_doubles2<10>(1) - sizeof(double2) * 3 * NL) * layers;
  cudaFuncSetAttribute((const void*)&prefix_cluster_timed<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t lc{}; lc.gridDim = dim3(8, 1); lc.blockDim = dim3(NL); lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 8;
  at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; lc.attrs = at; lc.numAttrs = 1;
  int ent = 0;
  void* args[] = {(void*)&layers, (void*)&ent, (void*)&dth, (void*)&dx, (void*)&dts};
  for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelExC(&lc, (const void*)&prefix_cluster_timed<10>, args);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 20; ++rep) cudaLaunchKernelExC(&lc, (const void*)&prefix_cluster_timed<10>, args);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[64]; cudaMemcpy(h, dts, sizeof h, cudaMemcpyDeviceToHost);
  printf("{\"err\": \"%s\", \"us_per_launch_back_to_back\": %.2f, \"tables_cyc\": %lld", cudaGetErrorString(cudaGetLastError()), 1e3 * ms / 20, h[1] - h[0]);
  long long s[4] = {0, 0, 0, 0};
  for (int l = 0; l < layers; ++l) for (int q = 0; q < 4; ++q) s[q] += h[2 + 4 * l + q] - h[1 + 4 * l + q];
  printf(", \"lane_cyc_per_layer\": %lld, \"warp_cyc_per_layer\": %lld, \"cbar_cyc_per_layer\": %lld, \"gather_cyc_per_layer\": %lld, \"final_cyc\": %lld, \"total_cyc\": %lld}\n",
         s[0] / layers, s[1] / layers, s[2] / layers, s[3] / layers, h[2 + 4 * layers] - h[1 + 4 * layers], h[2 + 4 * layers] - h[0]);
  return 0;
}
