// cluster_bench.cu - latency microbenchmark of the pieces of the cluster prefix on this GPU:
// barrier.cluster arrive+wait, a dependent chain of ld.shared::cluster (DSMEM) loads from a peer
// CTA, the same chain on the CTA's own SMEM, and __syncthreads, in SM clock cycles per operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_bench tools/cluster_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned rank_() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned mapa_(unsigned a, unsigned r) { unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ unsigned ldc(unsigned a) { unsigned v; asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; }
__device__ __forceinline__ unsigned lds(unsigned a) { unsigned v; asm volatile("ld.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; }
__device__ __forceinline__ void cbar() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__global__ void __cluster_dims__(8, 1, 1) kern(long long* out, int iters) {
  __shared__ unsigned chain[1024];
  const unsigned r = rank_();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) chain[i] = (unsigned)__cvta_generic_to_shared(&chain[(i + 33) & 1023]);
  cbar();
  long long t0, t1;
  // 1. cluster barrier
  t0 = clock64();
  for (int i = 0; i < iters; ++i) cbar();
  t1 = clock64();
  if (threadIdx.x == 0) out[r * 8 + 0] = (t1 - t0) / iters;
  // 2. dependent DSMEM chain in the next CTA's SMEM (addresses are local-window; remap each hop)
  unsigned peer = (r + 1) & 7;
  unsigned a = mapa_((unsigned)__cvta_generic_to_shared(&chain[threadIdx.x]), peer);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = mapa_(ldc(a), peer);
  t1 = clock64();
  if (threadIdx.x == 0) out[r * 8 + 1] = (t1 - t0) / iters;
  out[r * 8 + 7] = a;
  // 3. same chain in own SMEM
  unsigned b = (unsigned)__cvta_generic_to_shared(&chain[threadIdx.x]);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) b = lds(b);
  t1 = clock64();
  if (threadIdx.x == 0) out[r * 8 + 2] = (t1 - t0) / iters;
  out[r * 8 + 6] = b;
  // 4. __syncthreads
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[r * 8 + 3] = (t1 - t0) / iters;
  // 5. 8 independent DSMEM loads (one per peer) then use: the gather of one layer
  unsigned base = (unsigned)__cvta_generic_to_shared(&chain[threadIdx.x]);
  unsigned rem[8];
  for (int c = 0; c < 8; ++c) rem[c] = mapa_(base, c);
  unsigned s = 0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    unsigned v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = ldc(rem[c] + (s & 4));
#pragma unroll
    for (int c = 0; c < 8; ++c) s += v[c];
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[r * 8 + 4] = (t1 - t0) / iters;
  out[r * 8 + 5] = s;
  cbar();
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  kern<<<8, 128>>>(d, 200);
  kern<<<8, 128>>>(d, 2000);
  long long h[64];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("{\"cluster_barrier_cyc\": %lld, \"dsmem_chain_cyc\": %lld, \"smem_chain_cyc\": %lld, \"syncthreads_cyc\": %lld, "
         "\"dsmem_8_independent_cyc\": %lld, \"err\": \"%s\"}\n",
         h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
