// decomp.cuh - NEXT-4: Pauli decomposition + pruning of a dense A on the GPU,
// Alg. 1 Steps 1-2 (FWHT-based decomposition P:379, 1 % pruning P:490).
//
//   c_{P(m,z)} = tr(P A) / 2^n = i^{popcount(m & z)} / 2^n * sum_k (-1)^{popcount(k & z)} A[k, k ^ m]
//
// P(m, z)|k> = i^{popcount(m&z)} (-1)^{popcount(k&z)} |k ^ m> has one nonzero per column, so for a
// fixed x-mask m the 2^n coefficients are one Walsh-Hadamard transform (over k) of the "XOR
// diagonal" a_m[k] = A[k, k ^ m].  xor_transpose_kernel lays the diagonals out as contiguous
// rows B[m, :] (coalesced tiles), then one CTA per m runs the FWHT in SMEM, phase and scale.
// dvqls_decompose runs that twice (norm pass, then a bitwise-identical recompute that compacts
// the survivors), so no 4^n coefficient array is stored: A read, B written, B read twice =
// 64 * 4^n algorithmic bytes, all coalesced, HBM-bound.
//
// Pruning keeps |c| >= 1e-14 and |c| >= eps * ||c||_2 (reading 15); survivors are compacted and
// sorted by (round(|c| / (1e-12 ||c||_2)) descending, lexicographic I<X<Y<Z ascending) in one CTA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dvqls {
namespace decomp {

constexpr int THREADS = 512;
constexpr int SORT_MAX = 4096;
constexpr size_t SORT_SMEM = SORT_MAX * (8 + 8 + 4);

// XOR-diagonal transposition B[m, k] = A[k, k ^ m] in 32 x 32 tiles: the tile of rows
// [k0, k0+32) x columns [j0, j0+32) holds exactly the elements of B rows M0 + (a ^ b) (M0 =
// (k0 ^ j0) & ~31), columns k0 + a; read along j and written along k, both coalesced.
__global__ void __launch_bounds__(256) xor_transpose_kernel(const double2* __restrict__ A, int n,
                                                            double2* __restrict__ B) {
  __shared__ double2 t[32][33];
  const uint32_t N = 1u << n, tiles = N >> 5;
  const uint32_t k0 = (blockIdx.x / tiles) << 5, j0 = (blockIdx.x % tiles) << 5;
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (uint32_t r = ty; r < 32; r += 8) t[r][tx] = A[size_t(k0 + r) * N + j0 + tx];
  __syncthreads();
  const uint32_t M0 = (k0 ^ j0) & ~31u;
  for (uint32_t ml = ty; ml < 32; ml += 8)  // row M0 + ml of B gets A[k0 + tx, j0 + (tx ^ ml)]
    B[size_t(M0 + ml) * N + k0 + tx] = t[tx][tx ^ ml];
}

// MODE 0: write C[m, :];  MODE 1: only the CTA's sum of |c|^2 (norm pass);  MODE 2: recompute
// and compact the survivors |c| >= max(1e-14, eps ||c||_2) (prune pass; bitwise the same values as
// MODE 0/1, so no 4^n coefficient array is written or re-read).  Row m of B (XOR diagonal m of
// A, contiguous) is read coalesced.  n < 5 (tiny) reads A directly.
template <int MODE>
__global__ void __launch_bounds__(THREADS)
fwht_rows_kernel(const double2* __restrict__ B, int n, double2* __restrict__ C, double* __restrict__ sq,
                 double eps, const double* __restrict__ norm, uint64_t cap, unsigned long long* __restrict__ count,
                 uint64_t* __restrict__ idx, int direct) {
  extern __shared__ double2 rows_smem[];  // dynamic: 2^n amplitudes
  __shared__ double red[THREADS / 32];
  constexpr int NV = 1;
  const uint32_t N = 1u << n;
  const uint32_t m0 = blockIdx.x;
  for (uint32_t k = threadIdx.x; k < N; k += THREADS)
    rows_smem[k] = direct ? __ldg(B + size_t(k) * N + (k ^ m0)) : __ldg(B + size_t(m0) * N + k);
  __syncthreads();
  for (int b = 0; b < n; ++b) {  // radix-2 stages; (a, b) -> (a + b, a - b)
    const uint32_t h = 1u << b;
    for (uint32_t i = threadIdx.x; i < NV * N / 2; i += THREADS) {
      const uint32_t v = i >> (n - 1), j = i & (N / 2 - 1);
      double2* s = rows_smem + v * N;
      const uint32_t lo = ((j >> b) << (b + 1)) | (j & (h - 1)), hi = lo | h;
      const double2 p = s[lo], q = s[hi];
      s[lo] = make_double2(p.x + q.x, p.y + q.y);
      s[hi] = make_double2(p.x - q.x, p.y - q.y);
    }
    __syncthreads();
  }
  const double inv = 1.0 / double(N);
  const double thr = MODE == 2 ? eps * *norm : 0.0;
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < NV * N; i += THREADS) {
    const uint32_t m = m0 + (i >> n), z = i & (N - 1);
    const double2 v = rows_smem[i];
    const int q = __popc(m & z) & 3;  // i^q
    const double re = (q == 0 ? v.x : q == 1 ? -v.y : q == 2 ? -v.x : v.y) * inv;
    const double im = (q == 0 ? v.y : q == 1 ? v.x : q == 2 ? -v.y : -v.x) * inv;
    if (MODE == 0) C[size_t(m) * N + z] = make_double2(re, im);
    if (MODE == 2) {
      const double a = sqrt(fma(re, re, im * im));
      if (a >= 1e-14 && a >= thr) {
        const unsigned long long slot = atomicAdd(count, 1ull);
        if (slot < cap) {
          idx[slot] = uint64_t(m) * N + z;
          C[slot] = make_double2(re, im);  // survivor values, in slot order
        }
      }
    }
    acc = fma(re, re, fma(im, im, acc));
  }
  if (MODE == 2) return;
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < THREADS / 32; ++w) t += red[w];  // fixed order
    sq[blockIdx.x] = t;
  }
}

// ||c||_2 = sqrt(sum_m sq[m]) in a fixed order (one CTA); also zeroes the survivor counter
__global__ void __launch_bounds__(THREADS) norm_kernel(const double* __restrict__ sq, uint32_t N, double* norm,
                                                       unsigned long long* count) {
  __shared__ double red[THREADS];
  double a = 0.0;
  for (uint32_t i = threadIdx.x; i < N; i += THREADS) a += sq[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int off = THREADS / 2; off >= 1; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *norm = sqrt(red[0]);
    *count = 0ull;
  }
}

// lexicographic code of P(m, z): 2 bits per qubit from qubit 0 (MSB), I=0 X=1 Y=2 Z=3
__device__ __forceinline__ uint64_t lex_code(uint32_t m, uint32_t z, int n) {
  uint64_t code = 0;
  for (int q = 0; q < n; ++q) {
    const int b = n - 1 - q;
    const uint32_t xb = (m >> b) & 1u, zb = (z >> b) & 1u;
    code = (code << 2) | (xb ? (zb ? 2u : 1u) : (zb ? 3u : 0u));
  }
  return code;
}

// one CTA: bitonic sort of the L survivors (values C[slot], indices idx[slot] from MODE 2) by (quantised |c| desc, lex asc), then write the
// coefficients and the Pauli strings (n chars each) in that order
__global__ void __launch_bounds__(THREADS)
sort_emit_kernel(const double2* __restrict__ C, int n, const uint64_t* __restrict__ idx,
                 const unsigned long long* __restrict__ count, const double* __restrict__ norm,
                 double2* __restrict__ out_c, char* __restrict__ out_s) {
  extern __shared__ uint64_t sort_smem[];  // dynamic: SORT_MAX * 20 B
  uint64_t* kq = sort_smem;
  uint64_t* kl = sort_smem + SORT_MAX;
  uint32_t* ki = reinterpret_cast<uint32_t*>(sort_smem + 2 * SORT_MAX);
  const uint32_t L = uint32_t(*count);
  uint32_t P = 1;
  while (P < L) P <<= 1;
  const uint32_t N = 1u << n;
  const double q = 1e-12 * *norm;
  for (uint32_t i = threadIdx.x; i < P; i += THREADS) {
    if (i < L) {
      const uint64_t id = idx[i];
      const double2 c = C[i];
      const double a = sqrt(fma(c.x, c.x, c.y * c.y));
      kq[i] = ~uint64_t(llround(a / q));  // descending magnitude
      kl[i] = lex_code(uint32_t(id / N), uint32_t(id % N), n);
      ki[i] = i;
    } else {
      kq[i] = ~0ull; kl[i] = ~0ull; ki[i] = 0xffffffffu;  // padding sorts last
    }
  }
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += THREADS) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const bool gt = kq[i] > kq[l] || (kq[i] == kq[l] && kl[i] > kl[l]);
          if (gt == up) {
            uint64_t t = kq[i]; kq[i] = kq[l]; kq[l] = t;
            t = kl[i]; kl[i] = kl[l]; kl[l] = t;
            const uint32_t u = ki[i]; ki[i] = ki[l]; ki[l] = u;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t r = threadIdx.x; r < L; r += THREADS) {
    const uint64_t id = idx[ki[r]];
    out_c[r] = C[ki[r]];
    const uint32_t m = uint32_t(id / N), z = uint32_t(id % N);
    for (int qq = 0; qq < n; ++qq) {
      const int b = n - 1 - qq;
      const uint32_t xb = (m >> b) & 1u, zb = (z >> b) & 1u;
      out_s[size_t(r) * n + qq] = xb ? (zb ? 'Y' : 'X') : (zb ? 'Z' : 'I');
    }
  }
}

}  // namespace decomp
}  // namespace dvqls
