// decomp.cuh - NEXT-4: Pauli decomposition + pruning of a dense A on the GPU,
// Alg. 1 Steps 1-2 (FWHT-based decomposition P:379, 1 % pruning P:490).
//
//   c_{P(m,z)} = tr(P A) / 2^n = i^{popcount(m & z)} / 2^n * sum_k (-1)^{popcount(k & z)} A[k, k ^ m]
//
// P(m, z)|k> = i^{popcount(m&z)} (-1)^{popcount(k&z)} |k ^ m> has one nonzero per column, so for a
// fixed x-mask m the 2^n coefficients are one Walsh-Hadamard transform (over k) of the "XOR
// diagonal" a_m[k] = A[k, k ^ m].  One CTA per m gathers its diagonal straight from A (element k
// from row k: a 16-byte read per row; the CTAs of m, m^1, ..., m^7 -- launched together -- read the
// same 128-byte line of each row, so DRAM delivers A once), runs the FWHT (n >= 9: 16 amplitudes per
// thread in registers, ceil(n/4) register passes joined by SMEM exchanges; n <= 8: radix-2 in SMEM),
// phase and scale.  Round 1 wrote the diagonals as rows of a second matrix B first (A read, B
// written, B read: 48 * 4^n bytes); this reads A once (16 * 4^n).
//
// Pruning needs ||c||_2 before the pass that compacts survivors.  Parseval, sum_P |c_P|^2 =
// ||A||_F^2 / 2^n, gives it up to rounding, and ||A||_F^2 is summed row block by row block as A is
// uploaded (fro_rows_kernel after each chunk of the host-to-device copy, while the chunk is in L2),
// so ONE pass compacts every CANDIDATE |c| >= max(1e-14, eps ||A||_F / 2^{n/2} (1 - 1e-9)) and, in
// the same pass, sums |c|^2 per row in a fixed order; the exact ||c||_2 = sqrt(sum |c|^2) (the
// definition, reading 15) then applies the pruning rule to the candidates inside the sort.
//
// Pruning keeps |c| >= 1e-14 and |c| >= eps * ||c||_2 (reading 15); survivors are sorted by
// (round(|c| / (1e-12 ||c||_2)) descending, lexicographic I<X<Y<Z ascending) in one CTA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dvqls {
namespace decomp {

constexpr int THREADS = 512;

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
constexpr int SORT_MAX = 4096;
constexpr size_t SORT_SMEM = SORT_MAX * (8 + 8 + 4);

// |A|^2 of rows [r0, r0 + gridDim.x * rows_per_cta): CTA b sums its rows in a fixed order into
// fro[r0 / rows_per_cta + b] (run after each chunk of the upload, on the chunk just copied)
__global__ void __launch_bounds__(256) fro_rows_kernel(const double2* __restrict__ A, uint32_t N, uint32_t r0,
                                                       uint32_t rows_per_cta, double* __restrict__ fro) {
  __shared__ double red[8];
  const size_t base = (size_t(r0) + size_t(blockIdx.x) * rows_per_cta) * N;
  const uint32_t cnt = rows_per_cta * N;
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < cnt; i += 256) {
    const double2 a = __ldcg(A + base + i);
    acc = fma(a.x, a.x, fma(a.y, a.y, acc));
  }
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double f = 0.0;
    for (int w = 0; w < 8; ++w) f += red[w];
    fro[r0 / rows_per_cta + blockIdx.x] = f;
  }
}

// candidate threshold from Parseval: thr0 = eps * sqrt(sum fro / 2^n) * (1 - 1e-9) (below the
// exact eps ||c||_2 by far more than the rounding gap), floor 1e-14, stored as the bound on the
// unscaled FWHT value f = 2^n c:  *thrf2 = (2^n thr0)^2;  zeroes the candidate counter
__global__ void __launch_bounds__(256) prenorm_kernel(const double* __restrict__ fro, uint32_t nf, uint32_t N,
                                                      double eps, double* __restrict__ thrf2,
                                                      unsigned long long* __restrict__ count) {
  __shared__ double red[256];
  double a = 0.0;
  for (uint32_t i = threadIdx.x; i < nf; i += 256) a += fro[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int off = 128; off >= 1; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double thr0 = fmax(1e-14, eps * sqrt(red[0] / double(N)) * (1.0 - 1e-9));
    *thrf2 = (thr0 * double(N)) * (thr0 * double(N));
    *count = 0ull;
  }
}

// Epilogue of one coefficient c = i^{popcount(m&z)} f / 2^n (f = FWHT value):
// MODE 0 writes C[m, z];  MODE 1 compacts candidates |f|^2 >= thrf2 (i.e. |c| >= thr0) into
// (idx, C[slot]) and returns |f|^2 for the row's fixed-order sum (scaled by 4^-n once per row:
// a power of two, so sum |c|^2 is exact to the same rounding).  No square root or phase work on
// the common (non-candidate) path.
template <int MODE>
__device__ __forceinline__ double emit_coef(double2 f, uint32_t m, uint32_t z, uint32_t N, double inv, double thrf2,
                                            double2* __restrict__ C, uint64_t cap,
                                            unsigned long long* __restrict__ count, uint64_t* __restrict__ idx) {
  const double a2 = fma(f.x, f.x, f.y * f.y);
  if (MODE == 0 || a2 >= thrf2) {
    const int q = __popc(m & z) & 3;  // i^q
    const double re = (q == 0 ? f.x : q == 1 ? -f.y : q == 2 ? -f.x : f.y) * inv;
    const double im = (q == 0 ? f.y : q == 1 ? f.x : q == 2 ? -f.y : -f.x) * inv;
    if (MODE == 0) {
      C[size_t(m) * N + z] = make_double2(re, im);
    } else {
      const unsigned long long slot = atomicAdd(count, 1ull);
      if (slot < cap) {
        idx[slot] = uint64_t(m) * N + z;
        C[slot] = make_double2(re, im);
      }
    }
  }
  return a2;
}

// CTA sum of per-thread |f|^2 partials in a fixed order, times 4^-n -> sq[m] = sum_z |c_(m,z)|^2
template <int NT>
__device__ __forceinline__ void row_sq(double acc, double* __restrict__ sq, double inv, uint32_t m) {
  __shared__ double red[NT / 32];
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += red[w];  // fixed order
    sq[m] = t * (inv * inv);
  }
}

// n <= 8: radix-2 FWHT of the XOR diagonal m of A in SMEM
template <int MODE>
__global__ void __launch_bounds__(THREADS)
fwht_rows_kernel(const double2* __restrict__ A, int n, double2* __restrict__ C, double* __restrict__ sq,
                 const double* __restrict__ thrf2, uint64_t cap, unsigned long long* __restrict__ count,
                 uint64_t* __restrict__ idx) {
  extern __shared__ double2 rows_smem[];  // dynamic: 2^n amplitudes
  constexpr int NV = 1;
  const uint32_t N = 1u << n;
  const uint32_t m0 = blockIdx.x;
  for (uint32_t k = threadIdx.x; k < N; k += THREADS) rows_smem[k] = __ldcg(A + size_t(k) * N + (k ^ m0));
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
  const double thr = MODE == 1 ? *thrf2 : 0.0;
  double acc = 0.0;
  for (uint32_t z = threadIdx.x; z < N; z += THREADS)
    acc += emit_coef<MODE>(rows_smem[z], m0, z, N, inv, thr, C, cap, count, idx);
  if (MODE == 1) row_sq<THREADS>(acc, sq, inv, blockIdx.x);
}

// n = NB >= 9: XOR diagonal m of A in registers, RG = 16 amplitudes per thread (2^(NB-4) threads).
// Pass g puts index bits [b_g, b_g + 4) in registers (b_0 = NB - 4, b_1 = NB - 8, ..., last 0)
// and butterflies the bits of that window not done before; consecutive passes exchange through
// SMEM (slot(i) = i ^ ((i >> 4) & 7): conflict-free LDS.128/STS.128 in every layout).  Element k
// of the diagonal is A[k, k ^ m] (pass 0 layout, k = r << (NB - 4) | t: one 16-byte read per row).
constexpr int RG = 16;
template <int NB>
__device__ __forceinline__ uint32_t rows_idx(uint32_t t, uint32_t r, int b) {
  return ((t >> b) << (b + 4)) | (r << b) | (t & ((1u << b) - 1u));
}
__device__ __forceinline__ uint32_t rows_slot(uint32_t i) { return i ^ ((i >> 4) & 7u); }

template <int NB, int MODE>
__global__ void __launch_bounds__(1 << (NB - 4), NB <= 12 ? 3 : 1)
fwht_rows_reg_kernel(const double2* __restrict__ A, double2* __restrict__ C, double* __restrict__ sq,
                     const double* __restrict__ thrf2, uint64_t cap, unsigned long long* __restrict__ count,
                     uint64_t* __restrict__ idx) {
  static_assert(NB >= 9 && NB <= 13, "register FWHT rows: 9 <= n <= 13");
  constexpr int NT = 1 << (NB - 4);
  constexpr uint32_t N = 1u << NB;
  constexpr int NPASS = (NB + 3) / 4;
  extern __shared__ double2 rows_smem[];
  const uint32_t t = threadIdx.x, m0 = blockIdx.x;  // one row per CTA (a persistent variant with
  double2 v[RG];                                     // an L2 prefetch of the next row measured slower)
#pragma unroll
  for (int r = 0; r < RG; ++r) {
    const uint32_t k = rows_idx<NB>(t, uint32_t(r), NB - 4);
    v[r] = __ldcg(A + size_t(k) * N + (k ^ m0));
  }
#pragma unroll
  for (int g = 0; g < NPASS; ++g) {
    const int b = NB - 4 * (g + 1) > 0 ? NB - 4 * (g + 1) : 0;  // register window [b, b + 4)
    const int hi = NB - 4 * g;                                    // bits [lo, hi) still to do
    if (g > 0) {
      const int bp = NB - 4 * g > 0 ? NB - 4 * g : 0;  // previous window
#pragma unroll
      for (int r = 0; r < RG; ++r) rows_smem[rows_slot(rows_idx<NB>(t, uint32_t(r), bp))] = v[r];
      __syncthreads();
#pragma unroll
      for (int r = 0; r < RG; ++r) v[r] = rows_smem[rows_slot(rows_idx<NB>(t, uint32_t(r), b))];
      __syncthreads();
    }
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      if (b + bb >= hi) continue;  // done in an earlier window
#pragma unroll
      for (int r = 0; r < RG; ++r)
        if (!(r & (1 << bb))) {
          const double2 p = v[r], q = v[r | (1 << bb)];
          v[r] = make_double2(p.x + q.x, p.y + q.y);
          v[r | (1 << bb)] = make_double2(p.x - q.x, p.y - q.y);
        }
    }
  }
  const double inv = 1.0 / double(N);
  const double thr = MODE == 1 ? *thrf2 : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < RG; ++r)
    acc += emit_coef<MODE>(v[r], m0, rows_idx<NB>(t, uint32_t(r), 0), N, inv, thr, C, cap, count, idx);
  if (MODE == 1) row_sq<NT>(acc, sq, inv, m0);
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

// one CTA: keep the candidates (values C[slot], indices idx[slot] from MODE 1) with |c| >= max(1e-14,
// eps ||c||_2), bitonic-sort them by (quantised |c| desc, lex asc), write the coefficients and the
// Pauli strings (n chars each) in that order and the survivor count *out_L
__global__ void __launch_bounds__(THREADS)
sort_emit_kernel(const double2* __restrict__ C, int n, const uint64_t* __restrict__ idx,
                 const unsigned long long* __restrict__ count, const double* __restrict__ sq,
                 double* __restrict__ norm, double eps, double2* __restrict__ out_c, char* __restrict__ out_s,
                 unsigned long long* __restrict__ out_L) {
  extern __shared__ uint64_t sort_smem[];  // dynamic: SORT_MAX * 20 B
  uint64_t* kq = sort_smem;
  uint64_t* kl = sort_smem + SORT_MAX;
  uint32_t* ki = reinterpret_cast<uint32_t*>(sort_smem + 2 * SORT_MAX);
  {  // ||c||_2 = sqrt(sum_m sq[m]) in a fixed order (strided partials, then a tree); SMEM reused below
    double* red = reinterpret_cast<double*>(sort_smem);
    double a = 0.0;
    const uint32_t nm = 1u << n, per = (nm + THREADS - 1) / THREADS;  // a contiguous chunk per thread,
#pragma unroll 8
    for (uint32_t j = 0; j < per; ++j) {                               // its loads issued together
      const uint32_t i = threadIdx.x * per + j;
      if (i < nm) a += sq[i];
    }
    red[threadIdx.x] = a;
    __syncthreads();
    for (int off = THREADS / 2; off >= 1; off >>= 1) {
      if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
      __syncthreads();
    }
    if (threadIdx.x == 0) *norm = sqrt(red[0]);
    __syncthreads();
  }
  const uint32_t L = uint32_t(min(*count, (unsigned long long)SORT_MAX));  // candidates
  uint32_t P = 1;
  while (P < L) P <<= 1;
  const uint32_t N = 1u << n;
  __threadfence_block();
  const double nrm = *norm;
  const double q = 1e-12 * nrm;
  const double thr = fmax(1e-14, eps * nrm);  // the pruning rule with the exact ||c||_2
  int kept = 0;
  for (uint32_t i = threadIdx.x; i < P; i += THREADS) {
    const double2 c = i < L ? C[i] : make_double2(0.0, 0.0);
    const double a = sqrt(fma(c.x, c.x, c.y * c.y));
    if (i < L && a >= thr) {
      const uint64_t id = idx[i];
      kq[i] = ~uint64_t(llround(a / q));  // descending magnitude
      kl[i] = lex_code(uint32_t(id / N), uint32_t(id % N), n);
      ki[i] = i;
      ++kept;
    } else {
      kq[i] = ~0ull; kl[i] = ~0ull; ki[i] = 0xffffffffu;  // dropped candidates and padding sort last
    }
  }
  __shared__ unsigned s_kept;
  if (threadIdx.x == 0) s_kept = 0u;
  __syncthreads();
  if (kept) atomicAdd(&s_kept, unsigned(kept));
  __syncthreads();
  const uint32_t LK = s_kept;
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
  if (threadIdx.x == 0) *out_L = LK;
  for (uint32_t r = threadIdx.x; r < LK; r += THREADS) {
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

// ---- more than SORT_MAX candidates: the same order with a global bitonic sort --------------
// ||c||_2 = sqrt(sum_m sq[m]) in the fixed order of sort_emit_kernel (one CTA of THREADS)
__global__ void __launch_bounds__(THREADS) norm_kernel(const double* __restrict__ sq, int n, double* __restrict__ norm) {
  __shared__ double red[THREADS];
  double a = 0.0;
  const uint32_t nm = 1u << n, per = (nm + THREADS - 1) / THREADS;
#pragma unroll 8
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t i = threadIdx.x * per + j;
    if (i < nm) a += sq[i];
  }
  red[threadIdx.x] = a;
  __syncthreads();
  for (int off = THREADS / 2; off >= 1; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *norm = sqrt(red[0]);
}

// sort keys of the L candidates, padded to P (a power of two): kept ones (|c| >= max(1e-14,
// eps ||c||_2)) get (~round(|c| / (1e-12 ||c||_2)), lex code), the rest sort last; *kept counts them
__global__ void keys_kernel(const double2* __restrict__ C, const uint64_t* __restrict__ idx, uint64_t L, uint64_t P,
                            int n, const double* __restrict__ norm, double eps, uint64_t* __restrict__ kq,
                            uint64_t* __restrict__ kl, uint32_t* __restrict__ ki, unsigned long long* __restrict__ kept) {
  const double nrm = *norm, q = 1e-12 * nrm, thr = fmax(1e-14, eps * nrm);
  const uint32_t N = 1u << n;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < P; i += uint64_t(gridDim.x) * blockDim.x) {
    const double2 c = i < L ? C[i] : make_double2(0.0, 0.0);
    const double a = sqrt(fma(c.x, c.x, c.y * c.y));
    if (i < L && a >= thr) {
      const uint64_t id = idx[i];
      kq[i] = ~uint64_t(llround(a / q));
      kl[i] = lex_code(uint32_t(id / N), uint32_t(id % N), n);
      ki[i] = uint32_t(i);
      atomicAdd(kept, 1ull);
    } else {
      kq[i] = ~0ull; kl[i] = ~0ull; ki[i] = 0xffffffffu;
    }
  }
}

// one (k, j) step of the bitonic network over P keys (ascending (kq, kl))
__global__ void bitonic_step_kernel(uint64_t* __restrict__ kq, uint64_t* __restrict__ kl, uint32_t* __restrict__ ki,
                                    uint64_t P, uint64_t k, uint64_t j) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < P; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t l = i ^ j;
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
}

// survivors in sorted order: coefficients and Pauli strings
__global__ void emit_kernel(const double2* __restrict__ C, const uint64_t* __restrict__ idx,
                            const uint32_t* __restrict__ ki, const unsigned long long* __restrict__ kept, int n,
                            double2* __restrict__ out_c, char* __restrict__ out_s, unsigned long long* __restrict__ out_L) {
  const uint64_t LK = *kept;
  const uint32_t N = 1u << n;
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_L = LK;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < LK; r += uint64_t(gridDim.x) * blockDim.x) {
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
