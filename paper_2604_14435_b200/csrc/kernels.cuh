// kernels.cuh - sm_100a kernels of the D-VQLS hot path (arXiv 2604.14435).
//
//   prefix_kernel    SURVEY §8(a) a2: x = V(theta)|0^n> once per theta
//   hadamard_kernel  a3-a9: every Hadamard-test circuit of the rank's block,
//                    one circuit per thread group, state in registers, x in SMEM,
//                    coefficient-weighted partial sums fused in (Alg. 1 4a-4b)
//   reduce_kernel    a9-a10: fixed-order sum of the partials -> (E, Psi) [-> C]
//   finalize_kernel  a10 after the NCCL allreduce: C = 1/2 - Re E / (2 n Re Psi)
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

namespace dvqls {

struct PauliTerm {  // P|j> = i^{ny} (-1)^{popcount(j & zm)} |j ^ xm>, big-endian masks
  uint32_t xm, zm;
  int32_t ny, pad;
};

// sign flip of a double by XOR of the IEEE sign bit (m = 0 or 0x80000000):
// one ALU LOP3 on the high word, no FP64-pipe instruction.
__device__ __forceinline__ double flip(double v, uint32_t m) {
  return __hiloint2double(__double2hiint(v) ^ int(m), __double2loint(v));
}

// ---------------------------------------------------------------------------
// a2: shared ansatz prefix.  One CTA per theta; state in SMEM (n <= 12).
// Each layer: n fused single-qubit unitaries U_q = Ry(t2) Rz(t1) Ry(t0)
// (within-circuit gate fusion of the three rotations on one qubit), then the
// entangling ring as ONE index permutation (CNOT) or ONE diagonal sign (CZ).
// ---------------------------------------------------------------------------
__global__ void prefix_kernel(int n, int layers, int entangler, const double* __restrict__ thetas,
                              double2* __restrict__ x_all) {
  extern __shared__ double2 psm[];
  const int N = 1 << n;
  const int P = 3 * n * layers;
  const int G = n * layers;
  double2* a = psm;
  double2* b = psm + N;
  double2* U = psm + 2 * N;  // 4 entries per fused gate
  const double* th = thetas + (size_t)blockIdx.x * P;

  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    double s0, c0, s1, c1, s2, c2;
    sincos(0.5 * th[3 * g + 0], &s0, &c0);
    sincos(0.5 * th[3 * g + 1], &s1, &c1);
    sincos(0.5 * th[3 * g + 2], &s2, &c2);
    // M = Rz(t1) Ry(t0) = [[e0 c0, -e0 s0], [e1 s0, e1 c0]], e0 = e^{-i t1/2}, e1 = e^{+i t1/2}
    const double2 e0 = make_double2(c1, -s1), e1 = make_double2(c1, s1);
    const double2 m00 = make_double2(e0.x * c0, e0.y * c0), m01 = make_double2(-e0.x * s0, -e0.y * s0);
    const double2 m10 = make_double2(e1.x * s0, e1.y * s0), m11 = make_double2(e1.x * c0, e1.y * c0);
    // U = Ry(t2) M = [[c2 m00 - s2 m10, c2 m01 - s2 m11], [s2 m00 + c2 m10, s2 m01 + c2 m11]]
    U[4 * g + 0] = make_double2(c2 * m00.x - s2 * m10.x, c2 * m00.y - s2 * m10.y);
    U[4 * g + 1] = make_double2(c2 * m01.x - s2 * m11.x, c2 * m01.y - s2 * m11.y);
    U[4 * g + 2] = make_double2(s2 * m00.x + c2 * m10.x, s2 * m00.y + c2 * m10.y);
    U[4 * g + 3] = make_double2(s2 * m01.x + c2 * m11.x, s2 * m01.y + c2 * m11.y);
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) a[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
  __syncthreads();

  for (int layer = 0; layer < layers; ++layer) {
    for (int q = 0; q < n; ++q) {
      const int pos = n - 1 - q;
      const double2 u00 = U[4 * (layer * n + q) + 0], u01 = U[4 * (layer * n + q) + 1];
      const double2 u10 = U[4 * (layer * n + q) + 2], u11 = U[4 * (layer * n + q) + 3];
      for (int p = threadIdx.x; p < N / 2; p += blockDim.x) {
        const int i0 = ((p >> pos) << (pos + 1)) | (p & ((1 << pos) - 1));
        const int i1 = i0 | (1 << pos);
        const double2 va = a[i0], vb = a[i1];
        a[i0] = make_double2(u00.x * va.x - u00.y * va.y + u01.x * vb.x - u01.y * vb.y,
                             u00.x * va.y + u00.y * va.x + u01.x * vb.y + u01.y * vb.x);
        a[i1] = make_double2(u10.x * va.x - u10.y * va.y + u11.x * vb.x - u11.y * vb.y,
                             u10.x * va.y + u10.y * va.x + u11.x * vb.y + u11.y * vb.x);
      }
      __syncthreads();
    }
    if (n >= 2) {
      if (entangler == 0) {
        // CNOT ring C_{n-1} ... C_0 (C_q: control q -> target (q+1) mod n, C_0 first):
        // new[i] = old[c_0(c_1(...c_{n-1}(i)))]
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
          int j = i;
          for (int q = n - 1; q >= 0; --q) {
            const int pc = n - 1 - q, pt = n - 1 - ((q + 1) % n);
            if ((j >> pc) & 1) j ^= 1 << pt;
          }
          b[i] = a[j];
        }
        __syncthreads();
        double2* tmp = a; a = b; b = tmp;
      } else {
        // CZ ring: diagonal (-1)^{sum_q b_q b_{q+1 mod n}}
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
          int par = 0;
          for (int q = 0; q < n; ++q) par ^= ((i >> (n - 1 - q)) & (i >> (n - 1 - (q + 1) % n))) & 1;
          if (par) a[i] = make_double2(-a[i].x, -a[i].y);
        }
        __syncthreads();
      }
    }
  }
  double2* x = x_all + (size_t)blockIdx.x * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) x[i] = a[i];
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

template <int NQ, bool A_TO_B>
__device__ __forceinline__ void exchange(double2 (&v)[Shape<NQ>::R], double2* buf, int t, unsigned gmask) {
  using S = Shape<NQ>;
  __syncwarp(gmask);  // previous readers of buf are done
#pragma unroll
  for (int r = 0; r < S::R; ++r) {
    const int i = A_TO_B ? ((r << S::TB) | t) : ((t << S::RB) | r);
    buf[swz<NQ>(i)] = v[r];
  }
  __syncwarp(gmask);
#pragma unroll
  for (int r = 0; r < S::R; ++r) {
    const int i = A_TO_B ? ((t << S::RB) | r) : ((r << S::TB) | t);
    v[r] = buf[swz<NQ>(i)];
  }
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

template <int NQ, int WARPS, bool HH>
__global__ void __launch_bounds__(WARPS * 32, 1)
hadamard_kernel(const double2* __restrict__ x_all, const PauliTerm* __restrict__ tab,
                const double2* __restrict__ coef, const double2* __restrict__ hv, double hv_scale, int L,
                int64_t c0, int64_t C, double* __restrict__ out_terms, double* __restrict__ partials) {
  using S = Shape<NQ>;
  constexpr int TB = S::TB, RB = S::RB, GT = S::GT, R = S::R, N = S::N, GPW = S::GPW;
  extern __shared__ double2 smem[];
  double2* sx = smem;
  double2* shv = smem + N;
  double2* sbuf = smem + (HH ? 2 : 1) * N;

  const int kth = blockIdx.y;  // theta index within a batch
  const double2* x = x_all + (size_t)kth * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) sx[i] = x[i];
  if (HH)
    for (int i = threadIdx.x; i < N; i += blockDim.x) shv[i] = hv[i];
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane / GT, t = lane % GT;
  const unsigned gmask = (GT == 32) ? 0xffffffffu : (((1u << GT) - 1u) << (gw * GT));
  double2* buf = sbuf + (size_t)(warp * GPW + gw) * N;

  const int64_t NG = (int64_t)gridDim.x * WARPS * GPW;
  const int64_t g = ((int64_t)blockIdx.x * WARPS + warp) * GPW + gw;
  const int64_t cb = g * C / NG, ce = (g + 1) * C / NG;  // local circuit range
  const int n1 = NQ + 1;

  double Er = 0.0, Ei = 0.0, Pr = 0.0, Pi = 0.0;
  for (int64_t cl = cb; cl < ce; ++cl) {
    const int64_t c = c0 + cl;
    const int64_t tk = c >> 1;
    const int part = int(c & 1);
    const int s = int(tk % n1);
    const int64_t lk = tk / n1;
    const int k = int(lk % L), l = int(lk / L);
    const PauliTerm Tk = tab[k], Tl = tab[l];

    // ---- a4: branch init + c-A_k as a signed gather from x (layout A) -----
    double2 v[R];
    {
      const uint32_t mh = Tk.xm >> TB, ml = Tk.xm & (GT - 1), zh = Tk.zm >> TB, zl = Tk.zm & (GT - 1);
      const uint32_t ts = __popc((t ^ ml) & zl) & 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t rr = uint32_t(r) ^ mh;
        const double2 a = sx[(rr << TB) | (t ^ ml)];
        const uint32_t sg = ((__popc(rr & zh) & 1) ^ ts) << 31;
        v[r] = make_double2(flip(a.x, sg), flip(a.y, sg));
      }
    }
    double scale = 1.0;
    if (s > 0) {
      const int p = NQ - 1 - (s - 1);  // bit position of Z_j, j = s - 1
      if (!HH) {
        // ---- a5: c-U_b^+ = unnormalised FWHT ------------------------------
        fwht_regs<R, 0, RB>(v);
        exchange<NQ, true>(v, buf, t, gmask);
        fwht_regs<R, 0, TB>(v);
        // ---- a6: c-Z_j (layout B) -------------------------------------------
        if (p < RB) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint32_t m = uint32_t((r >> p) & 1) << 31;
            v[r] = make_double2(flip(v[r].x, m), flip(v[r].y, m));
          }
        } else {
          const uint32_t m = uint32_t((t >> (p - RB)) & 1) << 31;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = make_double2(flip(v[r].x, m), flip(v[r].y, m));
        }
        // ---- a7: c-U_b ------------------------------------------------------
        fwht_regs<R, 0, TB>(v);
        exchange<NQ, false>(v, buf, t, gmask);
        fwht_regs<R, 0, RB>(v);
        scale = 1.0 / double(N);
      } else {
        householder<NQ>(v, shv, hv_scale, t, gmask);
        if (p >= TB) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint32_t m = uint32_t((r >> (p - TB)) & 1) << 31;
            v[r] = make_double2(flip(v[r].x, m), flip(v[r].y, m));
          }
        } else {
          const uint32_t m = uint32_t((t >> p) & 1) << 31;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = make_double2(flip(v[r].x, m), flip(v[r].y, m));
        }
        householder<NQ>(v, shv, hv_scale, t, gmask);
      }
    }
    // ---- a8: c-A_l + ancilla readout, Re(i^q S) with S = sum_j conj(x_{j^m}) sgn_l(j) phi_j
    const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    {
      const uint32_t mh = Tl.xm >> TB, ml = Tl.xm & (GT - 1), zh = Tl.zm >> TB, zl = Tl.zm & (GT - 1);
      const uint32_t ts = __popc(t & zl) & 1;
      if (q & 1) {  // Im S = sum (xr phi_i - xi phi_r)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2 a = sx[((uint32_t(r) ^ mh) << TB) | (t ^ ml)];
          const uint32_t sg = ((__popc(uint32_t(r) & zh) & 1) ^ ts) << 31;
          const double xr = flip(a.x, sg), xi = flip(a.y, sg ^ 0x80000000u);
          double& acc = (r & 3) == 0 ? acc0 : (r & 3) == 1 ? acc1 : (r & 3) == 2 ? acc2 : acc3;
          acc = fma(xr, v[r].y, acc);
          acc = fma(xi, v[r].x, acc);
        }
      } else {  // Re S = sum (xr phi_r + xi phi_i)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2 a = sx[((uint32_t(r) ^ mh) << TB) | (t ^ ml)];
          const uint32_t sg = ((__popc(uint32_t(r) & zh) & 1) ^ ts) << 31;
          const double xr = flip(a.x, sg), xi = flip(a.y, sg);
          double& acc = (r & 3) == 0 ? acc0 : (r & 3) == 1 ? acc1 : (r & 3) == 2 ? acc2 : acc3;
          acc = fma(xr, v[r].x, acc);
          acc = fma(xi, v[r].y, acc);
        }
      }
    }
    double val = group_sum<GT>((acc0 + acc1) + (acc2 + acc3), gmask);
    val *= (q == 1 || q == 2) ? -scale : scale;

    // ---- a9 (fused): write the term, accumulate c_l^* c_k (Re + i Im) -----
    if (t == 0) {
      out_terms[(size_t)kth * C + cl] = val;
      const double2 cl_ = coef[l], ck = coef[k];
      const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
      const double cr = part == 0 ? wr * val : -wi * val;
      const double ci = part == 0 ? wi * val : wr * val;
      if (s == 0) { Pr += cr; Pi += ci; } else { Er += cr; Ei += ci; }
    }
  }
  if (t == 0) {
    double* o = partials + ((size_t)kth * NG + g) * 4;
    o[0] = Er; o[1] = Ei; o[2] = Pr; o[3] = Pi;
  }
}

// ---------------------------------------------------------------------------
// a9/a10: fixed-order reduction of NG partial quadruples per theta.  One CTA
// per theta, REDUCE_THREADS threads, strided accumulation then a fixed SMEM
// tree: bitwise deterministic for a given launch configuration.
// out: with_cost -> 5 doubles (C, ReE, ImE, RePsi, ImPsi), else 4 (E, Psi).
// ---------------------------------------------------------------------------
constexpr int REDUCE_THREADS = 256;

__device__ __forceinline__ double cost_of(double ReE, double RePsi, int n) {
  return RePsi <= 1e-12 ? __longlong_as_double(0x7ff8000000000000ll) : 0.5 - 0.5 * ReE / (double(n) * RePsi);
}

__global__ void __launch_bounds__(REDUCE_THREADS)
reduce_kernel(const double* __restrict__ partials, int64_t NG, int n, int with_cost, double* __restrict__ out) {
  __shared__ double sh[4][REDUCE_THREADS];
  const double* p = partials + (size_t)blockIdx.x * NG * 4;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int64_t i = threadIdx.x; i < NG; i += REDUCE_THREADS) {
    a0 += p[4 * i + 0]; a1 += p[4 * i + 1]; a2 += p[4 * i + 2]; a3 += p[4 * i + 3];
  }
  sh[0][threadIdx.x] = a0; sh[1][threadIdx.x] = a1; sh[2][threadIdx.x] = a2; sh[3][threadIdx.x] = a3;
  __syncthreads();
  for (int off = REDUCE_THREADS / 2; off >= 1; off >>= 1) {
    if (threadIdx.x < off)
      for (int c = 0; c < 4; ++c) sh[c][threadIdx.x] += sh[c][threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (with_cost) {
      double* o = out + (size_t)blockIdx.x * 5;
      o[0] = cost_of(sh[0][0], sh[2][0], n);
      o[1] = sh[0][0]; o[2] = sh[1][0]; o[3] = sh[2][0]; o[4] = sh[3][0];
    } else {
      double* o = out + (size_t)blockIdx.x * 4;
      o[0] = sh[0][0]; o[1] = sh[1][0]; o[2] = sh[2][0]; o[3] = sh[3][0];
    }
  }
}

// a10 after the cross-rank allreduce: (E, Psi)[K] -> (C, E, Psi)[K]
__global__ void finalize_kernel(const double* __restrict__ ep, int K, int n, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double* e = ep + 4 * k;
  double* o = out + 5 * k;
  o[0] = cost_of(e[0], e[2], n);
  o[1] = e[0]; o[2] = e[1]; o[3] = e[2]; o[4] = e[3];
}

}  // namespace dvqls
