// onchip_plane.cuh - n = 11, 12 (uniform b): the single-tile Hadamard-test circuit on real planes with
// TWO layout exchanges per numerator circuit instead of four.
//
// Same circuit and algorithmic work as the n >= 11 tile kernels (stream.cuh / stream_plane.cuh,
// SURVEY §8(a) a3-a9) and the same real-plane split as plane.cuh (every gate after the first
// ancilla H is a real matrix, so Re(phi) and Im(phi) evolve independently; one thread group runs
// the Re plane, then the Im plane, and adds the two readout halves).  The difference is the
// register blocking: a thread holds 64 doubles (6 register bits), so the 2^n-amplitude plane is
// covered by two layouts of 2^(n-6) threads,
//     A: i = (r << TB) | t   (register bits = index bits [TB, n))      TB = n - 6
//     B: i = (t << 6)  | r   (register bits = index bits [0, 6))
// and each FWHT (c-U_b^+, c-U_b) is "butterflies in A, one exchange, butterflies in B" (n = 11:
// index bit 5 is a register bit in both layouts and is butterflied once, in A).  SMEM carries
// 2 exchanges x 16 B per amplitude per plane instead of the tile kernels' 4.  x is read from a
// planar global copy [x_re | -x_re | x_im | -x_im] (L2-resident, each theta's block aligned to its
// size), so Pauli signs are an address bit and the gather / readout are Gray-code XOR chains on the
// global address, as in plane.cuh on the SMEM one.
//
// Groups: n = 11 one warp, n = 12 two warps (a named barrier per group); 12 warps per CTA and SM
// (168 registers), per-group exchange buffers with rows padded to 65 doubles (slot(i) = i +
// (i >> 6): base + immediate addressing, conflict-free LDS.64/STS.64 in both layouts).
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace onchip {

constexpr int RB = 6, R = 64;
constexpr int WARPS = 12;

__device__ __forceinline__ uint32_t sbase() { return uint32_t(__cvta_generic_to_shared(dvqls_smem)); }
__device__ __forceinline__ double lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
// x block of a theta is aligned to its size (2^(n+5) bytes, host-side), so base + off == base ^ off
// and the Gray-code chain runs on the address itself: one LOP3 per load, no 64-bit adds
__device__ __forceinline__ double ldx(const double* base, uint32_t byte_off) {
  return __ldg(reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(base) ^ uintptr_t(byte_off)));
}

// XS: the x planes [x_re | x_im] staged in SMEM per theta (signs by LOP3 instead of the -x copies);
// fewer groups then fit (n = 11: 10 warps, n = 12: 8 warps).  Default for n = 12, where the x
// reads from L2 (128 KB per theta, no room in L1) stalled the 12-warp kernel: 0.60 vs 0.51 of the
// FP64 pipe at cfg5 n = 12 (profiles/r2_onchip/); n = 11 keeps x in L2 (32 KB, 10 warps no faster).
template <int NQ, bool XS>
constexpr int warps_of() { return XS ? (NQ == 11 ? 10 : 8) : WARPS; }

template <int NQ, bool XS = false>
struct Sh {
  static constexpr int W = warps_of<NQ, XS>();
  static constexpr int TB = NQ - RB;          // thread bits per plane group
  static constexpr int GT = 1 << TB;          // threads per group (32 or 64)
  static constexpr int N = 1 << NQ;
  static constexpr int NG = W * 32 / GT;      // groups per CTA
  static constexpr uint32_t BUFB = uint32_t(N + N / 64) * 8u;  // padded exchange buffer bytes
};
__host__ __device__ constexpr uint32_t pslot(uint32_t i) { return i + (i >> 6); }

template <int NQ, bool XS = false>
__host__ __device__ constexpr size_t smem_bytes() {
  return size_t(Sh<NQ, XS>::NG) * (Sh<NQ, XS>::BUFB + 4 * 8 + 2 * 8) + (XS ? sizeof(double) * 2 * (size_t(1) << NQ) : 0);
}

// xq[K][4][N] = [x_re | -x_re | x_im | -x_im] per theta
__global__ void __launch_bounds__(256) to_planar4_kernel(const double2* __restrict__ x, uint32_t N, uint32_t K,
                                                         double* __restrict__ xq) {
  const size_t total = size_t(N) * K;
  for (size_t i = size_t(blockIdx.x) * 256 + threadIdx.x; i < total; i += size_t(gridDim.x) * 256) {
    const size_t k = i / N, j = i - k * N;
    const double2 a = x[i];
    double* o = xq + 4 * k * N + j;
    o[0] = a.x;
    o[N] = -a.x;
    o[2 * size_t(N)] = a.y;
    o[3 * size_t(N)] = -a.y;
  }
}

template <int B0, int B1>
__device__ __forceinline__ void fwht(double (&v)[R]) {
#pragma unroll
  for (int bb = B0; bb < B1; ++bb) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!(r & (1 << bb))) {
        const double p = v[r], q = v[r | (1 << bb)];
        v[r] = p + q;
        v[r | (1 << bb)] = p - q;
      }
    }
  }
}

template <int GT>
__device__ __forceinline__ void gsync(int group) {
  if constexpr (GT == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(GT) : "memory");
  }
}

// layout change through the group's padded buffer: A (i = r << TB | t) <-> B (i = t << 6 | r)
template <int NQ, bool A_TO_B>
__device__ __forceinline__ void exchange(double (&v)[R], uint32_t buf, uint32_t t, int group) {
  using S = Sh<NQ>;
  const uint32_t a0 = buf + pslot(t) * 8u;          // layout A, r = 0
  const uint32_t b0 = buf + pslot(t << RB) * 8u;    // layout B, r = 0
  gsync<S::GT>(group);  // previous readers of the buffer are done
#pragma unroll
  for (int r = 0; r < R; ++r)
    sts(A_TO_B ? a0 + (pslot(uint32_t(r) << S::TB) - 0u) * 8u : b0 + uint32_t(r) * 8u, v[r]);
  gsync<S::GT>(group);
#pragma unroll
  for (int r = 0; r < R; ++r)
    v[r] = lds(A_TO_B ? b0 + uint32_t(r) * 8u : a0 + pslot(uint32_t(r) << S::TB) * 8u);
}

// Gray-code walk of the signed, XOR-permuted x reads in layout A: register r reads
// (-1)^{sg0 ^ parity(r & zh)} x_plane[((r ^ mh) << TB) | tl]; the sign is plane bit 0 (the -x copy)
template <int NQ>
__device__ __forceinline__ void gather(double (&v)[R], const double* xt, uint32_t pl, uint32_t mh, uint32_t tl,
                                       uint32_t zh, uint32_t sg0) {
  using S = Sh<NQ>;
  uint32_t a = ((((pl << 1) | sg0) << NQ) | (mh << S::TB) | tl) * 8u;
#pragma unroll
  for (int kk = 0; kk < R; ++kk) {
    const int r = kk ^ (kk >> 1);
    if (kk) {
      const int bb = ctz_c(kk);
      a ^= ((1u << (S::TB + bb)) | (((zh >> bb) & 1u) << NQ)) * 8u;
    }
    v[r] = ldx(xt, a);
  }
}

// XS: the same walks over the SMEM planes [x_re | x_im] at shared-window address xs; the Pauli
// sign of register r is sg0 ^ parity(r & zh), toggled along the Gray code, applied by flip()
template <int NQ>
__device__ __forceinline__ void gather_s(double (&v)[R], uint32_t xs, uint32_t pl, uint32_t mh, uint32_t tl,
                                         uint32_t zh, uint32_t sg0) {
  using S = Sh<NQ>;
  // (xs is not aligned to the plane size: the Gray-code chain runs on the offset, added to xs)
  uint32_t a = ((pl << NQ) | (mh << S::TB) | tl) * 8u;
  uint32_t sg = sg0 << 31;
#pragma unroll
  for (int kk = 0; kk < R; ++kk) {
    const int r = kk ^ (kk >> 1);
    if (kk) {
      const int bb = ctz_c(kk);
      a ^= (1u << (S::TB + bb)) * 8u;
      sg ^= ((zh >> bb) & 1u) << 31;
    }
    v[r] = flip(lds(xs + a), sg);
  }
}
template <int NQ>
__device__ __forceinline__ double readout_s(const double (&v)[R], uint32_t xs, uint32_t rp, uint32_t mh, uint32_t tl,
                                            uint32_t zh, uint32_t sg0) {
  using S = Sh<NQ>;
  uint32_t a = ((rp << NQ) | (mh << S::TB) | tl) * 8u;
  uint32_t sg = sg0 << 31;
  double ac[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int kk = 0; kk < R; ++kk) {
    const int r = kk ^ (kk >> 1);
    if (kk) {
      const int bb = ctz_c(kk);
      a ^= (1u << (S::TB + bb)) * 8u;
      sg ^= ((zh >> bb) & 1u) << 31;
    }
    ac[kk & 3] = fma(flip(lds(xs + a), sg), v[r], ac[kk & 3]);
  }
  return (ac[0] + ac[1]) + (ac[2] + ac[3]);
}

template <int NQ>
__device__ __forceinline__ double readout(const double (&v)[R], const double* xt, uint32_t rp, uint32_t mh,
                                          uint32_t tl, uint32_t zh, uint32_t sg0) {
  using S = Sh<NQ>;
  uint32_t a = ((((rp << 1) | sg0) << NQ) | (mh << S::TB) | tl) * 8u;
  double ac[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int kk = 0; kk < R; ++kk) {
    const int r = kk ^ (kk >> 1);
    if (kk) {
      const int bb = ctz_c(kk);
      a ^= ((1u << (S::TB + bb)) | (((zh >> bb) & 1u) << NQ)) * 8u;
    }
    ac[kk & 3] = fma(ldx(xt, a), v[r], ac[kk & 3]);
  }
  return (ac[0] + ac[1]) + (ac[2] + ac[3]);
}

template <int NQ, bool XS = false>
__global__ void __launch_bounds__(warps_of<NQ, XS>() * 32, 1)  // <= 168 registers
onchip_plane_kernel(const double* __restrict__ xq_all, const PauliTerm* __restrict__ tab,
                    const double2* __restrict__ coef, int L, int64_t c0, int64_t C, int K,
                    double* __restrict__ out_terms, double* __restrict__ partials, int with_cost,
                    double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {
  using S = Sh<NQ, XS>;
  constexpr int TB = S::TB, GT = S::GT, N = S::N, NG = S::NG;
  // SMEM: NG padded exchange buffers | acc[NG][4] | half[NG][2] (cross-warp readout sums) | XS: [x_re | x_im]
  const uint32_t sb = sbase();
  double* sacc = reinterpret_cast<double*>(reinterpret_cast<char*>(dvqls_smem) + size_t(NG) * S::BUFB);
  double* shalf = sacc + 4 * NG;
  double* sx = shalf + 2 * NG;  // 16-byte aligned: NG * (BUFB + 48) is a multiple of 16
  const uint32_t xs = sb + uint32_t(size_t(NG) * (S::BUFB + 48));
  const int group = int(threadIdx.x) / GT;
  const uint32_t t = threadIdx.x % GT;
  const uint32_t buf = sb + uint32_t(group) * S::BUFB;
  const int n1 = NQ + 1;
  double* gacc = sacc + 4 * group;

  const int64_t G = gridDim.x;
  const int64_t w0 = wcum(c0, NQ), Wt = wcum(c0 + C, NQ) - w0, Wall = Wt * K;
  auto flat_of = [&](int64_t w) -> int64_t {
    if (w >= Wall) return int64_t(K) * C;
    const int64_t th = w / Wt, rem = w - th * Wt;
    const int64_t c = min(max(winv(w0 + rem, NQ) - c0, int64_t(0)), C);
    return th * C + c;
  };
  const int64_t Fb = Wall > 0 ? flat_of(Wall * (int64_t)blockIdx.x / G) : 0;
  const int64_t Fe =
      Wall <= 0 ? 0 : blockIdx.x + 1 == G ? int64_t(K) * C : flat_of(Wall * ((int64_t)blockIdx.x + 1) / G);
  const int th_first = C > 0 ? int(Fb / C) : 0, th_last = Fe > Fb ? int((Fe - 1) / C) : th_first - 1;
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    if (k < th_first || k > th_last)
      for (int q = 0; q < 4; ++q) partials[(size_t(k) * G + blockIdx.x) * 4 + q] = 0.0;

  for (int kth = th_first; kth <= th_last; ++kth) {
    const int64_t pa = max(Fb, int64_t(kth) * C) - int64_t(kth) * C;
    const int64_t pb = min(Fe, int64_t(kth + 1) * C) - int64_t(kth) * C;
    const double* xt = xq_all + size_t(kth) * 4 * N;
    __syncthreads();  // previous phase's accumulators have been summed (and its x reads done)
    if (XS) {  // stage [x_re | x_im] (planes 0 and 2 of the planar copy)
      for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) sx[i] = xt[i < N ? i : N + i];
      __syncthreads();
    }
    if (t == 0) gacc[0] = gacc[1] = gacc[2] = gacc[3] = 0.0;
    int cb, ce;
    {
      int64_t b, e;
      weighted_range(c0 + pa, pb - pa, group, NG, NQ, &b, &e);
      cb = int(pa + b);
      ce = int(pa + e);
    }
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
      const PauliTerm Tk = tab[k], Tl = tab[l];
      const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
      const uint32_t qi = uint32_t(q & 1);
      double acc = 0.0;
#pragma unroll 1
      for (uint32_t pl = 0; pl < 2; ++pl) {
        double v[R];
        {  // ---- a4: c-A_k on this plane (layout A)
          const uint32_t mh = Tk.xm >> TB, tl = t ^ (Tk.xm & (GT - 1)), zh = Tk.zm >> TB;
          const uint32_t sg0 = (__popc(tl & Tk.zm & (GT - 1)) ^ __popc(mh & zh)) & 1u;
          if (XS) gather_s<NQ>(v, xs, pl, mh, tl, zh, sg0);
          else gather<NQ>(v, xt, pl, mh, tl, zh, sg0);
        }
        if (s > 0) {
          const int p = NQ - 1 - (s - 1);  // index bit of Z_j
          // ---- a5: c-U_b^+: A bits [TB, n), exchange, B bits [0, min(6, TB)) ----
          fwht<0, RB>(v);
          exchange<NQ, true>(v, buf, t, group);
          fwht<0, (TB < RB ? TB : RB)>(v);
          // ---- a6: c-Z_j in layout B: register bit p (p < 6), else thread bit p - 6 ----
          if (p < RB) {
#pragma unroll
            for (int bb = 0; bb < RB; ++bb)
              if (bb == p) {
#pragma unroll
                for (int r = 0; r < R; ++r)
                  if (r & (1 << bb)) v[r] = flip(v[r], 0x80000000u);
              }
          } else {
            const uint32_t m = ((t >> (p - RB)) & 1u) << 31;
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = flip(v[r], m);
          }
          // ---- a7: c-U_b ----
          fwht<0, (TB < RB ? TB : RB)>(v);
          exchange<NQ, false>(v, buf, t, group);
          fwht<0, RB>(v);
        }
        {  // ---- a8: c-A_l + this plane's readout half (Re S: own plane; Im S: the other one)
          const uint32_t rp = pl ^ qi, xsg = qi & (pl ^ 1u);
          const uint32_t mh = Tl.xm >> TB, tl = t ^ (Tl.xm & (GT - 1)), zh = Tl.zm >> TB;
          const uint32_t sg0 = (__popc(t & Tl.zm & (GT - 1)) & 1u) ^ xsg;
          acc += XS ? readout_s<NQ>(v, xs, rp, mh, tl, zh, sg0) : readout<NQ>(v, xt, rp, mh, tl, zh, sg0);
        }
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if constexpr (GT == 64) {  // two warps per group: add the second warp's sum
        const int wig = int(t) >> 5;
        if ((t & 31) == 0) shalf[2 * group + wig] = acc;
        gsync<GT>(group);
        acc = shalf[2 * group] + shalf[2 * group + 1];
        gsync<GT>(group);  // both read before the next circuit's writes
      }
      if (t == 0) {
        double val = acc;
        if (s > 0) val *= 1.0 / double(N);      // two unnormalised FWHTs
        val = (q == 1 || q == 2) ? -val : val;  // Re(i^q S)
        out_terms[(size_t)kth * C + cl] = val;
        const double2 cl_ = coef[l], ck = coef[k];
        const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
        const double cr = part == 0 ? wr * val : -wi * val;
        const double ci = part == 0 ? wi * val : wr * val;
        double* d = gacc + (s == 0 ? 2 : 0);
        d[0] += cr;
        d[1] += ci;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // fixed group order
      double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
      for (int g = 0; g < NG; ++g) {
        e0 += sacc[4 * g]; e1 += sacc[4 * g + 1]; e2 += sacc[4 * g + 2]; e3 += sacc[4 * g + 3];
      }
      double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
      o[0] = e0; o[1] = e1; o[2] = e2; o[3] = e3;
    }
  }
  if (red_out) finish_all(partials, int(G), K, NQ, with_cost, red_out, counter, p2p);
}

}  // namespace onchip
}  // namespace dvqls
