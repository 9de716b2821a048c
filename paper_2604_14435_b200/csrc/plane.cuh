// plane.cuh - n = 10, uniform-b Hadamard-test kernel with the branch split into real planes.
//
// SURVEY §8(a) a3-a9 for the headline workload (BASELINE.json cfg3/cfg4: n = 10).
// Same circuit, same gate sequence and the same algorithmic work as hadamard_kernel
// (kernels.cuh), laid out differently:
//
// After the first ancilla H every gate of the Hadamard test (Eq. 4) is a controlled
// signed permutation (c-A_k, c-A_l), a controlled H^{(x)n} (c-U_b, c-U_b^+ for uniform b) or a
// controlled Z_j -- all REAL matrices.  A real matrix acts on Re(phi) and Im(phi) independently,
// so the 2^n complex amplitudes of a circuit's ancilla-|1> branch are two independent real
// vectors ("planes").  A circuit is owned by a warp PAIR: warp 2p holds the Re plane, warp 2p+1
// the Im plane, each lane 32 doubles in registers (64 registers, half of the complex layout's
// 128), so 20 warps fit on an SM instead of 12 and nothing spills.
//
// The readout S = sum_j conj(x'_j) phi_j (x'_j = sgn_l(j) x_{j ^ m_l}) splits per plane:
//     Re S = sum x'_re phi_re + sum x'_im phi_im      (each warp: its own plane of x)
//     Im S = sum x'_re phi_im - sum x'_im phi_re      (each warp: the other plane, Re warp negated)
// and SMEM holds [x_re, -x_re, x_im, -x_im], so plane and sign are address bits.  The two halves
// of a circuit are added by the Re warp every 8 circuits (one 64-thread named barrier per pair),
// which also writes the 8 terms (one coalesced 64-byte store) and accumulates c_l^* c_k (Re + i Im).
//
// Layouts per plane (N = 1024, lane t, register r): A: i = (r << 5) | t;  B: i = (t << 5) | r.
// The exchange buffer has 33-double rows: in both layouts every half-warp's 16 doubles fall in
// 16 distinct 8-byte bank pairs (LDS.64/STS.64, 2 wavefronts) and addresses are base + immediate.
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace plane {

constexpr int NQ = 10, TB = 5, RB = 5, R = 32, N = 1 << NQ;
constexpr int BATCH = 32;                         // circuits per pair combine (one per lane)
constexpr uint32_t ROW = (R + 1) * 8;             // padded exchange row (33 doubles)
constexpr uint32_t BUF = (1u << TB) * ROW;        // exchange buffer per warp: 8448 B
constexpr uint32_t XREG = 4u * N * 8u;            // [x_re, -x_re, x_im, -x_im]: 32 KB
constexpr uint32_t XALIGN = 16384;                // (x_p, -x_p) pair = 16 KB, XOR-addressed
// (the plane offset p * 16 KB is ADDED to the 16 KB-aligned base; only bits 3..13 -- index and
// sign -- are OR/XOR-addressed)

// All SMEM accesses of the hot loop use 32-bit shared-window addresses directly, so the
// per-access address work is at most one LOP3 (gather/readout Gray-code chain) or nothing
// (exchange rows: base register + immediate).  The dynamic-SMEM base is not a link-time
// constant on sm_100 (it carries the CTA's cluster-window bits), so the XOR-addressed x region
// is placed at a 16 KB-aligned window address inside the allocation.
__device__ __forceinline__ uint32_t sbase() { return uint32_t(__cvta_generic_to_shared(dvqls_smem)); }
__device__ __forceinline__ double lds_a(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_a(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
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

// Layout change of one plane through the warp's buffer.  Rows are padded to 33 doubles:
// slot(i) = i + (i >> 5), so layout A (i = r << 5 | t) is t * 8 + r * ROW and layout B
// (i = t << 5 | r) is t * ROW + r * 8 -- a per-lane base plus a compile-time immediate, and in
// both layouts a half-warp's 16 doubles sit in 16 distinct 8-byte bank pairs.
template <bool A_TO_B>
__device__ __forceinline__ void exchange(double (&v)[R], uint32_t baseA, uint32_t baseB) {
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) sts_a(A_TO_B ? baseA + uint32_t(r) * ROW : baseB + uint32_t(r) * 8u, v[r]);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = lds_a(A_TO_B ? baseB + uint32_t(r) * 8u : baseA + uint32_t(r) * ROW);
}

template <int WARPS>
__host__ __device__ constexpr size_t small_bytes() {
  return sizeof(double) * (size_t(WARPS / 2) * 2 * BATCH * 2 + size_t(WARPS / 2) * 4);
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) __maxnreg__(reg_cap<WARPS>())
plane_kernel(const double2* __restrict__ x_all, const PauliTerm* __restrict__ tab, const double2* __restrict__ coef,
             const double2* __restrict__ hv, double hv_scale, int L, int64_t c0, int64_t C, int K,
             double* __restrict__ out_terms, double* __restrict__ partials, int with_cost,
             double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {
  static_assert(WARPS % 2 == 0 && WARPS / 2 <= 15, "warp pairs use named barriers 1..15");
  pdl_wait();
  (void)hv; (void)hv_scale;
  constexpr int NP = WARPS / 2;  // circuit groups (warp pairs) per CTA
  constexpr size_t SMALL = small_bytes<WARPS>();
  // SMEM: slots[NP][2][BATCH][2] | acc[NP][4] | pad to a 16 KB window address |
  //       [x_re, -x_re, x_im, -x_im] | WARPS padded exchange buffers   (host: smem_bytes(sb))
  double* sslot = reinterpret_cast<double*>(dvqls_smem);
  double* sacc = sslot + NP * 2 * BATCH * 2;
  const uint32_t sb = sbase();
  const uint32_t xa = (sb + uint32_t(SMALL) + XALIGN - 1) & ~(XALIGN - 1);  // window address of x
  {
    uint32_t dsz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
    if (xa + XREG + WARPS * BUF - sb > dsz) __trap();  // host sized the allocation for another base
  }
  double* sd = reinterpret_cast<double*>(reinterpret_cast<char*>(dvqls_smem) + (xa - sb));

  const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int pair = warp >> 1;
  const uint32_t pl = uint32_t(warp & 1);
  const uint32_t buf = xa + XREG + uint32_t(warp) * BUF;
  const uint32_t baseA = buf + uint32_t(t) * 8u, baseB = buf + uint32_t(t) * ROW;
  const int n1 = NQ + 1;
  double* slot = sslot + pair * (2 * BATCH * 2);
  double* pacc = sacc + 4 * pair;

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
    const double2* x = x_all + (size_t)kth * N;
    __syncthreads();  // previous phase's readers of the x planes are done
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double2 a = x[i];
      sd[i] = a.x;
      sd[N + i] = -a.x;
      sd[2 * N + i] = a.y;
      sd[3 * N + i] = -a.y;
    }
    __syncthreads();
    int cb, ce;
    {
      int64_t b, e;
      weighted_range(c0 + pa, pb - pa, pair, NP, NQ, &b, &e);
      cb = int(pa + b);
      ce = int(pa + e);
    }
    if (pl == 0 && t == 0) pacc[0] = pacc[1] = pacc[2] = pacc[3] = 0.0;
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
      double v[R];
      // ---- a4: branch init + c-A_k, this plane: phi_i = sgn_k(i ^ m_k) x_pl[i ^ m_k] (layout A)
      {
        const uint32_t mh = Tk.xm >> TB, tl = uint32_t(t) ^ (Tk.xm & 31u), zh = Tk.zm >> TB;
        const uint32_t sg0 = (__popc(tl & Tk.zm & 31u) ^ __popc(mh & zh)) & 1u;
        uint32_t a = (xa + (pl << (NQ + 4))) | (((sg0 << NQ) | (mh << TB) | tl) * 8u);
#pragma unroll
        for (int kk = 0; kk < R; ++kk) {
          const int r = kk ^ (kk >> 1);
          if (kk) {
            const int bb = ctz_c(kk);
            a ^= ((1u << (TB + bb)) | (((zh >> bb) & 1u) << NQ)) * 8u;
          }
          v[r] = lds_a(a);
        }
      }
      double scale = 1.0;
      if (s > 0) {
        const int p = NQ - 1 - (s - 1);  // index bit of Z_j, j = s - 1
        // ---- a5: c-U_b^+ = unnormalised FWHT: layout A register bits (index bits 5..9),
        //      exchange, layout B register bits (index bits 0..4)
        fwht<0, RB>(v);
        exchange<true>(v, baseA, baseB);
        fwht<0, TB>(v);
        // ---- a6: c-Z_j (layout B: register bit p, or lane bit p - 5) ----
        if (p < RB) {
#pragma unroll
          for (int bb = 0; bb < RB; ++bb)
            if (bb == p) {
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (r & (1 << bb)) v[r] = flip(v[r], 0x80000000u);
            }
        } else {
          const uint32_t m = uint32_t((t >> (p - RB)) & 1) << 31;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = flip(v[r], m);
        }
        // ---- a7: c-U_b ----
        fwht<0, TB>(v);
        exchange<false>(v, baseA, baseB);
        fwht<0, RB>(v);
        scale = 1.0 / double(N);
      }
      // ---- a8: c-A_l + readout, this plane's half of Re(i^q S) ----
      const PauliTerm Tl = tab[l];
      const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
      double half;
      {
        const uint32_t qi = uint32_t(q & 1);
        const uint32_t rp = pl ^ qi, xs = qi & (pl ^ 1u);  // plane read, extra sign (Re warp, Im S)
        const uint32_t mh = Tl.xm >> TB, tl = uint32_t(t) ^ (Tl.xm & 31u), zh = Tl.zm >> TB;
        const uint32_t sg0 = (__popc(uint32_t(t) & Tl.zm & 31u) & 1u) ^ xs;
        uint32_t a = (xa + (rp << (NQ + 4))) | (((sg0 << NQ) | (mh << TB) | tl) * 8u);
        double ac[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < R; ++kk) {
          const int r = kk ^ (kk >> 1);
          if (kk) {
            const int bb = ctz_c(kk);
            a ^= ((1u << (TB + bb)) | (((zh >> bb) & 1u) << NQ)) * 8u;
          }
          ac[kk & 3] = fma(lds_a(a), v[r], ac[kk & 3]);
        }
        half = (ac[0] + ac[1]) + (ac[2] + ac[3]);
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) half += __shfl_xor_sync(0xffffffffu, half, off);
      half *= (q == 1 || q == 2) ? -scale : scale;

      // ---- a9 (fused): pair combine every BATCH circuits.  Re-warp lane u owns circuit u of
      // the batch: adds the two plane halves, writes the term (coalesced), decodes (l, k, s, part)
      // and weights by c_l^* c_k; a fixed shuffle tree sums the batch into the pair's quadruple.
      const int j = (cl - cb) & (BATCH - 1);
      double* sl = slot + (((cl - cb) / BATCH) & 1) * (BATCH * 2);
      if (t == 0) sl[2 * j + pl] = half;
      if (j == BATCH - 1 || cl + 1 == ce) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(64) : "memory");
        if (pl == 0) {
          double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
          if (t <= j) {
            const double val = sl[2 * t] + sl[2 * t + 1];
            const int cc = cl - j + t;
            out_terms[(size_t)kth * C + cc] = val;
            const int64_t c = c0 + cc, tk = c >> 1, lk = tk / n1;
            const int prt = int(c & 1), ss = int(tk - lk * n1), kk = int(lk % L), ll = int(lk / L);
            const double2 cl_ = coef[ll], ck = coef[kk];
            const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
            const double cr = (prt == 0 ? wr : -wi) * val, ci = (prt == 0 ? wi : wr) * val;
            if (ss == 0) { e2 = cr; e3 = ci; } else { e0 = cr; e1 = ci; }
          }
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) {
            e0 += __shfl_xor_sync(0xffffffffu, e0, off);
            e1 += __shfl_xor_sync(0xffffffffu, e1, off);
            e2 += __shfl_xor_sync(0xffffffffu, e2, off);
            e3 += __shfl_xor_sync(0xffffffffu, e3, off);
          }
          if (t == 0) { pacc[0] += e0; pacc[1] += e1; pacc[2] += e2; pacc[3] += e3; }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // fixed pair order
      double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
      for (int g = 0; g < NP; ++g) {
        e0 += sacc[4 * g]; e1 += sacc[4 * g + 1]; e2 += sacc[4 * g + 2]; e3 += sacc[4 * g + 3];
      }
      double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
      o[0] = e0; o[1] = e1; o[2] = e2; o[3] = e3;
    }
  }
  if (red_out) finish_all(partials, int(G), K, NQ, with_cost, red_out, counter, p2p);
}

// dynamic SMEM to request when the dynamic base sits at shared-window address sb
template <int WARPS>
__host__ __device__ constexpr size_t smem_bytes(uint32_t sb) {
  return ((sb + small_bytes<WARPS>() + XALIGN - 1) & ~size_t(XALIGN - 1)) - sb + XREG + size_t(WARPS) * BUF;
}

}  // namespace plane
}  // namespace dvqls
