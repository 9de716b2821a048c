// stream.cuh - the n >= 11 Hadamard-test path (north_star item (3)):
// circuits whose 2^n-amplitude ancilla-|1> branch no longer fits one warp's registers.
//
// One CTA owns one circuit at a time.  The branch is processed in tiles of TN = 2^TB
// amplitudes (TB = 12, or 11 for n = 11), 16 amplitudes per thread in registers.  A thread's
// 16 registers cover 4 tile bits; three register layouts cover the tile:
//     LM: register bits = tile bits [4, 8)      lanes on tile bits 0..3 (+8): coalesced
//     LL: register bits = tile bits [0, 4)      SMEM-only (lanes stride 256 B)
//     LH: register bits = tile bits [TB-4, TB)  lanes on tile bits 0..4: coalesced
// Butterflies run on register bits only; moving between layouts is one SMEM exchange
// (STS, barrier, LDS; XOR-swizzled, conflict-free).  Global memory is read straight into
// registers (LM or LH) and written straight from registers: no SMEM staging of I/O.
//
// Tile bits map onto global index bits per pass ("passengers" [0, c) = global [0, c) keep
// 2^c-amplitude segments contiguous; active tile bits [c, TB) = global [b, b + TB - c)):
//     n <= TB : one tile, the whole circuit in registers + SMEM (4 exchanges):
//               gather(LM) F1: LM>LL>LH, Z_j, F2: LH>LL>LM, readout(LM)
//     n <= 22 : g0 = global bits [0,12), g1 = [12, n); 3 passes over a per-CTA scratch
//               P0: gather(LM) F1(g0) LM>LL>LH store(LH)
//               P1: load F1(g1) Z_j F2(g1) store           (0, 2 or 4 exchanges)
//               P2: load(LH) F2(g0) LH>LL>LM readout(LM)
//     n = 23,24: g1 = [12, 21), g2 = [21, n); 5 passes (F1 g1 and F2 g1 separately)
// HBM per numerator circuit: 16N (P0 store) + 32N (P1) + 16N (P2 load) + x reads 32N (L2
// resident for n <= 22): the SURVEY §8(d) streaming model, 96N.  Every circuit is simulated
// on its own (no sharing between circuits).
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace stream {

template <int TB>
struct TS {
  static constexpr int TN = 1 << TB;
  static constexpr int THREADS = TN >> 4;  // 16 amplitudes per thread
  static constexpr int SH = TB - 4;        // register base bit of layout LH
};

constexpr int LL_ = 0, LM_ = 4;

// tile element held by (thread t, register r) in the layout with register bits [S, S+4)
template <int S>
__device__ __forceinline__ uint32_t lelem(uint32_t t, uint32_t r) {
  return ((t >> S) << (S + 4)) | (r << S) | (t & ((1u << S) - 1u));
}

// SMEM slot: XOR of tile bits 0..2 with bits 4..6 -> every layout is conflict-free per
// quarter-warp (8 x 16 B).  GF(2)-linear: slot(a ^ b) = slot(a) ^ slot(b).
__device__ __forceinline__ uint32_t slot(uint32_t e) { return e ^ ((e >> 4) & 7u); }

// FWHT butterflies (a, b) -> (a + b, a - b) on register bit i, for the tile bits of layout S
// that are in [lo, hi).  Stage ownership: LL bits 0..3, LM bits 4..7, LH bits 8..TB-1.
template <int S, int TB>
__device__ __forceinline__ void stages(double2 (&v)[16], int lo, int hi) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = S + i;
    if (S == TS<TB>::SH && q < 8) continue;  // TB = 11: bit 7 belongs to LM
    if (q >= lo && q < hi) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (!(r & (1 << i))) {
          const double2 p = v[r], w = v[r | (1 << i)];
          v[r] = make_double2(p.x + w.x, p.y + w.y);
          v[r | (1 << i)] = make_double2(p.x - w.x, p.y - w.y);
        }
    }
  }
}

// layout SA -> layout SB through the CTA's SMEM tile buffer.  Addresses are walked in
// Gray-code order from a base the compiler cannot hoist (opaque t): one LOP3 per access
// and no loop-invariant address set kept live across the tile loops.
template <int SA, int SB>
__device__ __forceinline__ void xchg(double2 (&v)[16], double2* sm, uint32_t t) {
  const uint32_t to = opaque(t, 0xffffffffu);
  __syncthreads();  // previous readers of the buffer are done
  {
    uint32_t a = slot(lelem<SA>(to, 0));
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k) a ^= slot(1u << (SA + ctz_c(k)));
      sm[a] = v[k ^ (k >> 1)];
    }
  }
  __syncthreads();
  {
    uint32_t a = slot(lelem<SB>(to, 0));
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k) a ^= slot(1u << (SB + ctz_c(k)));
      v[k ^ (k >> 1)] = sm[a];
    }
  }
}

// &base[idx] as one IMAD.WIDE.U32 (idx < 2^28): keeps the per-element address to one
// instruction instead of a 64-bit add chain
__device__ __forceinline__ const double2* at(const double2* base, uint32_t idx) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, 16, %2;" : "=l"(r) : "r"(idx), "l"(base));
  return reinterpret_cast<const double2*>(r);
}
__device__ __forceinline__ double2* at(double2* base, uint32_t idx) {
  return const_cast<double2*>(at(const_cast<const double2*>(base), idx));
}

// Tile-to-global map of one pass: passengers [0, c), active tile bits at global [b, ...)
struct Geo {
  int c, b, tb;
  __device__ __forceinline__ uint32_t gpos(int q) const { return q < c ? q : b + q - c; }
  __device__ __forceinline__ uint32_t gidx(uint32_t e, uint32_t tau) const {
    const uint32_t a = tb - c;
    const uint32_t low = e & ((1u << c) - 1u), act = e >> c;
    const uint32_t mid = tau & ((1u << (b - c)) - 1u), hi = tau >> (b - c);
    return low | (mid << c) | (act << b) | (hi << (b + a));
  }
};

// Bulk L2 prefetch of tile tau of a pass (cp.async.bulk.prefetch.L2): issued one tile ahead,
// so the register loads of the next tile hit L2 instead of waiting on HBM.  The tile is
// contiguous (64 KB) when its active bits continue its passengers (b == c), else 2^(tb-c)
// runs of 2^c amplitudes.  `flip_hi` relocates the tile (x gathered at j ^ m: m's bits above
// the tile select another contiguous tile; its low bits only permute inside it).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tile(const double2* __restrict__ base, const Geo& g, uint32_t tau,
                                              uint32_t flip_hi, uint32_t t, uint32_t nthreads) {
  if (g.b == g.c) {
    const uint32_t chunk = (1u << g.tb) / 16u;  // 16 requests of 4 KB (TB = 12)
    if (t < 16u) prefetch_l2(base + ((g.gidx(t * chunk, tau)) ^ flip_hi), chunk * 16u);
  } else {
    const uint32_t runs = 1u << (g.tb - g.c);
    for (uint32_t u = t; u < runs; u += nthreads) prefetch_l2(base + (g.gidx(u << g.c, tau) ^ flip_hi), 16u << g.c);
  }
}

// Global indices of a thread's 16 registers in layout S: j_r = jb ^ (sum of r's bit columns)
template <int S>
struct Cols {
  uint32_t jb, o[4];
  __device__ __forceinline__ Cols(const Geo& g, uint32_t t, uint32_t tau) {
    jb = g.gidx(lelem<S>(t, 0), tau);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = 1u << g.gpos(S + i);
  }
  __device__ __forceinline__ uint32_t j(int r) const {
    uint32_t v = jb;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (r & (1 << i)) v ^= o[i];
    return v;
  }
  // Gray-code walk: visit k = 0..15 as r_k = k ^ (k >> 1); j_{r_k} = j_{r_{k-1}} ^ o[ctz(k)]
  // (the walk starts from an opaque copy of jb: a load and a store of the same registers do
  //  not share 16 live addresses across the butterflies between them)
  __device__ __forceinline__ uint32_t step(uint32_t jprev, int k) const {
    return k ? jprev ^ o[ctz_c(k)] : opaque(jb, 0xffffffffu);
  }
  // 16-bit word: bit r = parity(j_r & m) ^ parity(jb & m)
  __device__ __forceinline__ uint32_t parity_word(uint32_t m) const {
    uint32_t w = 0;
    w ^= (o[0] & m) ? 0xAAAAu : 0u;
    w ^= (o[1] & m) ? 0xCCCCu : 0u;
    w ^= (o[2] & m) ? 0xF0F0u : 0u;
    w ^= (o[3] & m) ? 0xFF00u : 0u;
    return w;
  }
};

// sign mask (0 or 0x80000000) of register r from a parity word (bit r = sign of register r).
// The word goes through opaque() so the compiler cannot hoist its 16 shifted copies out of
// the tile loops (they are one SHF each to recompute).
__device__ __forceinline__ uint32_t sword(uint32_t word, uint32_t base) {
  return opaque(word ^ (base ? 0xFFFFu : 0u), 0xffffffffu);
}
__device__ __forceinline__ uint32_t smask(uint32_t w, int r) { return (w << (31 - r)) & 0x80000000u; }

// v_r = sgn_k(j_r ^ m) x[j_r ^ m],  sgn_k(i) = (-1)^{popcount(i & z)}  (c-A_k)
template <int S>
__device__ __forceinline__ void gather(double2 (&v)[16], const double2* __restrict__ x, const Cols<S>& cc,
                                       uint32_t m, uint32_t z) {
  const uint32_t w = sword(cc.parity_word(z), __popc((cc.jb ^ m) & z) & 1u);
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int r = k ^ (k >> 1);
    jj = cc.step(jj, k);
    const double2 a = __ldg(at(x, jj ^ m));
    const uint32_t f = smask(w, r);
    v[r] = make_double2(flip(a.x, f), flip(a.y, f));
  }
}

// readout (c-A_l, a8): sum_r Re or Im of conj(sgn_l(j_r) x[j_r ^ m]) v_r
template <int S, bool IM>
__device__ __forceinline__ double readout_t(const double2 (&v)[16], const double2* __restrict__ x, const Cols<S>& cc,
                                            uint32_t m, uint32_t z) {
  const uint32_t w = sword(cc.parity_word(z), __popc(cc.jb & z) & 1u);
  double a0 = 0.0, a1 = 0.0;
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int r = k ^ (k >> 1);
    if (k == 8) asm volatile("" ::: "memory");  // at most 8 x loads in flight (register cap)
    jj = cc.step(jj, k);
    const double2 a = __ldg(at(x, jj ^ m));
    const uint32_t f = smask(w, r);
    const double xr = flip(a.x, f), xi = flip(a.y, f);
    if (k & 1) {
      a1 = IM ? fma(xr, v[r].y, fma(-xi, v[r].x, a1)) : fma(xr, v[r].x, fma(xi, v[r].y, a1));
    } else {
      a0 = IM ? fma(xr, v[r].y, fma(-xi, v[r].x, a0)) : fma(xr, v[r].x, fma(xi, v[r].y, a0));
    }
  }
  return a0 + a1;
}

template <int S>
__device__ __forceinline__ double readout(const double2 (&v)[16], const double2* __restrict__ x, const Cols<S>& cc,
                                          uint32_t m, uint32_t z, bool im) {
  return im ? readout_t<S, true>(v, x, cc, m, z) : readout_t<S, false>(v, x, cc, m, z);
}

// c-Z_j (a6): v_r = -v_r where global bit p of j_r is set
template <int S>
__device__ __forceinline__ void zsign(double2 (&v)[16], const Cols<S>& cc, int p) {
  const uint32_t w = sword(cc.parity_word(1u << p), (cc.jb >> p) & 1u);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t f = smask(w, r);
    v[r] = make_double2(flip(v[r].x, f), flip(v[r].y, f));
  }
}

template <int S>
__device__ __forceinline__ void gload(double2 (&v)[16], const double2* __restrict__ src, const Cols<S>& cc) {
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    jj = cc.step(jj, k);
    v[k ^ (k >> 1)] = __ldcg(at(src, jj));
  }
}

template <int S>
__device__ __forceinline__ void gstore(const double2 (&v)[16], double2* __restrict__ dst, const Cols<S>& cc) {
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    jj = cc.step(jj, k);
    __stcg(at(dst, jj), v[k ^ (k >> 1)]);
  }
}

__device__ __forceinline__ double block_sum(double v, double* red, int nthreads) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nthreads / 32; ++w) tot += red[w];  // fixed order
  return tot;  // valid in thread 0
}

// Householder U_b (n <= TB, one tile, layout LM): v <- v - hv_scale (h^+ v) h   (reading 5)
__device__ __forceinline__ void householder(double2 (&v)[16], const double2* __restrict__ hv, const Cols<LM_>& cc,
                                            double hv_scale, double* red, double* bc, int nthreads) {
  double dr = 0.0, di = 0.0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double2 h = __ldg(hv + cc.j(r));
    dr = fma(h.x, v[r].x, fma(h.y, v[r].y, dr));
    di = fma(h.x, v[r].y, fma(-h.y, v[r].x, di));
  }
  dr = block_sum(dr, red, nthreads);
  di = block_sum(di, red, nthreads);
  if (threadIdx.x == 0) { bc[0] = dr * hv_scale; bc[1] = di * hv_scale; }
  __syncthreads();
  dr = bc[0]; di = bc[1];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double2 h = __ldg(hv + cc.j(r));
    v[r].x -= dr * h.x - di * h.y;
    v[r].y -= dr * h.y + di * h.x;
  }
}

__device__ __forceinline__ int ngroups(int n, int TB) { return n <= TB ? 1 : (n <= 22 ? 2 : 3); }

// group gi of the bit partition (see header)
__device__ __forceinline__ Geo group(int n, int gi, int TB) {
  Geo g;
  g.tb = TB;
  if (gi == 0) { g.c = 0; g.b = 0; }
  else if (gi == 1) { const int a = n <= 22 ? n - 12 : 9; g.c = TB - a; g.b = 12; }
  else { const int a = n - 21; g.c = TB - a; g.b = 21; }
  return g;
}

// One pass over the branch of one circuit for group g of a multi-pass (n > TB) circuit.
// kind: 0 = F1 only, 1 = F1 + Z_j + F2 (middle), 2 = F2 only.
// (C = g.c is a template parameter: with constant stage bounds the butterfly code has no
//  run-time branches, so no register copies at their joins)
template <int TB, int C>
__device__ __forceinline__ void mid_pass_c(double2* __restrict__ phi, double2* sm, const Geo& g, int kind, int p,
                                           uint32_t t0, uint32_t t1, uint32_t t) {
  constexpr int lo = C, hi = TB;
  constexpr bool needLM = lo < 8, needLL = lo < 4;
  for (uint32_t tau = t0; tau < t1; ++tau) {
    if (tau + 1 < t1) prefetch_tile(phi, g, tau + 1, 0u, t, TS<TB>::THREADS);
    double2 v[16];
    if (!needLM) {  // all active bits in LH: no exchange
      const Cols<TS<TB>::SH> cc(g, t, tau);
      gload(v, phi, cc);
      stages<TS<TB>::SH, TB>(v, lo, hi);
      if (kind == 1) { zsign(v, cc, p); stages<TS<TB>::SH, TB>(v, lo, hi); }
      gstore(v, phi, cc);
    } else if (kind == 2) {  // F2 only: LH > (LL) > LM, store LM
      const Cols<TS<TB>::SH> ch(g, t, tau);
      gload(v, phi, ch);
      stages<TS<TB>::SH, TB>(v, lo, hi);
      if (needLL) {
        xchg<TS<TB>::SH, LL_>(v, sm, t);
        stages<LL_, TB>(v, lo, hi);
        xchg<LL_, LM_>(v, sm, t);
      } else {
        xchg<TS<TB>::SH, LM_>(v, sm, t);
      }
      stages<LM_, TB>(v, lo, hi);
      gstore(v, phi, Cols<LM_>(g, t, tau));
    } else {  // F1 [+ Z + F2]: LM > (LL) > LH [Z LH > (LL) > LM]
      const Cols<LM_> cm(g, t, tau);
      gload(v, phi, cm);
      stages<LM_, TB>(v, lo, hi);
      if (needLL) {
        xchg<LM_, LL_>(v, sm, t);
        stages<LL_, TB>(v, lo, hi);
        xchg<LL_, TS<TB>::SH>(v, sm, t);
      } else {
        xchg<LM_, TS<TB>::SH>(v, sm, t);
      }
      stages<TS<TB>::SH, TB>(v, lo, hi);
      if (kind == 0) {
        gstore(v, phi, Cols<TS<TB>::SH>(g, t, tau));
      } else {
        zsign(v, Cols<TS<TB>::SH>(g, t, tau), p);
        stages<TS<TB>::SH, TB>(v, lo, hi);
        if (needLL) {
          xchg<TS<TB>::SH, LL_>(v, sm, t);
          stages<LL_, TB>(v, lo, hi);
          xchg<LL_, LM_>(v, sm, t);
        } else {
          xchg<TS<TB>::SH, LM_>(v, sm, t);
        }
        stages<LM_, TB>(v, lo, hi);
        gstore(v, phi, cm);
      }
    }
  }
}

template <int TB>
__device__ __forceinline__ void mid_pass(double2* __restrict__ phi, double2* sm, const Geo& g, int kind, int p,
                                         uint32_t t0, uint32_t t1, uint32_t t) {
  switch (g.c) {
    case 2: mid_pass_c<TB, 2>(phi, sm, g, kind, p, t0, t1, t); break;
    case 3: mid_pass_c<TB, 3>(phi, sm, g, kind, p, t0, t1, t); break;
    case 4: mid_pass_c<TB, 4>(phi, sm, g, kind, p, t0, t1, t); break;
    case 5: mid_pass_c<TB, 5>(phi, sm, g, kind, p, t0, t1, t); break;
    case 6: mid_pass_c<TB, 6>(phi, sm, g, kind, p, t0, t1, t); break;
    case 7: mid_pass_c<TB, 7>(phi, sm, g, kind, p, t0, t1, t); break;
    case 8: mid_pass_c<TB, 8>(phi, sm, g, kind, p, t0, t1, t); break;
    case 9: mid_pass_c<TB, 9>(phi, sm, g, kind, p, t0, t1, t); break;
    case 10: mid_pass_c<TB, 10>(phi, sm, g, kind, p, t0, t1, t); break;
    default: mid_pass_c<TB, 11>(phi, sm, g, kind, p, t0, t1, t); break;
  }
}

// P0 of a multi-pass numerator circuit on tiles [t0, t1): gather (c-A_k) + F1 on bits 0..TB-1
template <int TB>
__device__ __forceinline__ void first_pass(double2* __restrict__ phi, const double2* __restrict__ x, double2* sm,
                                           const Geo& g0, const PauliTerm& Tk, bool big_x, uint32_t t0, uint32_t t1,
                                           uint32_t t) {
  constexpr int SH = TS<TB>::SH;
  for (uint32_t tau = t0; tau < t1; ++tau) {
    if (big_x && tau + 1 < t1) prefetch_tile(x, g0, tau + 1, Tk.xm & ~uint32_t(TS<TB>::TN - 1), t, TS<TB>::THREADS);
    double2 v[16];
    gather(v, x, Cols<LM_>(g0, t, tau), Tk.xm, Tk.zm);
    stages<LM_, TB>(v, 0, TB);
    xchg<LM_, LL_>(v, sm, t);
    stages<LL_, TB>(v, 0, TB);
    xchg<LL_, SH>(v, sm, t);
    stages<SH, TB>(v, 0, TB);
    gstore(v, phi, Cols<SH>(g0, t, tau));
  }
}

// last pass on tiles [t0, t1): F2 on bits 0..TB-1 + readout (c-A_l); returns this thread's sum
template <int TB>
__device__ __forceinline__ double last_pass(const double2* __restrict__ phi, const double2* __restrict__ x,
                                            double2* sm, const Geo& g0, const PauliTerm& Tl, bool im, bool big_x,
                                            uint32_t t0, uint32_t t1, uint32_t t) {
  constexpr int SH = TS<TB>::SH;
  double acc = 0.0;
  for (uint32_t tau = t0; tau < t1; ++tau) {
    if (tau + 1 < t1) {
      prefetch_tile(phi, g0, tau + 1, 0u, t, TS<TB>::THREADS);
      if (big_x) prefetch_tile(x, g0, tau + 1, Tl.xm & ~uint32_t(TS<TB>::TN - 1), t, TS<TB>::THREADS);
    }
    double2 v[16];
    gload(v, phi, Cols<SH>(g0, t, tau));
    stages<SH, TB>(v, 0, TB);
    xchg<SH, LL_>(v, sm, t);
    stages<LL_, TB>(v, 0, TB);
    xchg<LL_, LM_>(v, sm, t);
    stages<LM_, TB>(v, 0, TB);
    acc += readout(v, x, Cols<LM_>(g0, t, tau), Tl.xm, Tl.zm, im);
  }
  return acc;
}

// denominator circuit on tiles [t0, t1): sum_j conj(sgn_l(j) x_{j^m_l}) sgn_k(j^m_k) x_{j^m_k}
template <int TB>
__device__ __forceinline__ double den_pass(const double2* __restrict__ x, const Geo& g0, const PauliTerm& Tk,
                                           const PauliTerm& Tl, bool im, uint32_t t0, uint32_t t1, uint32_t t) {
  double acc = 0.0;
  for (uint32_t tau = t0; tau < t1; ++tau) {
    const Cols<LM_> cm(g0, t, tau);
    double2 v[16];
    gather(v, x, cm, Tk.xm, Tk.zm);
    acc += readout(v, x, cm, Tl.xm, Tl.zm, im);
  }
  return acc;
}

template <int TB, bool HH>
__global__ void __launch_bounds__(TS<TB>::THREADS, 2)
stream_hadamard_kernel(const double2* __restrict__ x_all, const PauliTerm* __restrict__ tab,
                       const double2* __restrict__ coef, const double2* __restrict__ hv, double hv_scale, int L,
                       int n, int64_t c0, int64_t C, const int64_t* __restrict__ cidx, double2* __restrict__ scratch,
                       double* __restrict__ out_terms, double* __restrict__ partials, int with_cost,
                       double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {
  using T = TS<TB>;
  constexpr int SH = T::SH;
  double2* sm = dvqls_smem;  // TN amplitudes (exchange buffer)
  __shared__ double red[T::THREADS / 32];
  __shared__ double bc[2];
  __shared__ double acc4[4];
  const int kth = blockIdx.y;
  const uint32_t N = 1u << n;
  const double2* __restrict__ x = x_all + (size_t)kth * N;
  double2* __restrict__ phi = scratch + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * N;  // n > TB only
  const int ng = ngroups(n, TB);
  const uint32_t t = threadIdx.x;
  const int64_t G = gridDim.x;
  const int64_t cb = (int64_t)blockIdx.x * C / G, ce = ((int64_t)blockIdx.x + 1) * C / G;
  const uint32_t ntiles = N > uint32_t(T::TN) ? N >> TB : 1u;
  const Geo g0 = group(n, 0, TB);
  const bool big_x = n > 22;  // x tiles prefetched too (measured at n = 22: no gain, x of 2 thetas ~ L2)
  if (t == 0) acc4[0] = acc4[1] = acc4[2] = acc4[3] = 0.0;

  for (int64_t cl = cb; cl < ce; ++cl) {
    const int64_t c = cidx ? cidx[cl] : c0 + cl;
    const int64_t tk = c >> 1;
    const int part = int(c & 1);
    const int sidx = int(tk % (n + 1));
    const int64_t lk = tk / (n + 1);
    const int k = int(lk % L), l = int(lk / L);
    const PauliTerm Tk = tab[k], Tl = tab[l];
    const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
    const bool im = q & 1;
    double acc = 0.0;
    if (sidx == 0) {
      // ---- denominator: <x| A_l A_k |x> term, straight from x
      acc = den_pass<TB>(x, g0, Tk, Tl, im, 0, ntiles, t);
    } else if (n <= TB) {
      // ---- one tile: the whole numerator circuit on chip
      const int p = n - 1 - (sidx - 1);  // Z_j bit position, j = s - 1
      const Cols<LM_> cm(g0, t, 0);
      double2 v[16];
      gather(v, x, cm, Tk.xm, Tk.zm);
      if (HH) {
        householder(v, hv, cm, hv_scale, red, bc, T::THREADS);
        zsign(v, cm, p);
        householder(v, hv, cm, hv_scale, red, bc, T::THREADS);
      } else {
        stages<LM_, TB>(v, 0, TB);
        xchg<LM_, LL_>(v, sm, t);
        stages<LL_, TB>(v, 0, TB);
        xchg<LL_, SH>(v, sm, t);
        stages<SH, TB>(v, 0, TB);
        zsign(v, Cols<SH>(g0, t, 0), p);
        stages<SH, TB>(v, 0, TB);
        xchg<SH, LL_>(v, sm, t);
        stages<LL_, TB>(v, 0, TB);
        xchg<LL_, LM_>(v, sm, t);
        stages<LM_, TB>(v, 0, TB);
      }
      acc = readout(v, x, cm, Tl.xm, Tl.zm, im);
    } else {
      // ---- multi-pass numerator circuit through the CTA's scratch
      const int p = n - 1 - (sidx - 1);
      first_pass<TB>(phi, x, sm, g0, Tk, big_x, 0, ntiles, t);
      __syncthreads();
      if (ng == 2) {
        mid_pass<TB>(phi, sm, group(n, 1, TB), 1, p, 0, ntiles, t);
      } else {
        mid_pass<TB>(phi, sm, group(n, 1, TB), 0, p, 0, ntiles, t);
        __syncthreads();
        mid_pass<TB>(phi, sm, group(n, 2, TB), 1, p, 0, ntiles, t);
        __syncthreads();
        mid_pass<TB>(phi, sm, group(n, 1, TB), 2, p, 0, ntiles, t);
      }
      __syncthreads();
      acc = last_pass<TB>(phi, x, sm, g0, Tl, im, big_x, 0, ntiles, t);
      __syncthreads();  // scratch reads of this circuit done before the next circuit's P0
    }
    double val = block_sum(acc, red, T::THREADS);
    if (t == 0) {
      if (sidx > 0 && !HH) val *= 1.0 / double(N);  // two unnormalised FWHTs
      val = (q == 1 || q == 2) ? -val : val;        // i^q phase: Re(i^q S)
      out_terms[(size_t)kth * C + cl] = val;
      const double2 cl_ = coef[l], ck = coef[k];
      const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
      const double cr = part == 0 ? wr * val : -wi * val;
      const double ci = part == 0 ? wi * val : wr * val;
      if (sidx == 0) { acc4[2] += cr; acc4[3] += ci; } else { acc4[0] += cr; acc4[1] += ci; }
    }
  }
  if (t == 0) {
    double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
    o[0] = acc4[0]; o[1] = acc4[1]; o[2] = acc4[2]; o[3] = acc4[3];
  }
  if (red_out) finish_partials(partials, G, kth, n, with_cost, red_out, counter, p2p.world > 1 ? &p2p : nullptr);
}

// Householder U_b for n > TB (SURVEY §8(c) reading 5; "fixed unitary U_b", P:505 general b):
// U_b^+ and U_b act on the branch as phi <- phi - s (h^+ phi) h (the phase w cancels, s = 2/h^+h),
// so a numerator circuit needs only two inner products with h.  phi_0 = c-A_k x is a signed gather
// of x, which can be re-read instead of stored, so the circuit is three read-only sweeps over the
// tiles of x and h and no per-circuit scratch exists:
//   S1: d1 = h^+ phi_0
//   S2: phi_1 = Z_j (phi_0 - s d1 h),  d2 = h^+ phi_1
//   S3: <Z_anc> = Re(i^q sum_j conj(x'_j) (phi_1 - s d2 h)_j),  x' = c-A_l x (readout)
// Every circuit is still simulated on its own (the sweeps recompute its own phi_0, phi_1).
// Same launch signature as stream_hadamard_kernel (scratch unused); grid (G, K).
template <int TB>
__global__ void __launch_bounds__(TS<TB>::THREADS, 2)
stream_hh_kernel(const double2* __restrict__ x_all, const PauliTerm* __restrict__ tab,
                 const double2* __restrict__ coef, const double2* __restrict__ hv, double hv_scale, int L, int n,
                 int64_t c0, int64_t C, const int64_t* __restrict__ cidx, double2* __restrict__ scratch,
                 double* __restrict__ out_terms, double* __restrict__ partials, int with_cost,
                 double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {
  using T = TS<TB>;
  (void)scratch;
  __shared__ double red[T::THREADS / 32];
  __shared__ double bc[2];
  __shared__ double acc4[4];
  const int kth = blockIdx.y;
  const uint32_t N = 1u << n;
  const double2* __restrict__ x = x_all + (size_t)kth * N;
  const uint32_t t = threadIdx.x;
  const int64_t G = gridDim.x;
  const int64_t cb = (int64_t)blockIdx.x * C / G, ce = ((int64_t)blockIdx.x + 1) * C / G;
  const uint32_t ntiles = N >> TB;
  const Geo g0 = group(n, 0, TB);
  if (t == 0) acc4[0] = acc4[1] = acc4[2] = acc4[3] = 0.0;

  // (re, im) of s * h^+ v summed over the CTA, broadcast to every thread
  auto hdot = [&](double dr, double di, double& ar, double& ai) {
    dr = block_sum(dr, red, T::THREADS);
    di = block_sum(di, red, T::THREADS);
    if (t == 0) { bc[0] = dr * hv_scale; bc[1] = di * hv_scale; }
    __syncthreads();
    ar = bc[0];
    ai = bc[1];
    __syncthreads();  // bc / red reusable
  };

  for (int64_t cl = cb; cl < ce; ++cl) {
    const int64_t c = cidx ? cidx[cl] : c0 + cl;
    const int64_t tk = c >> 1;
    const int part = int(c & 1);
    const int sidx = int(tk % (n + 1));
    const int64_t lk = tk / (n + 1);
    const int k = int(lk % L), l = int(lk / L);
    const PauliTerm Tk = tab[k], Tl = tab[l];
    const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
    const bool im = q & 1;
    double acc = 0.0;
    if (sidx == 0) {
      acc = den_pass<TB>(x, g0, Tk, Tl, im, 0, ntiles, t);
    } else {
      const int p = n - 1 - (sidx - 1);  // Z_j bit position, j = s - 1
      // S1: d1 = h^+ phi_0
      double dr = 0.0, di = 0.0;
      for (uint32_t tau = 0; tau < ntiles; ++tau) {
        const Cols<LM_> cm(g0, t, tau);
        double2 v[16];
        gather(v, x, cm, Tk.xm, Tk.zm);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 h = __ldg(at(hv, cm.j(r)));
          dr = fma(h.x, v[r].x, fma(h.y, v[r].y, dr));
          di = fma(h.x, v[r].y, fma(-h.y, v[r].x, di));
        }
      }
      double ar, ai;
      hdot(dr, di, ar, ai);
      // S2: phi_1 = Z_j (phi_0 - a h), d2 = h^+ phi_1
      dr = 0.0;
      di = 0.0;
      for (uint32_t tau = 0; tau < ntiles; ++tau) {
        const Cols<LM_> cm(g0, t, tau);
        double2 v[16];
        gather(v, x, cm, Tk.xm, Tk.zm);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 h = __ldg(at(hv, cm.j(r)));
          v[r].x -= ar * h.x - ai * h.y;
          v[r].y -= ar * h.y + ai * h.x;
        }
        zsign(v, cm, p);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 h = __ldg(at(hv, cm.j(r)));
          dr = fma(h.x, v[r].x, fma(h.y, v[r].y, dr));
          di = fma(h.x, v[r].y, fma(-h.y, v[r].x, di));
        }
      }
      double br, bi;
      hdot(dr, di, br, bi);
      // S3: readout of phi_1 - b h
      for (uint32_t tau = 0; tau < ntiles; ++tau) {
        const Cols<LM_> cm(g0, t, tau);
        double2 v[16];
        gather(v, x, cm, Tk.xm, Tk.zm);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 h = __ldg(at(hv, cm.j(r)));
          v[r].x -= ar * h.x - ai * h.y;
          v[r].y -= ar * h.y + ai * h.x;
        }
        zsign(v, cm, p);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 h = __ldg(at(hv, cm.j(r)));
          v[r].x -= br * h.x - bi * h.y;
          v[r].y -= br * h.y + bi * h.x;
        }
        acc += readout(v, x, cm, Tl.xm, Tl.zm, im);
      }
    }
    double val = block_sum(acc, red, T::THREADS);
    if (t == 0) {
      val = (q == 1 || q == 2) ? -val : val;  // i^q phase: Re(i^q S)
      out_terms[(size_t)kth * C + cl] = val;
      const double2 cl_ = coef[l], ck = coef[k];
      const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
      const double cr = part == 0 ? wr * val : -wi * val;
      const double ci = part == 0 ? wi * val : wr * val;
      if (sidx == 0) { acc4[2] += cr; acc4[3] += ci; } else { acc4[0] += cr; acc4[1] += ci; }
    }
    __syncthreads();  // red reusable by the next circuit
  }
  if (t == 0) {
    double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
    o[0] = acc4[0]; o[1] = acc4[1]; o[2] = acc4[2]; o[3] = acc4[3];
  }
  if (red_out) finish_partials(partials, G, kth, n, with_cost, red_out, counter, p2p.world > 1 ? &p2p : nullptr);
}

}  // namespace stream
}  // namespace dvqls
