// stream_plane.cuh - the n >= 11, uniform-b Hadamard-test path on REAL planes.
//
// Same circuits, same passes and the same algorithmic work as stream_hadamard_kernel
// (stream.cuh, whose tile geometry, layouts, column walks and prefetch it reuses), with the
// branch split the way plane.cuh splits it at n = 10: for uniform b every gate after the first
// ancilla H is a real matrix (signed permutations c-A_k / c-A_l, c-H^{(x)n}, c-Z_j), so Re(phi)
// and Im(phi) evolve independently.  A CTA runs the whole pass sequence of one circuit twice,
// once per plane, and adds the two readout halves:
//     Re S = sum x'_re phi_re + sum x'_im phi_im,   Im S = sum x'_re phi_im - sum x'_im phi_re.
// A thread holds 16 doubles (32 registers instead of 64), so 4 CTAs fit on an SM instead of 2
// and their load / butterfly / exchange phases overlap; HBM bytes per circuit are unchanged
// (each plane's scratch is half the complex one).  x is read from a planar copy
// [x_re | x_im] (to_planar_kernel), so every x load uses whole sectors.
//
// SMEM: one tile of 2^TB doubles in rows padded to 17 (slot(e) = e + (e >> 4)): in every layout
// (LL, LM, LH) a half-warp's 16 doubles hit 16 distinct 8-byte bank pairs and the address is a
// per-lane base plus a compile-time immediate, issued as a shared-window access (no address
// arithmetic per element).
#pragma once

#include <type_traits>

#include "stream.cuh"

namespace dvqls {
namespace streamp {

using stream::Cols;
using stream::Geo;
using stream::LL_;
using stream::LM_;
using stream::TS;

// x_all (K thetas x 2^n complex, interleaved) -> xp (K x [re 2^n | im 2^n])
__global__ void __launch_bounds__(256) to_planar_kernel(const double2* __restrict__ x, uint32_t N, uint32_t K,
                                                        double* __restrict__ xp) {
  const size_t total = size_t(N) * K;
  for (size_t i = size_t(blockIdx.x) * 256 + threadIdx.x; i < total; i += size_t(gridDim.x) * 256) {
    const size_t k = i / N, j = i - k * N;
    const double2 a = x[i];
    xp[2 * k * N + j] = a.x;
    xp[(2 * k + 1) * N + j] = a.y;
  }
}

__device__ __forceinline__ uint32_t sbase() { return uint32_t(__cvta_generic_to_shared(dvqls_smem)); }
__device__ __forceinline__ double lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__host__ __device__ constexpr uint32_t pslot(uint32_t e) { return e + (e >> 4); }
template <int TB>
__host__ __device__ constexpr size_t tile_smem() {
  return (sizeof(double) * pslot(1u << TB) + 15) & ~size_t(15);
}
// exchange tile + TMA staging tile + mbarrier (STAGED kernels)
template <int TB>
__host__ __device__ constexpr size_t staged_smem() {
  return tile_smem<TB>() + sizeof(double) * (size_t(1) << TB) + 16;
}

// &base[idx] (8-byte elements) as one IMAD.WIDE.U32
__device__ __forceinline__ const double* atd(const double* base, uint32_t idx) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(r) : "r"(idx), "l"(base));
  return reinterpret_cast<const double*>(r);
}
__device__ __forceinline__ double* atd(double* base, uint32_t idx) {
  return const_cast<double*>(atd(const_cast<const double*>(base), idx));
}

// butterflies on register bit i for the tile bits of layout S in [lo, hi) (stream::stages, real)
template <int S, int TB>
__device__ __forceinline__ void stages(double (&v)[16], int lo, int hi) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = S + i;
    if (S == TS<TB>::SH && q < 8) continue;  // TB = 11: bit 7 belongs to LM
    if (q >= lo && q < hi) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (!(r & (1 << i))) {
          const double p = v[r], w = v[r | (1 << i)];
          v[r] = p + w;
          v[r | (1 << i)] = p - w;
        }
    }
  }
}

// layout SA -> SB through the padded tile buffer at shared-window address sm
template <int SA, int SB>
__device__ __forceinline__ void xchg(double (&v)[16], uint32_t sm, uint32_t t) {
  const uint32_t a = sm + pslot(stream::lelem<SA>(t, 0)) * 8u, b = sm + pslot(stream::lelem<SB>(t, 0)) * 8u;
  __syncthreads();  // previous readers of the buffer are done
#pragma unroll
  for (int r = 0; r < 16; ++r) sts(a + pslot(stream::lelem<SA>(0, uint32_t(r))) * 8u, v[r]);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = lds(b + pslot(stream::lelem<SB>(0, uint32_t(r))) * 8u);
}

// v_r = sgn_k(j_r ^ m) x_pl[j_r ^ m]   (c-A_k on one plane)
template <int S>
__device__ __forceinline__ void gather(double (&v)[16], const double* __restrict__ xpl, const Cols<S>& cc, uint32_t m,
                                       uint32_t z) {
  const uint32_t w = stream::sword(cc.parity_word(z), __popc((cc.jb ^ m) & z) & 1u);
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int r = k ^ (k >> 1);
    jj = cc.step(jj, k);
    v[r] = flip(__ldg(atd(xpl, jj ^ m)), stream::smask(w, r));
  }
}

// this plane's half of Re S (xr = own plane) or Im S (xr = other plane, negated for the Re plane
// through `neg`): sum_r sgn_l(j_r) xr[j_r ^ m] v_r
template <int S>
__device__ __forceinline__ double readout(const double (&v)[16], const double* __restrict__ xr, const Cols<S>& cc,
                                          uint32_t m, uint32_t z, uint32_t neg) {
  const uint32_t w = stream::sword(cc.parity_word(z), (__popc(cc.jb & z) & 1u) ^ neg);
  double a0 = 0.0, a1 = 0.0;
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int r = k ^ (k >> 1);
    jj = cc.step(jj, k);
    const double a = flip(__ldg(atd(xr, jj ^ m)), stream::smask(w, r));
    if (k & 1) a1 = fma(a, v[r], a1); else a0 = fma(a, v[r], a0);
  }
  return a0 + a1;
}

template <int S>
__device__ __forceinline__ void zsign(double (&v)[16], const Cols<S>& cc, int p) {
  const uint32_t w = stream::sword(cc.parity_word(1u << p), (cc.jb >> p) & 1u);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = flip(v[r], stream::smask(w, r));
}

template <int S>
__device__ __forceinline__ void gload(double (&v)[16], const double* __restrict__ src, const Cols<S>& cc) {
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    jj = cc.step(jj, k);
    v[k ^ (k >> 1)] = __ldcg(atd(src, jj));
  }
}

template <int S>
__device__ __forceinline__ void gstore(const double (&v)[16], double* __restrict__ dst, const Cols<S>& cc) {
  uint32_t jj = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    jj = cc.step(jj, k);
    __stcg(atd(dst, jj), v[k ^ (k >> 1)]);
  }
}

// ---- TMA bulk-copy staging of tiles (STAGED kernels) -----------------------------------------
// The tile of the NEXT iteration is copied global -> SMEM by cp.async.bulk (the TMA engine, SASS
// UBLKCP) into a staging buffer while the current tile is transformed in registers; completion is
// tracked by an mbarrier (expect_tx by thread 0, complete_tx by the copies).  The staging buffer
// holds the tile in natural element order, so the register layouts LM and LH read it conflict-free
// (a half-warp's 16 doubles are consecutive) with base + immediate addressing.
struct Stager {
  uint32_t buf;    // shared-window address of 2^TB staged doubles
  uint32_t mbar;   // shared-window address of the mbarrier
  uint32_t phase;  // parity of the next completion
};
__device__ __forceinline__ void mbar_init(uint32_t mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(mbar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// Copy tile tau of pass geometry g (2^tb doubles: one contiguous block when g.b == g.c, else
// 2^(tb-c) runs of 2^c doubles) into the staging buffer.  Called by all threads after a barrier
// that follows every read of the buffer; generic writes of the source (earlier passes) and reads of
// the buffer are ordered before the async-proxy copy by fence.proxy.async in each issuing thread.
template <int TB>
__device__ __forceinline__ void issue_tile(const Stager& st, const double* __restrict__ base, const Geo& g,
                                           uint32_t tau, uint32_t t) {
  constexpr uint32_t TN = 1u << TB, NT = TS<TB>::THREADS;
  if (g.b == g.c) {
    constexpr uint32_t CH = 512;  // doubles per request (4 KB)
    if (t < TN / CH) {
      asm volatile("fence.proxy.async;" ::: "memory");
      bulk_g2s(st.buf + t * CH * 8u, base + g.gidx(t * CH, tau), CH * 8u, st.mbar);
    }
  } else {
    const uint32_t runs = 1u << (g.tb - g.c);
    if (t < runs) asm volatile("fence.proxy.async;" ::: "memory");
    for (uint32_t u = t; u < runs; u += NT)
      bulk_g2s(st.buf + (u << g.c) * 8u, base + g.gidx(u << g.c, tau), 8u << g.c, st.mbar);
  }
  if (t == 0) mbar_expect(st.mbar, TN * 8u);
}

// wait for the staged tile, read it into registers in layout S, release the buffer
template <int S>
__device__ __forceinline__ void stage_load(double (&v)[16], Stager& st, uint32_t t) {
  mbar_wait(st.mbar, st.phase);
  st.phase ^= 1u;
  const uint32_t a = st.buf + stream::lelem<S>(t, 0) * 8u;
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = lds(a + stream::lelem<S>(0, uint32_t(r)) * 8u);
  __syncthreads();  // every thread has read the buffer: the next copy may overwrite it
}

// stream::prefetch_tile counts 16-byte amplitudes; a plane tile is half the bytes: prefetch the
// same index ranges of a double array (the base pointer is reinterpreted; sizes halve)
__device__ __forceinline__ void prefetch_tile_d(const double* __restrict__ base, const Geo& g, uint32_t tau,
                                                uint32_t flip_hi, uint32_t t, uint32_t nthreads) {
  if (g.b == g.c) {
    const uint32_t chunk = (1u << g.tb) / 16u;
    if (t < 16u) stream::prefetch_l2(base + ((g.gidx(t * chunk, tau)) ^ flip_hi), chunk * 8u);
  } else {
    const uint32_t runs = 1u << (g.tb - g.c);
    for (uint32_t u = t; u < runs; u += nthreads)
      stream::prefetch_l2(base + (g.gidx(u << g.c, tau) ^ flip_hi), 8u << g.c);
  }
}

// STAGED_ mid passes stage only when the tile's contiguous runs are >= 1 KB (c >= 7, n <= 17): TMA
// copies of 128-512 B runs (n = 18..20) measured no faster than direct register loads + L2 prefetch
template <int TB, int C, bool STAGED_>
__device__ __forceinline__ void mid_pass_c(double* __restrict__ phi, uint32_t sm, const Geo& g, int kind, int p,
                                           uint32_t t0, uint32_t t1, uint32_t t, Stager& st) {
  constexpr bool STAGED = STAGED_ && C >= 7;
  constexpr int lo = C, hi = TB, SH = TS<TB>::SH;
  constexpr bool needLM = lo < 8, needLL = lo < 4;
  if (STAGED && t0 < t1) issue_tile<TB>(st, phi, g, t0, t);
  for (uint32_t tau = t0; tau < t1; ++tau) {
    if (!STAGED && tau + 1 < t1) prefetch_tile_d(phi, g, tau + 1, 0u, t, TS<TB>::THREADS);
    double v[16];
    // STAGED: registers from the staged tile, then the next tile's copy overlaps this one's work
    auto fetch = [&](auto layout_tag, const auto& cols) {
      constexpr int S = decltype(layout_tag)::value;
      if constexpr (STAGED) {
        stage_load<S>(v, st, t);
        if (tau + 1 < t1) issue_tile<TB>(st, phi, g, tau + 1, t);
      } else {
        gload(v, phi, cols);
      }
    };
    if (!needLM) {
      const Cols<SH> cc(g, t, tau);
      fetch(std::integral_constant<int, SH>{}, cc);
      stages<SH, TB>(v, lo, hi);
      if (kind == 1) { zsign(v, cc, p); stages<SH, TB>(v, lo, hi); }
      gstore(v, phi, cc);
    } else if (kind == 2) {
      const Cols<SH> ch(g, t, tau);
      fetch(std::integral_constant<int, SH>{}, ch);
      stages<SH, TB>(v, lo, hi);
      if (needLL) {
        xchg<SH, LL_>(v, sm, t);
        stages<LL_, TB>(v, lo, hi);
        xchg<LL_, LM_>(v, sm, t);
      } else {
        xchg<SH, LM_>(v, sm, t);
      }
      stages<LM_, TB>(v, lo, hi);
      gstore(v, phi, Cols<LM_>(g, t, tau));
    } else {
      const Cols<LM_> cm(g, t, tau);
      fetch(std::integral_constant<int, LM_>{}, cm);
      stages<LM_, TB>(v, lo, hi);
      if (needLL) {
        xchg<LM_, LL_>(v, sm, t);
        stages<LL_, TB>(v, lo, hi);
        xchg<LL_, SH>(v, sm, t);
      } else {
        xchg<LM_, SH>(v, sm, t);
      }
      stages<SH, TB>(v, lo, hi);
      if (kind == 0) {
        gstore(v, phi, Cols<SH>(g, t, tau));
      } else {
        zsign(v, Cols<SH>(g, t, tau), p);
        stages<SH, TB>(v, lo, hi);
        if (needLL) {
          xchg<SH, LL_>(v, sm, t);
          stages<LL_, TB>(v, lo, hi);
          xchg<LL_, LM_>(v, sm, t);
        } else {
          xchg<SH, LM_>(v, sm, t);
        }
        stages<LM_, TB>(v, lo, hi);
        gstore(v, phi, cm);
      }
    }
  }
}

template <int TB, bool STAGED>
__device__ __forceinline__ void mid_pass(double* __restrict__ phi, uint32_t sm, const Geo& g, int kind, int p,
                                         uint32_t t0, uint32_t t1, uint32_t t, Stager& st) {
  switch (g.c) {
    case 2: mid_pass_c<TB, 2, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 3: mid_pass_c<TB, 3, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 4: mid_pass_c<TB, 4, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 5: mid_pass_c<TB, 5, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 6: mid_pass_c<TB, 6, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 7: mid_pass_c<TB, 7, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 8: mid_pass_c<TB, 8, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 9: mid_pass_c<TB, 9, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    case 10: mid_pass_c<TB, 10, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
    default: mid_pass_c<TB, 11, STAGED>(phi, sm, g, kind, p, t0, t1, t, st); break;
  }
}

// P0: gather (c-A_k) + F1 on tile bits, store the plane's scratch
template <int TB>
__device__ __forceinline__ void first_pass(double* __restrict__ phi, const double* __restrict__ xpl, uint32_t sm,
                                           const Geo& g0, const PauliTerm& Tk, bool big_x, uint32_t ntiles,
                                           uint32_t t) {
  constexpr int SH = TS<TB>::SH;
  for (uint32_t tau = 0; tau < ntiles; ++tau) {
    if (big_x && tau + 1 < ntiles)
      prefetch_tile_d(xpl, g0, tau + 1, Tk.xm & ~uint32_t(TS<TB>::TN - 1), t, TS<TB>::THREADS);
    double v[16];
    gather(v, xpl, Cols<LM_>(g0, t, tau), Tk.xm, Tk.zm);
    stages<LM_, TB>(v, 0, TB);
    xchg<LM_, LL_>(v, sm, t);
    stages<LL_, TB>(v, 0, TB);
    xchg<LL_, SH>(v, sm, t);
    stages<SH, TB>(v, 0, TB);
    gstore(v, phi, Cols<SH>(g0, t, tau));
  }
}

// last pass: F2 on tile bits + this plane's readout half
template <int TB, bool STAGED>
__device__ __forceinline__ double last_pass(const double* __restrict__ phi, const double* __restrict__ xr, uint32_t sm,
                                            const Geo& g0, const PauliTerm& Tl, uint32_t neg, bool big_x,
                                            uint32_t ntiles, uint32_t t, Stager& st) {
  constexpr int SH = TS<TB>::SH;
  double acc = 0.0;
  if (STAGED) issue_tile<TB>(st, phi, g0, 0, t);
  for (uint32_t tau = 0; tau < ntiles; ++tau) {
    if (tau + 1 < ntiles) {
      if (!STAGED) prefetch_tile_d(phi, g0, tau + 1, 0u, t, TS<TB>::THREADS);
      if (big_x) prefetch_tile_d(xr, g0, tau + 1, Tl.xm & ~uint32_t(TS<TB>::TN - 1), t, TS<TB>::THREADS);
    }
    double v[16];
    if constexpr (STAGED) {
      stage_load<SH>(v, st, t);
      if (tau + 1 < ntiles) issue_tile<TB>(st, phi, g0, tau + 1, t);
    } else {
      gload(v, phi, Cols<SH>(g0, t, tau));
    }
    stages<SH, TB>(v, 0, TB);
    xchg<SH, LL_>(v, sm, t);
    stages<LL_, TB>(v, 0, TB);
    xchg<LL_, LM_>(v, sm, t);
    stages<LM_, TB>(v, 0, TB);
    acc += readout(v, xr, Cols<LM_>(g0, t, tau), Tl.xm, Tl.zm, neg);
  }
  return acc;
}

// a3-a9 for n >= 11, uniform b: one circuit per CTA at a time, Re plane then Im plane.
// x_all: planar thetas [K][re 2^n | im 2^n];  scratch: 2^n doubles per CTA (n > TB).
// 3 CTAs per SM (80 registers; ptxas spills ~120-180 B): measured faster than 2 CTAs per SM with
// 112 registers and no spills (n = 18: 1237 vs 1299 ms, n = 20: 6144 vs 6300 ms per K = 2 step;
// profiles/r2_cfg5/minb_*.json)
constexpr int MIN_CTAS = 3;
template <int TB, bool STAGED = false>
__global__ void __launch_bounds__(TS<TB>::THREADS, MIN_CTAS)
stream_plane_kernel(const double* __restrict__ x_all, const PauliTerm* __restrict__ tab,
                    const double2* __restrict__ coef, int L, int n, int64_t c0, int64_t C,
                    const int64_t* __restrict__ cidx, double* __restrict__ scratch, double* __restrict__ out_terms,
                    double* __restrict__ partials, int with_cost, double* __restrict__ red_out,
                    unsigned* __restrict__ counter, P2PArgs p2p) {
  using T = TS<TB>;
  constexpr int SH = T::SH;
  __shared__ double red[T::THREADS / 32];
  __shared__ double acc4[4];
  const uint32_t sm = sbase();
  const int kth = blockIdx.y;
  const uint32_t N = 1u << n;
  const double* __restrict__ xre = x_all + (size_t)kth * 2 * N;
  double* __restrict__ phi = scratch + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * N;  // n > TB only
  const int ng = stream::ngroups(n, TB);
  const uint32_t t = threadIdx.x;
  const int64_t G = gridDim.x;
  const int64_t cb = (int64_t)blockIdx.x * C / G, ce = ((int64_t)blockIdx.x + 1) * C / G;
  const uint32_t ntiles = N > uint32_t(T::TN) ? N >> TB : 1u;
  const Geo g0 = stream::group(n, 0, TB);
  const bool big_x = n > 22;  // x tiles prefetched too (measured at n = 22: no gain, x of 2 thetas ~ L2)
  if (t == 0) acc4[0] = acc4[1] = acc4[2] = acc4[3] = 0.0;
  // STAGED: [exchange tile | staging tile | mbarrier] in dynamic SMEM
  Stager st{sm + uint32_t(tile_smem<TB>()), sm + uint32_t(tile_smem<TB>() + sizeof(double) * (size_t(1) << TB)), 0u};
  if (STAGED) {
    if (t == 0) {
      mbar_init(st.mbar);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }

  for (int64_t cl = cb; cl < ce; ++cl) {
    const int64_t c = cidx ? cidx[cl] : c0 + cl;
    const int64_t tk = c >> 1;
    const int part = int(c & 1);
    const int sidx = int(tk % (n + 1));
    const int64_t lk = tk / (n + 1);
    const int k = int(lk % L), l = int(lk / L);
    const PauliTerm Tk = tab[k], Tl = tab[l];
    const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
    const uint32_t im = uint32_t(q & 1);
    const int p = n - 1 - (sidx - 1);  // Z_j bit position (numerators)
    double acc = 0.0;
#pragma unroll 1
    for (uint32_t pl = 0; pl < 2; ++pl) {
      const double* __restrict__ xpl = xre + size_t(pl) * N;       // gather plane
      const double* __restrict__ xr = xre + size_t(pl ^ im) * N;   // readout plane
      const uint32_t neg = im & (pl ^ 1u);                         // Re plane of Im S: minus
      if (sidx == 0) {
        for (uint32_t tau = 0; tau < ntiles; ++tau) {
          const Cols<LM_> cm(g0, t, tau);
          double v[16];
          gather(v, xpl, cm, Tk.xm, Tk.zm);
          acc += readout(v, xr, cm, Tl.xm, Tl.zm, neg);
        }
      } else if (n <= TB) {
        const Cols<LM_> cm(g0, t, 0);
        double v[16];
        gather(v, xpl, cm, Tk.xm, Tk.zm);
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
        acc += readout(v, xr, cm, Tl.xm, Tl.zm, neg);
      } else {
        first_pass<TB>(phi, xpl, sm, g0, Tk, big_x, ntiles, t);
        __syncthreads();
        if (ng == 2) {
          mid_pass<TB, STAGED>(phi, sm, stream::group(n, 1, TB), 1, p, 0, ntiles, t, st);
        } else {
          mid_pass<TB, STAGED>(phi, sm, stream::group(n, 1, TB), 0, p, 0, ntiles, t, st);
          __syncthreads();
          mid_pass<TB, STAGED>(phi, sm, stream::group(n, 2, TB), 1, p, 0, ntiles, t, st);
          __syncthreads();
          mid_pass<TB, STAGED>(phi, sm, stream::group(n, 1, TB), 2, p, 0, ntiles, t, st);
        }
        __syncthreads();
        acc += last_pass<TB, STAGED>(phi, xr, sm, g0, Tl, neg, big_x, ntiles, t, st);
        __syncthreads();  // scratch reads done before the next plane's / circuit's P0
      }
    }
    double val = stream::block_sum(acc, red, T::THREADS);
    if (t == 0) {
      if (sidx > 0) val *= 1.0 / double(N);   // two unnormalised FWHTs
      val = (q == 1 || q == 2) ? -val : val;  // Re(i^q S)
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

}  // namespace streamp
}  // namespace dvqls
