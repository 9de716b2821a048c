// stream64.cuh - n >= 13, uniform-b Hadamard-test path with 64 doubles per thread and a
// transposed scratch layout (SURVEY §8(a) a3-a9 on the streaming path, north_star item (3)).
//
// Same circuits, passes, real-plane split and algorithmic HBM bytes as stream_plane_kernel
// (stream_plane.cuh): per numerator circuit and plane, P0 gathers x (c-A_k) and runs the FWHT over
// index bits 0..11 of each 4096-amplitude tile into a per-CTA scratch, P1 runs F1, c-Z_j, F2 over
// the bits >= 12, P2 runs F2 over bits 0..11 and the readout (c-A_l).  What changes is how a tile
// is laid out, because ncu put 38 % of the stall samples of the 16-doubles-per-thread kernel on
// its layout exchanges (two per 12-bit FWHT, barriers across 256 threads):
//   * a CTA is 64 threads holding 64 doubles each (6 register bits), so a tile is covered by two
//     layouts: B (registers = tile bits 6..11, threads = bits 0..5: coalesced in index order) and
//     A (registers = bits 0..5, threads = bits 6..11), and a 12-bit FWHT is butterflies in one
//     layout, ONE exchange, butterflies in the other;
//   * the scratch holds each tile with its two 6-bit halves swapped, sigma(i) = (i >> 12 << 12) |
//     ((i & 63) << 6) | ((i >> 6) & 63), so layout A -- P0's output and P2's input -- is coalesced
//     in scratch order;
//   * P1 works in sigma space with the tile geometry of stream_plane (passengers = the low c address
//     bits, active = index bits 12..): for n <= 18 every active bit is a register bit and P1 needs
//     no exchange at all; for n = 19..22 two layouts, two exchanges.
// Exchanges per numerator circuit-plane: 2 (n <= 18) or 4 (n = 19..22), against 6 before.  SMEM:
// one 4096-double tile buffer with rows padded to 65 doubles (33 KB; conflict-free LDS.64/STS.64,
// base + immediate addressing in every layout); 6 CTAs (12 warps) per SM.
#pragma once

#include "stream.cuh"

namespace dvqls {
namespace s64 {

constexpr int TB = 12;
constexpr uint32_t TN = 1u << TB;
constexpr int R = 64;          // doubles per thread (6 register bits)
constexpr int NT = 64;         // threads per CTA
// CTAs per SM the register budget is sized for: 4 (255 registers, ~2.6 KB static spills over all
// pass variants) or 6 (168 registers, spills in every pass); template parameter MINB
using stream::Geo;

__host__ __device__ constexpr uint32_t pslot(uint32_t e) { return e + (e >> 6); }
__host__ __device__ constexpr size_t smem_bytes() { return (sizeof(double) * pslot(TN) + 15) & ~size_t(15); }

__device__ __forceinline__ uint32_t sbase() { return uint32_t(__cvta_generic_to_shared(dvqls_smem)); }
__device__ __forceinline__ double lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ const double* atd(const double* base, uint32_t idx) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(r) : "r"(idx), "l"(base));
  return reinterpret_cast<const double*>(r);
}
__device__ __forceinline__ double* atd(double* base, uint32_t idx) {
  return const_cast<double*>(atd(const_cast<const double*>(base), idx));
}
__device__ __forceinline__ void bar() { asm volatile("bar.sync 0, 64;" ::: "memory"); }

// A layout of the 4096 tile elements over (thread t, register r): register bit b sits at tile
// position RP0 + b (six consecutive positions), the thread bits fill the other six positions in
// ascending order.  e(t, r) = ebits(t) | (r << RP0) is GF(2)-linear, and so is the address map.
template <int RP0>
__device__ __forceinline__ uint32_t tile_of_thread(uint32_t t) {  // thread bits -> tile positions
  const uint32_t lo = t & ((1u << RP0) - 1u), hi = t >> RP0;
  return lo | (hi << (RP0 + 6));
}

// Column walk of one layout over a pass geometry: register r <-> address jb ^ XOR_{b in r} o[b]
// (address = sigma space for the scratch, index space for x).  Gray-code order k -> r = k ^ k>>1.
struct Walk {
  uint32_t jb, o[6];
  __device__ __forceinline__ uint32_t step(uint32_t prev, int k) const {
    return k ? prev ^ o[ctz_c(k)] : opaque(jb, 0xffffffffu);
  }
};
template <int RP0>
__device__ __forceinline__ Walk walk(const Geo& g, uint32_t tau, uint32_t t) {
  Walk w;
  w.jb = g.gidx(tile_of_thread<RP0>(t), tau);
#pragma unroll
  for (int b = 0; b < 6; ++b) w.o[b] = 1u << g.gpos(RP0 + b);
  return w;
}

// butterflies on register bits [B0, B1)
template <int B0, int B1>
__device__ __forceinline__ void fwht(double (&v)[R]) {
#pragma unroll
  for (int bb = B0; bb < B1; ++bb) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (!(r & (1 << bb))) {
        const double p = v[r], q = v[r | (1 << bb)];
        v[r] = p + q;
        v[r | (1 << bb)] = p - q;
      }
  }
}

// layout RA -> layout RB through the padded tile buffer (tile positions: registers at RA.. / RB..)
template <int RA, int RB_>
__device__ __forceinline__ void xchg(double (&v)[R], uint32_t sm, uint32_t t) {
  const uint32_t a = sm + pslot(tile_of_thread<RA>(t)) * 8u, b = sm + pslot(tile_of_thread<RB_>(t)) * 8u;
  bar();  // previous readers of the buffer are done
#pragma unroll
  for (int r = 0; r < R; ++r) sts(a + pslot(uint32_t(r) << RA) * 8u, v[r]);
  bar();
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = lds(b + pslot(uint32_t(r) << RB_) * 8u);
}

__device__ __forceinline__ void gload(double (&v)[R], const double* __restrict__ src, const Walk& w) {
  uint32_t j = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    j = w.step(j, k);
    v[k ^ (k >> 1)] = __ldcg(atd(src, j));
  }
}
__device__ __forceinline__ void gstore(const double (&v)[R], double* __restrict__ dst, const Walk& w) {
  uint32_t j = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    j = w.step(j, k);
    __stcg(atd(dst, j), v[k ^ (k >> 1)]);
  }
}

// sign (-1)^{popcount(j & z)} of register r of a walk, as a 64-bit parity word (bit r)
__device__ __forceinline__ uint64_t parity64(const Walk& w, uint32_t z) {
  constexpr uint64_t cols[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                                0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
  uint64_t word = (__popc(w.jb & z) & 1u) ? ~0ull : 0ull;
#pragma unroll
  for (int b = 0; b < 6; ++b)
    if (w.o[b] & z) word ^= cols[b];
  return word;
}
__device__ __forceinline__ uint32_t smask64(uint64_t word, int r) { return uint32_t(word >> r) << 31; }

// v_r = sgn_k(j_r ^ m) x_pl[j_r ^ m] (c-A_k on one plane), walk in index space
__device__ __forceinline__ void gather(double (&v)[R], const double* __restrict__ xpl, const Walk& w, uint32_t m,
                                       uint32_t z) {
  Walk wm = w;
  wm.jb ^= m;
  const uint64_t s = parity64(wm, z);
  uint32_t j = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = k ^ (k >> 1);
    j = wm.step(j, k);
    v[r] = flip(__ldg(atd(xpl, j)), smask64(s, r));
  }
}

// this plane's readout half: sum_r sgn_l(j_r) xr[j_r ^ m] v_r (neg: the Re plane of Im S)
__device__ __forceinline__ double readout(const double (&v)[R], const double* __restrict__ xr, const Walk& w, uint32_t m,
                                          uint32_t z, uint32_t neg) {
  Walk wm = w;
  wm.jb ^= m;
  uint64_t s = parity64(w, z);  // sgn_l of j_r itself (P|j> = sgn(j) |j ^ m>)
  if (neg) s = ~s;
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  uint32_t j = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = k ^ (k >> 1);
    j = wm.step(j, k);
    a[k & 3] = fma(flip(__ldg(atd(xr, j)), smask64(s, r)), v[r], a[k & 3]);
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}

// c-Z_j: v_r = -v_r where bit p (of the walk's address space) of j_r is set
__device__ __forceinline__ void zsign(double (&v)[R], const Walk& w, int p) {
  const uint64_t s = parity64(w, 1u << p);
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = flip(v[r], smask64(s, r));
}

// scratch address of index i: the two 6-bit halves of the tile offset swapped
__device__ __forceinline__ int sigma_bit(int p) { return p >= TB ? p : (p < 6 ? p + 6 : p - 6); }

// P0 on tile tau: gather (layout B, index space), F1 on bits 6..11, exchange, F1 on bits 0..5,
// store in layout A = consecutive in sigma space
__device__ __forceinline__ void first_pass(double* __restrict__ phi, const double* __restrict__ xpl, uint32_t sm,
                                           const PauliTerm& Tk, bool big_x, uint32_t ntiles, uint32_t t) {
  const Geo g0{0, 0, TB};
  for (uint32_t tau = 0; tau < ntiles; ++tau) {
    if (big_x && tau + 1 < ntiles) {
      if (t < 16u) stream::prefetch_l2(xpl + (((tau + 1) << TB) ^ (Tk.xm & ~(TN - 1u))) + t * 256u, 2048u);
    }
    double v[R];
    gather(v, xpl, walk<6>(g0, tau, t), Tk.xm, Tk.zm);
    fwht<0, 6>(v);
    xchg<6, 0>(v, sm, t);
    fwht<0, 6>(v);
    gstore(v, phi, walk<6>(g0, tau, t));  // layout A (registers = index bits 0..5) -> sigma (r << 6) | t
  }
}

// P2 on tile tau: load layout A from sigma space, F2 on bits 0..5, exchange, F2 on bits 6..11,
// readout in layout B (index space)
__device__ __forceinline__ double last_pass(const double* __restrict__ phi, const double* __restrict__ xr, uint32_t sm,
                                            const PauliTerm& Tl, uint32_t neg, bool big_x, uint32_t ntiles,
                                            uint32_t t) {
  const Geo g0{0, 0, TB};
  double acc = 0.0;
  for (uint32_t tau = 0; tau < ntiles; ++tau) {
    if (tau + 1 < ntiles && t < 16u) {
      stream::prefetch_l2(phi + ((tau + 1) << TB) + t * 256u, 2048u);
      if (big_x) stream::prefetch_l2(xr + (((tau + 1) << TB) ^ (Tl.xm & ~(TN - 1u))) + t * 256u, 2048u);
    }
    double v[R];
    gload(v, phi, walk<6>(g0, tau, t));
    fwht<0, 6>(v);
    xchg<0, 6>(v, sm, t);
    fwht<0, 6>(v);
    acc += readout(v, xr, walk<6>(g0, tau, t), Tl.xm, Tl.zm, neg);
  }
  return acc;
}

// P1 in sigma space over group g (passengers c = g.c address bits, active = tile positions
// [c, 12) at address bits g.b..): kind 0 = F1, 1 = F1 Z_j F2, 2 = F2 (p = Z_j's sigma bit)
template <int C>
__device__ __forceinline__ void mid_pass_c(double* __restrict__ phi, uint32_t sm, const Geo& g, int kind, int p,
                                           uint32_t ntiles, uint32_t t) {
  for (uint32_t tau = 0; tau < ntiles; ++tau) {
    if (tau + 1 < ntiles) {  // L2 prefetch of the next tile's runs
      const uint32_t runs = 1u << (TB - C);
      for (uint32_t u = t; u < runs; u += NT) stream::prefetch_l2(phi + g.gidx(u << C, tau + 1), 8u << C);
    }
    double v[R];
    if constexpr (C >= 6) {
      // registers = tile positions 6..11 (C - 6 passengers, then the active bits), threads = 0..5
      const Walk w = walk<6>(g, tau, t);
      gload(v, phi, w);
      if (kind != 2) fwht<C - 6, 6>(v);
      if (kind == 1) {
        zsign(v, w, p);
        fwht<C - 6, 6>(v);
      }
      if (kind == 2) fwht<C - 6, 6>(v);
      gstore(v, phi, w);
    } else {
      // M1: registers = positions 6..11 (active), threads = 0..5 (C passengers + active);
      // M2: registers = positions C..C+5 (active), threads = 0..C-1 and C+6..11
      if (kind == 2) {
        const Walk w2 = walk<C>(g, tau, t);
        gload(v, phi, w2);
        fwht<0, 6>(v);
        xchg<C, 6>(v, sm, t);
        fwht<C, 6>(v);  // positions C + 6 .. 11 are register bits C .. 5 of M1
        gstore(v, phi, walk<6>(g, tau, t));
      } else {
        const Walk w1 = walk<6>(g, tau, t);
        gload(v, phi, w1);
        fwht<0, 6>(v);
        xchg<6, C>(v, sm, t);
        fwht<0, 6 - C>(v);  // positions C .. 5 are register bits 0 .. 5 - C of M2
        if (kind == 0) {
          gstore(v, phi, walk<C>(g, tau, t));
        } else {
          zsign(v, walk<C>(g, tau, t), p);
          fwht<0, 6>(v);
          xchg<C, 6>(v, sm, t);
          fwht<C, 6>(v);
          gstore(v, phi, w1);
        }
      }
    }
  }
}

__device__ __forceinline__ void mid_pass(double* __restrict__ phi, uint32_t sm, const Geo& g, int kind, int p,
                                         uint32_t ntiles, uint32_t t) {
  switch (g.c) {
    case 2: mid_pass_c<2>(phi, sm, g, kind, p, ntiles, t); break;
    case 3: mid_pass_c<3>(phi, sm, g, kind, p, ntiles, t); break;
    case 4: mid_pass_c<4>(phi, sm, g, kind, p, ntiles, t); break;
    case 5: mid_pass_c<5>(phi, sm, g, kind, p, ntiles, t); break;
    case 6: mid_pass_c<6>(phi, sm, g, kind, p, ntiles, t); break;
    case 7: mid_pass_c<7>(phi, sm, g, kind, p, ntiles, t); break;
    case 8: mid_pass_c<8>(phi, sm, g, kind, p, ntiles, t); break;
    case 9: mid_pass_c<9>(phi, sm, g, kind, p, ntiles, t); break;
    case 10: mid_pass_c<10>(phi, sm, g, kind, p, ntiles, t); break;
    default: mid_pass_c<11>(phi, sm, g, kind, p, ntiles, t); break;
  }
}

// a3-a9 for n >= 13, uniform b: one circuit per CTA at a time, Re plane then Im plane.
// x_all: planar thetas [K][re 2^n | im 2^n];  scratch: 2^n doubles per CTA.  Grid (G, K).
template <int MINB>
__global__ void __launch_bounds__(NT, MINB)
stream64_kernel(const double* __restrict__ x_all, const PauliTerm* __restrict__ tab, const double2* __restrict__ coef,
                int L, int n, int64_t c0, int64_t C, const int64_t* __restrict__ cidx, double* __restrict__ scratch,
                double* __restrict__ out_terms, double* __restrict__ partials, int with_cost,
                double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {
  __shared__ double red[NT / 32];
  __shared__ double acc4[4];
  const uint32_t sm = sbase();
  const int kth = blockIdx.y;
  const uint32_t N = 1u << n;
  const double* __restrict__ xre = x_all + (size_t)kth * 2 * N;
  double* __restrict__ phi = scratch + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * N;
  const int ng = stream::ngroups(n, TB);
  const uint32_t t = threadIdx.x;
  const int64_t G = gridDim.x;
  const int64_t cb = (int64_t)blockIdx.x * C / G, ce = ((int64_t)blockIdx.x + 1) * C / G;
  const uint32_t ntiles = N >> TB;
  const Geo g0{0, 0, TB};
  const bool big_x = n > 22;
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
    const uint32_t im = uint32_t(q & 1);
    const int p = sigma_bit(n - 1 - (sidx - 1));  // Z_j's bit in sigma space (numerators)
    double acc = 0.0;
#pragma unroll 1
    for (uint32_t pl = 0; pl < 2; ++pl) {
      const double* __restrict__ xpl = xre + size_t(pl) * N;       // gather plane
      const double* __restrict__ xr = xre + size_t(pl ^ im) * N;   // readout plane
      const uint32_t neg = im & (pl ^ 1u);                         // Re plane of Im S: minus
      if (sidx == 0) {
        for (uint32_t tau = 0; tau < ntiles; ++tau) {
          const Walk w = walk<6>(g0, tau, t);
          double v[R];
          gather(v, xpl, w, Tk.xm, Tk.zm);
          acc += readout(v, xr, w, Tl.xm, Tl.zm, neg);
        }
      } else {
        first_pass(phi, xpl, sm, Tk, big_x, ntiles, t);
        bar();
        if (ng == 2) {
          mid_pass(phi, sm, stream::group(n, 1, TB), 1, p, ntiles, t);
        } else {
          mid_pass(phi, sm, stream::group(n, 1, TB), 0, p, ntiles, t);
          bar();
          mid_pass(phi, sm, stream::group(n, 2, TB), 1, p, ntiles, t);
          bar();
          mid_pass(phi, sm, stream::group(n, 1, TB), 2, p, ntiles, t);
        }
        bar();
        acc += last_pass(phi, xr, sm, Tl, neg, big_x, ntiles, t);
        bar();  // scratch reads done before the next plane's / circuit's P0
      }
    }
    double val = stream::block_sum(acc, red, NT);
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

}  // namespace s64
}  // namespace dvqls
