// tile.cuh - the n >= 11 path: Hadamard-test circuits whose 2^n-amplitude branch no
// longer fits one warp's registers (north_star item (3)).
//
// The branch is processed in tiles of TN = 4096 amplitudes (64 KB of SMEM).  A tile
// pass maps tile bits to global index bits:
//     tile bits [0, c)   = global bits [0, c)         ("passengers": coalescing only)
//     tile bits [c, tb)  = global bits [b, b + tb - c) (the active bits of the pass)
// Inside a tile the FWHT stages run in rounds of 4 tile bits: every thread loads
// 16 amplitudes (the round's 4 bits) from SMEM into registers, applies the stages,
// stores them back.  Bit groups (SURVEY §8(d) "streaming model"):
//     g0 = [0, min(n,12)),  g1 = [12, 12 + min(n-12, 9)),  g2 = [21, n)
// n <= 12: one group, the whole circuit is one tile pass and never leaves SMEM.
// n >  12: the branch lives in a per-CTA global scratch; per numerator circuit the
// passes are gather+FWHT1(g0) | FWHT1(g1) ... | FWHT1(gm) Z_j FWHT2(gm) | ... |
// FWHT2(g0)+readout: 3 passes for n <= 21 (96 N bytes of HBM per circuit) and 5
// for n <= 24.  Every circuit is still simulated on its own (no sharing).
#pragma once

#include "kernels.cuh"

namespace dvqls {
namespace tile {

constexpr int TBITS = 12;
constexpr int TN = 1 << TBITS;
constexpr int THREADS = 256;
constexpr int RB = 4;          // register bits per round
constexpr int RR = 1 << RB;    // amplitudes per thread per round

struct Geo {
  int c, b, tb;  // passengers, first active global bit, tile bits
  __device__ __forceinline__ int a() const { return tb - c; }
  // global index of tile element e in tile number `tile`
  __device__ __forceinline__ uint32_t gidx(uint32_t tile, uint32_t e) const {
    const uint32_t lowp = e & ((1u << c) - 1u);
    const uint32_t act = e >> c;
    const uint32_t mid = tile & ((1u << (b - c)) - 1u);  // global bits [c, b)
    const uint32_t hi = tile >> (b - c);                  // global bits [b + a, n)
    return lowp | (mid << c) | (act << b) | (hi << (b + a()));
  }
};

__device__ __forceinline__ int ngroups(int n) { return n <= 12 ? 1 : (n <= 21 ? 2 : 3); }

__device__ __forceinline__ Geo group(int n, int gi) {
  Geo g;
  if (gi == 0) {
    g.c = 0; g.b = 0; g.tb = n < TBITS ? n : TBITS;
  } else if (gi == 1) {
    const int a = (n - 12) < 9 ? (n - 12) : 9;
    g.tb = TBITS; g.c = TBITS - a; g.b = 12;
  } else {
    const int a = n - 21;
    g.tb = TBITS; g.c = TBITS - a; g.b = 21;
  }
  return g;
}

// SMEM slot of tile element e: low 3 bits XOR bits 4..6 -> every round is conflict-free
__device__ __forceinline__ int tslot(int e) { return e ^ ((e >> 4) & 7); }

// element handled by (thread t, register r) in the round covering tile bits [4 rho, 4 rho + 4)
__device__ __forceinline__ int relem(int t, int r, int rho) {
  const int s = RB * rho;
  return ((t >> s) << (s + RB)) | (r << s) | (t & ((1 << s) - 1));
}

// One SMEM round: FWHT stages on the tile bits in [4 rho, 4 rho + 4) that lie in [lo, hi).
__device__ __forceinline__ void round_fwht(double2* s, int rho, int lo, int hi, int tb) {
  // Always the full 12-bit SMEM tile: for tb < 12 the elements >= 2^tb are inert (no
  // stage on a bit >= tb touches them and they are never read back).
  (void)tb;
  const int t = threadIdx.x;
  double2 v[RR];
#pragma unroll
  for (int r = 0; r < RR; ++r) v[r] = s[tslot(relem(t, r, rho))];
#pragma unroll
  for (int bb = 0; bb < RB; ++bb) {
    const int q = RB * rho + bb;
    if (q >= lo && q < hi) {
#pragma unroll
      for (int r = 0; r < RR; ++r)
        if (!(r & (1 << bb))) {
          const double2 p = v[r], w = v[r | (1 << bb)];
          v[r] = make_double2(p.x + w.x, p.y + w.y);
          v[r | (1 << bb)] = make_double2(p.x - w.x, p.y - w.y);
        }
    }
  }
#pragma unroll
  for (int r = 0; r < RR; ++r) s[tslot(relem(t, r, rho))] = v[r];
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < THREADS / 32; ++w) tot += red[w];  // fixed order
  return tot;  // valid in thread 0
}

// gather with sign: sgn_k(j ^ m_k) x[j ^ m_k] = (-1)^{popcount((j ^ m) & z)} x[j ^ m]
__device__ __forceinline__ double2 sgather(const double2* __restrict__ x, uint32_t j, uint32_t m, uint32_t z) {
  const uint32_t jj = j ^ m;
  const double2 a = __ldg(x + jj);
  return (__popc(jj & z) & 1) ? make_double2(-a.x, -a.y) : a;
}

template <bool HH>
__global__ void __launch_bounds__(THREADS, 2)
tile_hadamard_kernel(const double2* __restrict__ x_all, const PauliTerm* __restrict__ tab,
                     const double2* __restrict__ coef, const double2* __restrict__ hv, double hv_scale, int L,
                     int n, int64_t c0, int64_t C, const int64_t* __restrict__ cidx, double2* __restrict__ scratch,
                     double* __restrict__ out_terms, double* __restrict__ partials, int with_cost,
                     double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {  // TN amplitudes (dynamic: > 48 KB)
  double2* s = dvqls_smem;
  __shared__ double red[THREADS / 32];
  __shared__ double acc4[4];
  const int kth = blockIdx.y;
  const uint32_t N = 1u << n;
  const double2* __restrict__ x = x_all + (size_t)kth * N;
  double2* __restrict__ phi = scratch + (size_t)blockIdx.x * N;  // n > 12 only
  const int ng = ngroups(n);
  const int t = threadIdx.x;
  const int64_t G = gridDim.x;
  const int64_t cb = (int64_t)blockIdx.x * C / G, ce = ((int64_t)blockIdx.x + 1) * C / G;
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
    double acc = 0.0;
    if (sidx == 0) {
      // ---- denominator: sum_j conj(sgn_l(j) x_{j^m_l}) sgn_k(j^m_k) x_{j^m_k}, straight from x
      for (uint32_t j = t; j < N; j += THREADS) {
        const double2 ph = sgather(x, j, Tk.xm, Tk.zm);
        double2 xl = __ldg(x + (j ^ Tl.xm));
        if (__popc(j & Tl.zm) & 1) xl = make_double2(-xl.x, -xl.y);
        acc += (q & 1) ? (xl.x * ph.y - xl.y * ph.x) : (xl.x * ph.x + xl.y * ph.y);
      }
    } else {
      const int p = n - 1 - (sidx - 1);  // Z_j bit position
      const int npass = 2 * ng - 1;
      for (int pass = 0; pass < npass; ++pass) {
        // group of this pass and whether it is in FWHT1, the middle, or FWHT2
        const int gi = pass < ng ? pass : 2 * ng - 2 - pass;
        const Geo geo = group(n, gi);
        const bool first = pass == 0, last = pass == npass - 1;
        const bool do1 = pass <= ng - 1;   // FWHT1 stages on this group
        const bool do2 = pass >= ng - 1;   // FWHT2 stages on this group
        const bool zhere = pass == ng - 1; // Z_j between the two transforms
        const uint32_t ntiles = N >> geo.tb;
        for (uint32_t tile = 0; tile < ntiles; ++tile) {
          // ---- load: cp.async global -> SMEM, all copies of the tile in flight at once ----
          // (pass 0 copies the UNSIGNED x[j ^ m_k]; the Pauli sign of c-A_k is applied in
          //  the first SMEM round below)
          for (int e = t; e < (1 << geo.tb); e += THREADS) {
            const uint32_t j = geo.gidx(tile, e);
            const double2* src = first ? (x + (j ^ Tk.xm)) : (phi + j);
            const uint32_t dst = uint32_t(__cvta_generic_to_shared(s + tslot(e)));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          }
          asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
          __syncthreads();
          if (first && !HH) {  // sgn_k(j ^ m_k) = (-1)^{popcount((j ^ m_k) & z_k)}
            for (int e = t; e < (1 << geo.tb); e += THREADS)
              if (__popc((geo.gidx(tile, e) ^ Tk.xm) & Tk.zm) & 1) {
                const double2 f = s[tslot(e)];
                s[tslot(e)] = make_double2(-f.x, -f.y);
              }
            __syncthreads();
          }
          if (first && HH) {
            for (int e = t; e < (1 << geo.tb); e += THREADS)
              if (__popc((geo.gidx(tile, e) ^ Tk.xm) & Tk.zm) & 1) {
                const double2 f = s[tslot(e)];
                s[tslot(e)] = make_double2(-f.x, -f.y);
              }
            __syncthreads();
          }
          // ---- FWHT rounds on tile bits [c, tb) ----
          const int nr = TBITS / RB;
          if (HH) {
            // Householder U_b (n <= 12, single group): phi <- H_v Z_j H_v phi
            // dot = v^+ phi over the tile
            double dr = 0.0, di = 0.0;
            for (int e = t; e < (1 << geo.tb); e += THREADS) {
              const double2 h = __ldg(hv + e), f = s[tslot(e)];
              dr += h.x * f.x + h.y * f.y;
              di += h.x * f.y - h.y * f.x;
            }
            const double Dr = block_sum(dr, red), Di = block_sum(di, red);
            __shared__ double dd[2];
            if (t == 0) { dd[0] = Dr * hv_scale; dd[1] = Di * hv_scale; }
            __syncthreads();
            for (int e = t; e < (1 << geo.tb); e += THREADS) {
              const double2 h = __ldg(hv + e);
              double2 f = s[tslot(e)];
              f.x -= dd[0] * h.x - dd[1] * h.y;
              f.y -= dd[0] * h.y + dd[1] * h.x;
              if ((e >> p) & 1) f = make_double2(-f.x, -f.y);  // Z_j
              s[tslot(e)] = f;
            }
            __syncthreads();
            dr = di = 0.0;
            for (int e = t; e < (1 << geo.tb); e += THREADS) {
              const double2 h = __ldg(hv + e), f = s[tslot(e)];
              dr += h.x * f.x + h.y * f.y;
              di += h.x * f.y - h.y * f.x;
            }
            const double Er = block_sum(dr, red), Ei = block_sum(di, red);
            if (t == 0) { dd[0] = Er * hv_scale; dd[1] = Ei * hv_scale; }
            __syncthreads();
            for (int e = t; e < (1 << geo.tb); e += THREADS) {
              const double2 h = __ldg(hv + e);
              double2 f = s[tslot(e)];
              f.x -= dd[0] * h.x - dd[1] * h.y;
              f.y -= dd[0] * h.y + dd[1] * h.x;
              s[tslot(e)] = f;
            }
            __syncthreads();
          } else {
            if (do1) {
              for (int rho = 0; rho < nr; ++rho) {
                round_fwht(s, rho, geo.c, geo.tb, geo.tb);
                __syncthreads();
              }
            }
            if (zhere) {  // c-Z_j: FWHT1 is complete on every bit here; sign by the global index
              for (int e = t; e < (1 << geo.tb); e += THREADS)
                if ((geo.gidx(tile, e) >> p) & 1u) {
                  const double2 f = s[tslot(e)];
                  s[tslot(e)] = make_double2(-f.x, -f.y);
                }
              __syncthreads();
            }
            if (do2) {
              for (int rho = 0; rho < nr; ++rho) {
                round_fwht(s, rho, geo.c, geo.tb, geo.tb);
                __syncthreads();
              }
            }
          }
          // ---- store or read out ----
          if (last) {
            for (int e = t; e < (1 << geo.tb); e += THREADS) {
              const uint32_t j = geo.gidx(tile, e);
              const double2 f = s[tslot(e)];
              double2 xl = __ldg(x + (j ^ Tl.xm));
              if (__popc(j & Tl.zm) & 1) xl = make_double2(-xl.x, -xl.y);
              acc += (q & 1) ? (xl.x * f.y - xl.y * f.x) : (xl.x * f.x + xl.y * f.y);
            }
          } else {
            for (int e = t; e < (1 << geo.tb); e += THREADS) __stcs(phi + geo.gidx(tile, e), s[tslot(e)]);
          }
          __syncthreads();
        }
        if (!last) __threadfence_block();
      }
    }
    double val = block_sum(acc, red);
    if (t == 0) {
      if (sidx > 0 && !HH) val *= 1.0 / double(N);
      val = (q == 1 || q == 2) ? -val : val;
      out_terms[(size_t)kth * C + cl] = val;
      const double2 cl_ = coef[l], ck = coef[k];
      const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
      const double cr = part == 0 ? wr * val : -wi * val;
      const double ci = part == 0 ? wi * val : wr * val;
      if (sidx == 0) { acc4[2] += cr; acc4[3] += ci; } else { acc4[0] += cr; acc4[1] += ci; }
    }
    __syncthreads();
  }
  if (t == 0) {
    double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
    o[0] = acc4[0]; o[1] = acc4[1]; o[2] = acc4[2]; o[3] = acc4[3];
  }
  if (red_out) finish_partials(partials, G, kth, n, with_cost, red_out, counter, p2p.world > 1 ? &p2p : nullptr);
}

// ---------------------------------------------------------------------------
// Prefix for n >= 13 (state in global memory), one kernel per pass:
//   prefix_gates_kernel: SU(2) parameters (a, b) of every fused gate Ry Rz Ry
//   prefix_gate_pass:    one tile per CTA, the layer's gates on the group's bits
//   prefix_ring_kernel:  CNOT ring as a gather into the other buffer / CZ ring sign
// ---------------------------------------------------------------------------
__global__ void prefix_gates_kernel(const double* __restrict__ theta, int G, double2* __restrict__ gates) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  double s0, c0, s1, c1, s2, c2;
  sincos(0.5 * theta[3 * g + 0], &s0, &c0);
  sincos(0.5 * theta[3 * g + 1], &s1, &c1);
  sincos(0.5 * theta[3 * g + 2], &s2, &c2);
  gates[2 * g + 0] = make_double2(c1 * (c2 * c0 - s2 * s0), -s1 * (c2 * c0 + s2 * s0));
  gates[2 * g + 1] = make_double2(c1 * (s2 * c0 + c2 * s0), s1 * (c2 * s0 - s2 * c0));
}

__global__ void prefix_init_kernel(double2* __restrict__ x, uint32_t N) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
    x[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
}

__global__ void __launch_bounds__(THREADS)
prefix_gate_pass(double2* __restrict__ x, const double2* __restrict__ gates, int n, int gi, int layer) {
  double2* s = dvqls_smem;
  const Geo geo = group(n, gi);
  const uint32_t tile = blockIdx.x;
  const int t = threadIdx.x;
  for (int e = t; e < (1 << geo.tb); e += THREADS) s[tslot(e)] = x[geo.gidx(tile, e)];
  __syncthreads();
  for (int rho = 0; rho < TBITS / RB; ++rho) {
    double2 v[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) v[r] = s[tslot(relem(t, r, rho))];
#pragma unroll
    for (int bb = 0; bb < RB; ++bb) {
      const int q = RB * rho + bb;
      if (q >= geo.c && q < geo.tb) {
        const int pos = geo.b + (q - geo.c);
        const int g = layer * n + (n - 1 - pos);
        const double2 ua = gates[2 * g], ub = gates[2 * g + 1];
#pragma unroll
        for (int r = 0; r < RR; ++r)
          if (!(r & (1 << bb))) {
            const double2 x0 = v[r], x1 = v[r | (1 << bb)];
            v[r] = make_double2(fma(ua.x, x0.x, fma(-ua.y, x0.y, fma(-ub.x, x1.x, -ub.y * x1.y))),
                                fma(ua.x, x0.y, fma(ua.y, x0.x, fma(-ub.x, x1.y, ub.y * x1.x))));
            v[r | (1 << bb)] = make_double2(fma(ub.x, x0.x, fma(-ub.y, x0.y, fma(ua.x, x1.x, ua.y * x1.y))),
                                            fma(ub.x, x0.y, fma(ub.y, x0.x, fma(ua.x, x1.y, -ua.y * x1.x))));
          }
      }
    }
#pragma unroll
    for (int r = 0; r < RR; ++r) s[tslot(relem(t, r, rho))] = v[r];
    __syncthreads();
  }
  for (int e = t; e < (1 << geo.tb); e += THREADS) x[geo.gidx(tile, e)] = s[tslot(e)];
}

__global__ void prefix_ring_kernel(const double2* __restrict__ src, double2* __restrict__ dst, int n, int entangler) {
  const uint32_t N = 1u << n;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (entangler == 0) {
      uint32_t j = i;  // new[i] = old[c_0(c_1(...c_{n-1}(i)))]
      for (int q = n - 1; q >= 0; --q) {
        const int pc = n - 1 - q, pt = n - 1 - ((q + 1) % n);
        if ((j >> pc) & 1u) j ^= 1u << pt;
      }
      dst[i] = src[j];
    } else {
      int par = 0;
      for (int q = 0; q < n; ++q) par ^= int((i >> (n - 1 - q)) & (i >> (n - 1 - (q + 1) % n))) & 1;
      const double2 a = src[i];
      dst[i] = par ? make_double2(-a.x, -a.y) : a;
    }
  }
}

}  // namespace tile
}  // namespace dvqls
