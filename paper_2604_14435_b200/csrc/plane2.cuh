// plane2.cuh - n = 10, uniform-b Hadamard-test kernel, real-plane split (plane.cuh) with TWO
// circuits in flight per warp, software-pipelined.
//
// SURVEY §8(a) a3-a9 for the headline workload, same circuits, gate sequence, data layout and
// algorithmic work as plane_kernel (plane.cuh; every circuit simulated on its own).  What changes
// is the instruction stream of a warp.  A numerator circuit alternates SMEM-only phases (gather,
// two layout exchanges, readout) with FP64-only phases (four 5-stage FWHT blocks), and both
// resources are needed at ~85 % of their peaks (0.190 vs 0.224 ms per cfg3
// evaluation), so one circuit per warp leaves them overlapping only as well as the warp
// scheduler happens to mix warps in different phases.  Here a warp owns two consecutive circuits
// A, B of the same kind and skews them by one phase, so every code segment pairs one circuit's
// SMEM phase with the other's FP64 phase:
//     seg 1: F1(A)           | gather(B)
//     seg 2: X1(A)           | F1(B)
//     seg 3: F2 Z F3 (A)     | X1(B)
//     seg 4: X2(A)           | F2 Z F3 (B)
//     seg 5: F4(A)           | X2(B)
//     seg 6: readout(A)      | F4(B)
//     seg 7: readout(B)
// (F = five register butterfly stages, X = exchange through the warp's padded buffer, Z = c-Z_j,
// applied inside F3's or F4's stage on bit j as the sign of that stage's butterflies: fwht_z).
// Two 32-double planes per thread (168 registers): 12 warps (6 pairs, 12 circuits in flight per
// SM), one exchange buffer per warp (the segments use it in turn, guarded by __syncwarp).
#pragma once

#include "plane.cuh"

namespace dvqls {
namespace plane2 {

using plane::BATCH;
using plane::BUF;
using plane::lds_a;
using plane::N;
using plane::NQ;
using plane::R;
using plane::RB;
using plane::ROW;
using plane::sts_a;
using plane::TB;
using plane::XALIGN;
using plane::XREG;

constexpr int WARPS = 12;
constexpr int NP = WARPS / 2;

// %globaltimer stamps per CTA for tools/plane2_timing.cu (built with -DDVQLS_PLANE2_TS only):
// [0] entry, [1] after pdl_wait, [2] x staged, [3] all tasks of the last piece done, [4] piece
// reduction written, [5] kernel end of the CTA, [6 + pair] the pair's last task done
#ifdef DVQLS_PLANE2_TS
__device__ unsigned long long g_p2ts[160 * 16];
__device__ __forceinline__ void p2ts(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_p2ts[blockIdx.x * 16 + k] = t;
}
#define P2TS(k) p2ts(k)
#else
#define P2TS(k) do { } while (0)
#endif

template <int B0, int B1>
__device__ __forceinline__ void fwht(double (&v)[R]) { plane::fwht<B0, B1>(v); }

// a6 folded into the FWHT: c-Z_j negates every amplitude whose index bit p is set, and the
// butterflies on the other bits commute with that diagonal sign, so it is applied inside the
// stage on bit p as (a, b) -> (a - b, a + b) -- fma(+-1, b, a), bitwise the result of negating b
// first (no separate pass of 64 integer sign flips per plane).  ZB = that stage's register bit in
// [B0, B1), or -1 (none here).
template <int B0, int B1>
__device__ __forceinline__ void fwht_z(double (&v)[R], int zb) {
#pragma unroll
  for (int bb = B0; bb < B1; ++bb) {
    const double sg = bb == zb ? -1.0 : 1.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!(r & (1 << bb))) {
        const double a = v[r], b = v[r | (1 << bb)];
        v[r] = fma(sg, b, a);
        v[r | (1 << bb)] = fma(-sg, b, a);
      }
    }
  }
}

// a4: phi_i = sgn_k(i ^ m_k) x_pl[i ^ m_k] in layout A (sign and plane are address bits)
__device__ __forceinline__ void gather(double (&v)[R], uint32_t xa, uint32_t pl, uint32_t t, const PauliTerm& Tk) {
  const uint32_t mh = Tk.xm >> TB, tl = t ^ (Tk.xm & 31u), zh = Tk.zm >> TB;
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

__device__ __forceinline__ void store_A(const double (&v)[R], uint32_t baseA) {
#pragma unroll
  for (int r = 0; r < R; ++r) sts_a(baseA + uint32_t(r) * ROW, v[r]);
}
__device__ __forceinline__ void store_B(const double (&v)[R], uint32_t baseB) {
#pragma unroll
  for (int r = 0; r < R; ++r) sts_a(baseB + uint32_t(r) * 8u, v[r]);
}
__device__ __forceinline__ void load_A(double (&v)[R], uint32_t baseA) {
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = lds_a(baseA + uint32_t(r) * ROW);
}
__device__ __forceinline__ void load_B(double (&v)[R], uint32_t baseB) {
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = lds_a(baseB + uint32_t(r) * 8u);
}

// a8: this plane's half of Re(i^q S), S = sum_j conj(x'_j) phi_j (plane.cuh), warp-summed
__device__ __forceinline__ double readout(const double (&v)[R], uint32_t xa, uint32_t pl, uint32_t t,
                                          const PauliTerm& Tl, int q) {
  const uint32_t qi = uint32_t(q & 1);
  const uint32_t rp = pl ^ qi, xs = qi & (pl ^ 1u);
  const uint32_t mh = Tl.xm >> TB, tl = t ^ (Tl.xm & 31u), zh = Tl.zm >> TB;
  const uint32_t sg0 = (__popc(t & Tl.zm & 31u) & 1u) ^ xs;
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
  double half = (ac[0] + ac[1]) + (ac[2] + ac[3]);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) half += __shfl_xor_sync(0xffffffffu, half, off);
  return half;
}

// SMEM "small" region: per pair the task index and the Im warp's two readout halves, both double
// buffered by iteration parity; the CTA's task counter; the per-warp partial quadruples of the
// end-of-piece reduction
template <int W>
__host__ __device__ constexpr size_t small_bytes() {
  return sizeof(double) * (size_t(W / 2) * 4 + size_t(W) * 4) + sizeof(int) * (size_t(W / 2) * 2 + 2);
}

// a3 (within a CTA) + a9.  The CTA's share of the K x C flattened work is static and cost-weighted
// (as in plane_kernel: it decides which thetas' x the CTA stages); inside a theta piece the six warp
// pairs take tasks (the Re and Im circuit of one (k, l, j)) one at a time from a shared counter, so
// no pair idles while another still holds a statically assigned tail (ncu, K = 1: SM active cycles
// spread 6 % min-to-max under the static split).  Determinism does not depend on which pair ran a
// task: each task's two terms go to out_terms, and after the piece the CTA sums c_l^* c_k x term
// over the piece's circuits in a fixed order (per-thread strided loop, fixed warp tree, fixed warp
// order) -- the weighted sums are bitwise reproducible run to run.
__global__ void __launch_bounds__(WARPS * 32, 1)  // <= 168 registers: 12 warps per SM
plane2_kernel(const double2* __restrict__ x_all, const PauliTerm* __restrict__ tab, const double2* __restrict__ coef,
              const double2* __restrict__ hv, double hv_scale, int L, int64_t c0, int64_t C, int K,
              double* __restrict__ out_terms, double* __restrict__ partials, int with_cost,
              double* __restrict__ red_out, unsigned* __restrict__ counter, P2PArgs p2p) {
  (void)hv; (void)hv_scale;
  if (threadIdx.x == 0) P2TS(0);
  constexpr size_t SMALL = small_bytes<WARPS>();
  double* shalf = reinterpret_cast<double*>(dvqls_smem);  // [NP][2 parities][2 circuits]
  double* sred = shalf + NP * 4;                            // [WARPS][4]
  int* stask = reinterpret_cast<int*>(sred + WARPS * 4);    // [NP][2 parities]
  int* sctr = stask + NP * 2;
  const uint32_t sb = plane::sbase();
  const uint32_t xa = (sb + uint32_t(SMALL) + XALIGN - 1) & ~(XALIGN - 1);
  {
    uint32_t dsz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
    if (xa + XREG + WARPS * BUF - sb > dsz) __trap();
  }
  double* sd = reinterpret_cast<double*>(reinterpret_cast<char*>(dvqls_smem) + (xa - sb));

  const int warp = threadIdx.x >> 5;
  const uint32_t t = threadIdx.x & 31;
  const int pair = warp >> 1;
  const uint32_t pl = uint32_t(warp & 1);
  const uint32_t buf = xa + XREG + uint32_t(warp) * BUF;
  const uint32_t baseA = buf + t * 8u, baseB = buf + t * ROW;
  const int n1 = NQ + 1;

  const int64_t G = gridDim.x;
  const int64_t w0 = wcum(c0, NQ), Wt = wcum(c0 + C, NQ) - w0, Wall = Wt * K;
  // every boundary on a task boundary (even circuit index; c0 and C are even, dvqls_shard_range), so
  // a warp always holds the Re and Im circuits of one task together
  auto flat_of = [&](int64_t w) -> int64_t {
    if (w >= Wall) return int64_t(K) * C;
    const int64_t th = w / Wt, rem = w - th * Wt;
    const int64_t c = min(max(winv(w0 + rem, NQ) - c0, int64_t(0)), C) & ~int64_t(1);
    return th * C + c;
  };
  if ((c0 | C) & 1) __trap();  // host invariant: whole tasks per rank
  const int64_t Fb = Wall > 0 ? flat_of(Wall * (int64_t)blockIdx.x / G) : 0;
  const int64_t Fe =
      Wall <= 0 ? 0 : blockIdx.x + 1 == G ? int64_t(K) * C : flat_of(Wall * ((int64_t)blockIdx.x + 1) / G);
  const int th_first = C > 0 ? int(Fb / C) : 0, th_last = Fe > Fb ? int((Fe - 1) / C) : th_first - 1;
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    if (k < th_first || k > th_last)
      for (int q = 0; q < 4; ++q) partials[(size_t(k) * G + blockIdx.x) * 4 + q] = 0.0;
  const int64_t tk0 = c0 >> 1;  // global task index of local task 0
  // everything above overlaps the prefix kernel under programmatic dependent launch (it reads only
  // launch arguments and writes partials, which the previous call finished with before the prefix
  // started); x is read only after the prefix's completion
  pdl_wait();
  if (threadIdx.x == 0) P2TS(1);

  for (int kth = th_first; kth <= th_last; ++kth) {
    const int64_t pa = max(Fb, int64_t(kth) * C) - int64_t(kth) * C;
    const int64_t pb = min(Fe, int64_t(kth + 1) * C) - int64_t(kth) * C;
    const int ta = int(pa >> 1), tb = int(pb >> 1);  // this piece's tasks [ta, tb)
    const double2* x = x_all + (size_t)kth * N;
    double* terms = out_terms + (size_t)kth * C;
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double2 a = x[i];
      sd[i] = a.x;
      sd[N + i] = -a.x;
      sd[2 * N + i] = a.y;
      sd[3 * N + i] = -a.y;
    }
    if (threadIdx.x == 0) *sctr = ta;
    __syncthreads();
    if (threadIdx.x == 0) P2TS(2);

    // one task (Re and Im circuit) per iteration; one copy of each path (instruction-cache footprint)
    int prev = -1;
    double pha = 0.0, phb = 0.0;  // Re warp: its halves of the previous task
#pragma unroll 1
    for (int it = 0;; ++it) {
      const int par = it & 1;
      if (pl == 0 && t == 0) stask[2 * pair + par] = atomicAdd(sctr, 1);
      // the pair's barrier: publishes the new task index and the Im warp's halves of the previous task
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(64) : "memory");
      if (pl == 0 && prev >= 0 && t < 2) {  // a9: combine the two planes' halves of the previous task
        const double* sh = shalf + 4 * pair + 2 * (par ^ 1);
        terms[2 * prev + int(t)] = (t == 0 ? pha : phb) + sh[t];
      }
      const int task = stask[2 * pair + par];
      if (task >= tb) {
        if (pl == 0 && t == 0) P2TS(6 + pair);
        break;
      }
      const int64_t tk = tk0 + task, lk = tk / n1;
      const int s_ = int(tk - lk * n1);
      const int kq = int(lk % L), lq = int(lk / L);
      const PauliTerm Tk = tab[kq];
      const PauliTerm Tl = tab[lq];
      double ha, hb;
      if (s_ > 0) {  // numerator task: Re circuit A, Im circuit B, skewed by one phase
        const int p = NQ - s_;
        double va[R], vb[R];
        gather(va, xa, pl, t, Tk);
        // seg 1: F1(A) | gather(B)
        fwht<0, RB>(va);
        gather(vb, xa, pl, t, Tk);
        // seg 2: X1(A) | F1(B)
        __syncwarp();
        store_A(va, baseA);
        fwht<0, 3>(vb);
        __syncwarp();
        load_B(va, baseB);
        fwht<3, RB>(vb);
        // Z_j's stage: index bit p is register bit p of layout B (F3) for p < 5, register bit
        // p - 5 of layout A (F4) otherwise
        const int z3 = p < RB ? p : -1, z4 = p < RB ? -1 : p - RB;
        // seg 3: F2 Z F3 (A) | X1(B)
        __syncwarp();
        store_A(vb, baseA);
        fwht<0, TB>(va);
        __syncwarp();
        load_B(vb, baseB);
        fwht_z<0, TB>(va, z3);
        // seg 4: X2(A) | F2 Z F3 (B)
        __syncwarp();
        store_B(va, baseB);
        fwht<0, TB>(vb);
        __syncwarp();
        load_A(va, baseA);
        fwht_z<0, TB>(vb, z3);
        // seg 5: F4(A) | X2(B)
        __syncwarp();
        store_B(vb, baseB);
        fwht_z<0, 3>(va, z4);
        __syncwarp();
        load_A(vb, baseA);
        fwht_z<3, RB>(va, z4);
        // seg 6: readout(A) | F4(B);  seg 7: readout(B)
        const int qa = (Tk.ny + Tl.ny) & 3, qb = (Tk.ny + Tl.ny + 3) & 3;
        ha = readout(va, xa, pl, t, Tl, qa);
        fwht_z<0, RB>(vb, z4);
        hb = readout(vb, xa, pl, t, Tl, qb);
        constexpr double sc = 1.0 / double(N);
        ha *= (qa == 1 || qa == 2) ? -sc : sc;
        hb *= (qb == 1 || qb == 2) ? -sc : sc;
      } else {  // denominator task: c-A_k gather and c-A_l readout of each circuit
        ha = hb = 0.0;
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {
          double v[R];
          gather(v, xa, pl, t, Tk);
          const int q = (Tk.ny + Tl.ny + 3 * part) & 3;
          const double half = readout(v, xa, pl, t, Tl, q);
          if (part == 0) ha = (q == 1 || q == 2) ? -half : half;
          else hb = (q == 1 || q == 2) ? -half : half;
        }
      }
      if (pl == 1 && t == 0) {
        shalf[4 * pair + 2 * par] = ha;
        shalf[4 * pair + 2 * par + 1] = hb;
      }
      pha = ha;
      phb = hb;
      prev = task;
    }
    __syncthreads();  // every term of the piece is in out_terms
    if (threadIdx.x == 0) P2TS(3);
    // a9: sum_c c_l^* c_k term_c over the piece [pa, pb) in a fixed order
    {
      double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
      for (int64_t cc = pa + threadIdx.x; cc < pb; cc += blockDim.x) {
        const double val = terms[cc];
        const int64_t c = c0 + cc, tk = c >> 1, lk = tk / n1;
        const int prt = int(c & 1), ss = int(tk - lk * n1), kk = int(lk % L), ll = int(lk / L);
        const double2 cl_ = coef[ll], ck = coef[kk];
        const double wr = cl_.x * ck.x + cl_.y * ck.y, wi = cl_.x * ck.y - cl_.y * ck.x;
        const double cr = (prt == 0 ? wr : -wi) * val, ci = (prt == 0 ? wi : wr) * val;
        if (ss == 0) { e2 += cr; e3 += ci; } else { e0 += cr; e1 += ci; }
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        e0 += __shfl_xor_sync(0xffffffffu, e0, off);
        e1 += __shfl_xor_sync(0xffffffffu, e1, off);
        e2 += __shfl_xor_sync(0xffffffffu, e2, off);
        e3 += __shfl_xor_sync(0xffffffffu, e3, off);
      }
      if (t == 0) {
        sred[4 * warp] = e0; sred[4 * warp + 1] = e1; sred[4 * warp + 2] = e2; sred[4 * warp + 3] = e3;
      }
      __syncthreads();
      if (threadIdx.x == 0) {  // fixed warp order
        double f0 = 0, f1 = 0, f2 = 0, f3 = 0;
        for (int g = 0; g < WARPS; ++g) {
          f0 += sred[4 * g]; f1 += sred[4 * g + 1]; f2 += sred[4 * g + 2]; f3 += sred[4 * g + 3];
        }
        double* o = partials + ((size_t)kth * G + blockIdx.x) * 4;
        o[0] = f0; o[1] = f1; o[2] = f2; o[3] = f3;
        P2TS(4);
      }
    }
  }
  if (red_out) finish_all(partials, int(G), K, NQ, with_cost, red_out, counter, p2p);
  if (threadIdx.x == 0) P2TS(5);
}

// dynamic SMEM to request when the dynamic base sits at shared-window address sb
__host__ __device__ constexpr size_t smem_bytes(uint32_t sb) {
  return ((sb + small_bytes<WARPS>() + XALIGN - 1) & ~size_t(XALIGN - 1)) - sb + XREG + size_t(WARPS) * BUF;
}

}  // namespace plane2
}  // namespace dvqls
