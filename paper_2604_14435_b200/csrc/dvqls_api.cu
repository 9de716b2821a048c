// dvqls_api.cu - the C ABI of libdvqls.so (declared and documented in include/dvqls.h).
//
// Host side of the hot path: context build, launch of the
// sm_100a kernels (kernels.cuh), the cross-rank reduction (a10, "Global
// Reduction", Alg. 1 Step 4c P:461-463) over a library-owned NCCL communicator,
// and marshalling of host buffers.  No arithmetic of the method runs here; the
// host only validates inputs, precomputes the Householder vector of U_b and
// moves bytes.

#include <cuda_runtime.h>

#include <cmath>
#include <complex>
#include <cstdarg>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/dvqls.h"
#include "kernels.cuh"
#include "plane.cuh"
#include "tile.cuh"
#include "stream.cuh"
#include "stream_plane.cuh"
#include "onchip_plane.cuh"
#include "pauli.cuh"
#include "global.cuh"
#include "decomp.cuh"
#include "nccl_dl.h"

using namespace dvqls;

namespace {

constexpr int kMaxRegQubits = 10;  // register-resident path (one circuit per warp or less)
constexpr int kMaxQubits = 24;     // tile path: SMEM tile (n <= 12) or global streaming (n <= 24)
constexpr size_t kScratchBudget = size_t(48) << 30;  // bytes of per-CTA branch scratch (n > 12)

struct KernelCfg {
  const void* fn = nullptr;
  int warps = 0;
  size_t smem = 0;
  int gpw = 0;  // circuit groups per warp
  int groups = 0;  // circuit groups per CTA
};

template <int NQ, bool HH, int W>
KernelCfg make_cfg() {
  using S = Shape<NQ>;
  KernelCfg k;
  k.fn = (const void*)&hadamard_kernel<NQ, W, HH>;
  k.warps = W;
  k.gpw = S::GPW;
  k.smem = sizeof(double2) * (size_t(HH ? 3 : 2) * S::N + size_t(W) * S::GPW * S::N) +
           sizeof(double) * 4 * size_t(W) * S::GPW;
  k.groups = W * S::GPW;
  return k;
}

// n = 10, uniform b: the real-plane kernel (plane.cuh), one circuit per warp pair
template <int W>
KernelCfg make_plane_cfg() {
  KernelCfg k;
  k.fn = (const void*)&plane::plane_kernel<W>;
  k.warps = W;
  k.gpw = 1;
  k.groups = W / 2;
  // the x planes sit at a 16 KB-aligned shared-window address inside the allocation: size it
  // for the actual dynamic base (reserved SMEM + this kernel's static SMEM); the kernel traps
  // if the base differs
  cudaFuncAttributes fa{};
  int dev = 0, reserved = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaFuncGetAttributes(&fa, k.fn);
  const uint32_t sb = uint32_t(reserved) + ((uint32_t(fa.sharedSizeBytes) + 15u) & ~15u);
  k.smem = plane::smem_bytes<W>(sb);
  return k;
}

// n >= 9 keeps 32 amplitudes per thread (128 registers of branch state).
// Registers are split per SM sub-partition (16K each), so the choices are 8 warps
// (2 per scheduler, <= 255 registers) or 12 warps (3 per scheduler, <= 168).
// Measured on B200 (profiles/): 12 warps is faster for the uniform-b path; the
// Householder path needs a third N-vector of SMEM and only fits 8.
// DVQLS_WARPS=8 forces the 8-warp variant (tuning knob).
template <int NQ, bool HH>
KernelCfg pick_cfg() {
  if constexpr (NQ == 10 && !HH) {
    // DVQLS_PLANE=0 selects the complex-layout kernel (A/B comparison knob)
    const char* pe = getenv("DVQLS_PLANE");
    if (!pe || atoi(pe) != 0) {
      const char* e = getenv("DVQLS_WARPS");
      const int w = e ? atoi(e) : 20;
      // registers are split per SM sub-partition (16K each): 16 warps (4 per scheduler, <= 128
      // registers) or 20 (5 per scheduler, <= 96); measured on B200, 20 is faster
      if (w == 16) return make_plane_cfg<16>();
      return make_plane_cfg<20>();
    }
  }
  if constexpr (NQ >= 9) {
    const char* e = getenv("DVQLS_WARPS");
    const int w = e ? atoi(e) : 12;
    if (w == 12 && !HH) return make_cfg<NQ, HH, 12>();
    return make_cfg<NQ, HH, 8>();
  } else {
    return make_cfg<NQ, HH, 16>();
  }
}

template <bool HH>
KernelCfg cfg_for(int n) {
  switch (n) {
    case 1: return pick_cfg<1, HH>();
    case 2: return pick_cfg<2, HH>();
    case 3: return pick_cfg<3, HH>();
    case 4: return pick_cfg<4, HH>();
    case 5: return pick_cfg<5, HH>();
    case 6: return pick_cfg<6, HH>();
    case 7: return pick_cfg<7, HH>();
    case 8: return pick_cfg<8, HH>();
    case 9: return pick_cfg<9, HH>();
    case 10: return pick_cfg<10, HH>();
    default: return KernelCfg{};
  }
}

}  // namespace

struct dvqls_ctx {
  int n = 0, layers = 0, L = 0, P = 0, N = 0;
  int bkind = DVQLS_B_UNIFORM, entangler = 0;
  int device = 0, rank = 0, world = 1, max_batch = 16, timing = 0;
  int64_t C = 0, c0 = 0, c1 = 0, chunk = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;

  KernelCfg kc;
  int grid = 0;     // CTAs per theta (tile path) / for one theta (register path)
  int grid_cap = 0; // register path: resident CTAs (SMs x occupancy), the cap of a K-theta launch
  int64_t NG = 0;   // circuit groups per theta
  int prefix_threads = 0;
  int prefix_rb = 3;
  const void* prefix_fn = nullptr;
  bool pdl = false;  // Hadamard kernel launched as a programmatic dependent of the prefix
  size_t prefix_smem = 0;
  double hv_scale = 0.0;

  PauliTerm* d_tab = nullptr;
  double2* d_coef = nullptr;
  double2* d_hv = nullptr;
  double* d_theta = nullptr;     // max_batch * P
  double2* d_x = nullptr;        // max_batch * N
  double* d_terms = nullptr;     // max_batch * chunk
  double* d_partials = nullptr;  // max_batch * NG * 4
  double* d_ep = nullptr;        // max_batch * 4 (allreduce buffer)
  double* d_out = nullptr;       // max_batch * 5
  double* d_gather = nullptr;    // world * chunk (terms allgather)
  double* h_stage = nullptr;     // pinned staging
  unsigned* d_counter = nullptr; // last-CTA tickets, one per theta slot
  // fused NVLink allreduce (world > 1): own symmetric buffer + IPC-mapped peer buffers
  bool p2p = false;
  char* d_sym = nullptr;
  std::vector<char*> peer_ptrs;
  char** d_peers = nullptr;
  unsigned long long epoch = 0;
  bool tile_path = false;        // n > 10 (stream.cuh)
  int team = 0, nteams = 0;      // n >= 15: team mode (stream_team_kernel), T CTAs per circuit
  double* d_team_acc = nullptr;  // nteams * 2 * team
  unsigned* d_team_ctr = nullptr;  // nteams barrier counters + 1 error flag
  int tile_bits = 12;            // tile path: amplitudes per SMEM tile = 2^tile_bits
  double2* d_scratch = nullptr;  // grid * N (n > 12; doubles when pstream)
  bool pstream = false;          // n >= 11, uniform b: real-plane streaming kernel (stream_plane.cuh)
  bool onchip = false;           // n = 11, 12, uniform b: 2-exchange real-plane kernel (onchip_plane.cuh)
  double* d_xq = nullptr;        // onchip: [K][x_re | -x_re | x_im | -x_im]
  double* d_xp = nullptr;        // planar copy of x for pstream: [K][re N | im N]
  std::vector<void**> carved;    // device buffers carved from a caller workspace (not freed)
  double2* d_x2 = nullptr;       // ring ping-pong buffer (n > 12 prefix)
  double2* d_gates = nullptr;    // fused-gate table (n > 12 prefix)
  int64_t* d_cidx = nullptr;     // circuit subset (dvqls_terms_subset)
  double* d_sub = nullptr;
  int64_t sub_cap = 0;
  size_t h_stage_bytes = 0;

  // NEXT-2 algebraic fast path (opts.mode = DVQLS_MODE_PAULI; pauli.cuh)
  int mode = DVQLS_MODE_CIRCUITS;
  int64_t D = 0, d0 = 0, d1 = 0;  // distinct observables; this rank's block [d0, d1)
  int pgrid = 0;                  // CTAs of pauli_expect_kernel per theta (cost path)
  pauli::Obs* d_obs = nullptr;
  double2* d_wE = nullptr;        // per observable: sum of c_l^* c_k i^q over numerator tasks
  double2* d_wP = nullptr;        // ... over denominator tasks
  uint32_t* d_task = nullptr;     // per task: (observable << 2) | q
  double2* d_e = nullptr;         // D expectations of the last terms call
  size_t pauli_smem = 0;

  // NEXT-3 global cost (global.cuh)
  double2* d_b = nullptr;          // b amplitudes (AMPLITUDES only; uniform b needs none)
  double* d_beta = nullptr;        // max_batch * L * 2
  double* d_out6 = nullptr;        // max_batch * 6
  unsigned* d_gcounter = nullptr;  // last-CTA tickets of overlap_kernel

  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool timed_once = false;
  std::string err;
};

namespace {

int fail(dvqls_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return fail(ctx, DVQLS_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),     \
                  __FILE__, __LINE__);                                                           \
  } while (0)

#define CKN(call)                                                                                \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess)                                                                       \
      return fail(ctx, DVQLS_E_NCCL, "%s failed: %s", #call, nccl().GetErrorString(r_));         \
  } while (0)

thread_local std::string g_create_err;

// Symbolic product of Pauli operators in the representation P|i> = i^q (-1)^{popcount(i & z)}
// |i ^ m>:  (Q P)|i> = i^{q_P + q_Q + 2 popcount(m_P & z_Q)} (-1)^{i . (z_P ^ z_Q)} |i ^ m_P ^ m_Q>.
struct PauliOp {
  uint32_t m, z;
  int q;
};
PauliOp pauli_mul(const PauliOp& Q, const PauliOp& P) {  // Q * P (P applied first)
  return PauliOp{P.m ^ Q.m, P.z ^ Q.z, (P.q + Q.q + 2 * __builtin_popcount(P.m & Q.z)) & 3};
}
// Observable of task (l, k, s) for uniform b (NEXT-2): A_l X_j A_k (s = 1 + j) or A_l A_k (s = 0),
// X_j on system qubit j = index bit n - 1 - j (U_b Z_j U_b^+ = H Z H = X)
PauliOp task_observable(int n, const PauliTerm& Tl, const PauliTerm& Tk, int s) {
  PauliOp r{Tk.xm, Tk.zm, Tk.ny & 3};
  if (s > 0) r = pauli_mul(PauliOp{1u << (n - 1 - (s - 1)), 0u, 0}, r);
  return pauli_mul(PauliOp{Tl.xm, Tl.zm, Tl.ny & 3}, r);
}

P2PArgs make_p2p(dvqls_ctx* ctx, double* red_out, int with_cost) {
  P2PArgs p2p{1, 0, ctx->max_batch, 0ull, nullptr};
  if (red_out && with_cost && ctx->p2p) {
    p2p.world = ctx->world;
    p2p.rank = ctx->rank;
    p2p.epoch = ++ctx->epoch;
    p2p.peers = ctx->d_peers;
  }
  return p2p;
}

// NEXT-2: distinct observables [d0, d1) of every theta; e -> out_e (nullable), fused reduction
int launch_pauli(dvqls_ctx* ctx, int K, int64_t d0, int64_t d1, double2* out_e, int grid, double* red_out,
                 int with_cost) {
  P2PArgs p2p = make_p2p(ctx, red_out, with_cost);
  const int stage = ctx->pauli_smem > 0 ? 1 : 0;
  void* args[] = {(void*)&ctx->d_x, (void*)&ctx->n, (void*)&ctx->d_obs, (void*)&ctx->d_wE, (void*)&ctx->d_wP,
                  (void*)&d0, (void*)&d1, (void*)&ctx->D, (void*)&out_e, (void*)&ctx->d_partials,
                  (void*)&with_cost, (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p, (void*)&stage};
  CK(cudaLaunchKernel((const void*)&pauli::pauli_expect_kernel, dim3(grid, K), dim3(pauli::WARPS * 32), args,
                      ctx->pauli_smem, ctx->stream));
  return DVQLS_OK;
}

// Hadamard-test kernel over circuits [c0, c0 + C) (or the list cidx[0..C)) of every theta.
// red_out != NULL: the kernel's last CTA per theta also performs the fixed-order reduction
// (with_cost: 5 doubles C, E, Psi per theta; else 4 doubles E, Psi for the allreduce).
int launch_hadamard(dvqls_ctx* ctx, int K, int64_t c0, int64_t C, const int64_t* cidx, double* terms, int grid,
                    double* red_out = nullptr, int with_cost = 0) {
  P2PArgs p2p = make_p2p(ctx, red_out, with_cost);
  if (ctx->team > 0 && !cidx) {  // team mode: cooperative launch (team barriers need co-residency)
    int T = ctx->team;
    unsigned* err = ctx->d_team_ctr + ctx->nteams;
    void* args[] = {(void*)&ctx->d_x, (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->L, (void*)&ctx->n,
                    (void*)&c0, (void*)&C, (void*)&K, (void*)&T, (void*)&ctx->d_scratch, (void*)&terms,
                    (void*)&ctx->d_partials, (void*)&ctx->d_team_acc, (void*)&ctx->d_team_ctr, (void*)&err,
                    (void*)&with_cost, (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p};
    CK(cudaLaunchCooperativeKernel((const void*)&stream::stream_team_kernel<12>, dim3(ctx->nteams * T),
                                   dim3(stream::TS<12>::THREADS), args, sizeof(double2) * stream::TS<12>::TN,
                                   ctx->stream));
    return DVQLS_OK;
  }
  if (ctx->tile_path && ctx->n > ctx->tile_bits) grid = std::max(1, grid / K);  // scratch: grid CTAs in total
  dim3 g(grid, K);
  if (!ctx->tile_path) {  // one persistent 1-D grid over the flattened K x C work (kernels.cuh)
    // enough CTAs for all K thetas' circuits, up to one resident wave (a grid sized for one
    // theta would leave most SMs idle on small problems evaluated in large batches)
    grid = int(std::max<int64_t>(
        1, std::min<int64_t>(ctx->grid_cap, (int64_t(K) * C + ctx->kc.groups - 1) / std::max(1, ctx->kc.groups))));
    void* args[] = {(void*)&ctx->d_x,   (void*)&ctx->d_tab, (void*)&ctx->d_coef,  (void*)&ctx->d_hv,
                    (void*)&ctx->hv_scale, (void*)&ctx->L, (void*)&c0, (void*)&C, (void*)&K,
                    (void*)&terms, (void*)&ctx->d_partials, (void*)&with_cost, (void*)&red_out,
                    (void*)&ctx->d_counter, (void*)&p2p};
    if (ctx->pdl) {  // scheduled while the prefix runs; the kernel's griddepcontrol.wait orders the reads
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(ctx->kc.warps * 32);
      lc.dynamicSmemBytes = ctx->kc.smem;
      lc.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      CK(cudaLaunchKernelExC(&lc, ctx->kc.fn, args));
    } else {
      CK(cudaLaunchKernel(ctx->kc.fn, dim3(grid), dim3(ctx->kc.warps * 32), args, ctx->kc.smem, ctx->stream));
    }
  } else if (ctx->onchip) {  // [x_re | -x_re | x_im | -x_im], then the 2-exchange kernel, 1-D grid
    const size_t blk = sizeof(double) * 4 * size_t(ctx->N);  // one theta's x block, a power of two
    double* xq = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ctx->d_xq) + blk - 1) & ~uintptr_t(blk - 1));
    onchip::to_planar4_kernel<<<std::min<int64_t>(1184, (int64_t(K) * ctx->N + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->d_x, uint32_t(ctx->N), uint32_t(K), xq);
    const int g1 = int(std::max<int64_t>(
        1, std::min<int64_t>(ctx->grid_cap, (int64_t(K) * C + ctx->kc.groups - 1) / std::max(1, ctx->kc.groups))));
    void* args[] = {(void*)&xq, (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->L, (void*)&c0,
                    (void*)&C, (void*)&K, (void*)&terms, (void*)&ctx->d_partials, (void*)&with_cost,
                    (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p};
    CK(cudaLaunchKernel(ctx->kc.fn, dim3(g1), dim3(ctx->kc.warps * 32), args, ctx->kc.smem, ctx->stream));
  } else if (ctx->pstream) {  // planar x, then the real-plane streaming kernel
    streamp::to_planar_kernel<<<std::min<int64_t>(1184, (int64_t(K) * ctx->N + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->d_x, uint32_t(ctx->N), uint32_t(K), ctx->d_xp);
    double* scr = reinterpret_cast<double*>(ctx->d_scratch);
    void* args[] = {(void*)&ctx->d_xp, (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->L, (void*)&ctx->n,
                    (void*)&c0, (void*)&C, (void*)&cidx, (void*)&scr, (void*)&terms, (void*)&ctx->d_partials,
                    (void*)&with_cost, (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p};
    CK(cudaLaunchKernel(ctx->kc.fn, g, dim3(ctx->kc.warps * 32), args, ctx->kc.smem, ctx->stream));
  } else {
    void* args[] = {(void*)&ctx->d_x, (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->d_hv,
                    (void*)&ctx->hv_scale, (void*)&ctx->L, (void*)&ctx->n, (void*)&c0, (void*)&C,
                    (void*)&cidx, (void*)&ctx->d_scratch, (void*)&terms, (void*)&ctx->d_partials,
                    (void*)&with_cost, (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p};
    CK(cudaLaunchKernel(ctx->kc.fn, g, dim3(ctx->kc.warps * 32), args, ctx->kc.smem, ctx->stream));
  }
  return DVQLS_OK;
}

// n > 12: V(theta)|0> in global memory, one launch per pass (tile.cuh)
int launch_prefix_global(dvqls_ctx* ctx, int K, const double* thetas_dev) {
  const int n = ctx->n, G = n * ctx->layers;
  const uint32_t N = uint32_t(ctx->N);
  const int ng = n <= 12 ? 1 : (n <= 21 ? 2 : 3);
  for (int k = 0; k < K; ++k) {
    double2* x = ctx->d_x + size_t(k) * N;
    double2* y = ctx->d_x2;
    tile::prefix_gates_kernel<<<(G + 127) / 128, 128, 0, ctx->stream>>>(thetas_dev + size_t(k) * ctx->P, G,
                                                                           ctx->d_gates);
    tile::prefix_init_kernel<<<1024, 256, 0, ctx->stream>>>(x, N);
    for (int layer = 0; layer < ctx->layers; ++layer) {
      for (int gi = 0; gi < ng; ++gi)
        tile::prefix_gate_pass<<<N >> tile::TBITS, tile::THREADS, sizeof(double2) * tile::TN, ctx->stream>>>(
            x, ctx->d_gates, n, gi, layer);
      tile::prefix_ring_kernel<<<1024, 256, 0, ctx->stream>>>(x, y, n, ctx->entangler);
      CK(cudaMemcpyAsync(x, y, sizeof(double2) * N, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CK(cudaGetLastError());
  }
  return DVQLS_OK;
}

int launch_eval(dvqls_ctx* ctx, int K, const double* thetas_dev, bool want_cost, double* out_dev) {
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (ctx->prefix_rb < 0) {
    int rc = launch_prefix_global(ctx, K, thetas_dev);
    if (rc) return rc;
  } else if (ctx->prefix_rb == 0) {
    void* args[] = {(void*)&ctx->layers, (void*)&ctx->entangler, (void*)&thetas_dev, (void*)&ctx->d_x};
    CK(cudaLaunchKernel(ctx->prefix_fn, dim3(K), dim3(ctx->prefix_threads), args, ctx->prefix_smem, ctx->stream));
  } else {
    void* args[] = {(void*)&ctx->n, (void*)&ctx->layers, (void*)&ctx->entangler, (void*)&thetas_dev,
                    (void*)&ctx->d_x};
    CK(cudaLaunchKernel(ctx->prefix_fn, dim3(K), dim3(ctx->prefix_threads), args, ctx->prefix_smem, ctx->stream));
  }
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  const int64_t Cloc = ctx->c1 - ctx->c0;
  {
    // a9 (+ a10 on one rank) fused into the kernel tail (last-CTA fixed-order reduction)
    const bool direct = ctx->world == 1 || ctx->p2p;  // kernel writes the final (C, E, Psi)
    double* red = want_cost ? (direct ? out_dev : ctx->d_ep) : nullptr;
    if (ctx->mode == DVQLS_MODE_PAULI) {
      int rc;
      if (want_cost) {
        rc = launch_pauli(ctx, K, ctx->d0, ctx->d1, nullptr, ctx->pgrid, red, direct ? 1 : 0);
      } else {  // terms: every observable on every rank (cheap), then this rank's circuit block
        rc = launch_pauli(ctx, K, 0, ctx->D, ctx->d_e, ctx->pgrid, nullptr, 0);
        if (!rc) {
          pauli::pauli_scatter_kernel<<<296, 256, 0, ctx->stream>>>(ctx->d_e, ctx->d_task, ctx->c0, Cloc, ctx->d_terms);
          CK(cudaGetLastError());
        }
      }
      if (rc) return rc;
    } else {
      int rc = launch_hadamard(ctx, K, ctx->c0, Cloc, nullptr, ctx->d_terms, ctx->grid, red, direct ? 1 : 0);
      if (rc) return rc;
    }
  }
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  if (want_cost) {
    if (ctx->world > 1 && !ctx->p2p) {
      CKN(nccl().AllReduce(ctx->d_ep, ctx->d_ep, size_t(4) * K, ncclDouble, ncclSum, ctx->comm, ctx->stream));
      finalize_kernel<<<1, 32 * ((K + 31) / 32), 0, ctx->stream>>>(ctx->d_ep, K, ctx->n, out_dev);
      CK(cudaGetLastError());
    }
  }
  if (ctx->timing) {
    CK(cudaEventRecord(ctx->ev[3], ctx->stream));
    ctx->timed_once = true;
  }
  return DVQLS_OK;
}

void release(dvqls_ctx* c) {
  if (!c) return;
  for (void** p : c->carved) *p = nullptr;  // owned by the caller's workspace
  for (int q = 0; q < int(c->peer_ptrs.size()); ++q)
    if (q != c->rank && c->peer_ptrs[q]) cudaIpcCloseMemHandle(c->peer_ptrs[q]);
  cudaFree(c->d_sym); cudaFree(c->d_peers);
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  cudaFree(c->d_tab); cudaFree(c->d_coef); cudaFree(c->d_hv); cudaFree(c->d_theta); cudaFree(c->d_x);
  cudaFree(c->d_terms); cudaFree(c->d_partials); cudaFree(c->d_ep); cudaFree(c->d_out); cudaFree(c->d_gather);
  cudaFree(c->d_obs); cudaFree(c->d_wE); cudaFree(c->d_wP); cudaFree(c->d_task); cudaFree(c->d_e);
  cudaFree(c->d_team_acc); cudaFree(c->d_team_ctr);
  cudaFree(c->d_b); cudaFree(c->d_beta); cudaFree(c->d_out6); cudaFree(c->d_gcounter);
  cudaFree(c->d_counter); cudaFree(c->d_scratch); cudaFree(c->d_xp); cudaFree(c->d_xq); cudaFree(c->d_x2); cudaFree(c->d_gates); cudaFree(c->d_cidx); cudaFree(c->d_sub);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (auto& e : c->ev) if (e) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
}

}  // namespace

// Symmetric buffers for the fused allreduce: allocate, exchange IPC handles with an NCCL
// allgather (create-time only), map every peer's buffer.  If mapping fails the context
// falls back to ncclAllReduce on the cost path.
int setup_p2p(dvqls_ctx* ctx) {
  const size_t bytes = size_t(2) * ctx->world * ctx->max_batch * (32 + 8);
  CK(cudaMalloc((void**)&ctx->d_sym, bytes));
  CK(cudaMemset(ctx->d_sym, 0, bytes));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->d_sym));
  char* d_h = nullptr;
  CK(cudaMalloc((void**)&d_h, sizeof(h) * (ctx->world + 1)));
  CK(cudaMemcpy(d_h, &h, sizeof(h), cudaMemcpyHostToDevice));
  ncclResult_t r = nccl().AllGather(d_h, d_h + sizeof(h), sizeof(h), ncclChar, ctx->comm, ctx->stream);
  if (r != ncclSuccess) {
    cudaFree(d_h);
    return fail(ctx, DVQLS_E_NCCL, "handle allgather: %s", nccl().GetErrorString(r));
  }
  std::vector<cudaIpcMemHandle_t> all(ctx->world);
  CK(cudaMemcpyAsync(all.data(), d_h + sizeof(h), sizeof(h) * ctx->world, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(d_h);
  ctx->peer_ptrs.assign(ctx->world, nullptr);
  bool ok = true;
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) { ctx->peer_ptrs[q] = ctx->d_sym; continue; }
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      break;
    }
    ctx->peer_ptrs[q] = static_cast<char*>(p);
  }
  if (!ok) {  // every rank must agree: fall back together if any rank could not map
    ctx->p2p = false;
  } else {
    ctx->p2p = true;
  }
  int flag = ctx->p2p ? 1 : 0, all_ok = 0;
  {
    int* d_f = nullptr;
    CK(cudaMalloc((void**)&d_f, sizeof(int)));
    CK(cudaMemcpy(d_f, &flag, sizeof(int), cudaMemcpyHostToDevice));
    ncclResult_t r2 = nccl().AllReduce(d_f, d_f, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream);
    if (r2 != ncclSuccess) { cudaFree(d_f); return fail(ctx, DVQLS_E_NCCL, "p2p agreement"); }
    CK(cudaMemcpyAsync(&all_ok, d_f, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(d_f);
  }
  ctx->p2p = all_ok == 1;
  if (ctx->p2p) {
    CK(cudaMalloc((void**)&ctx->d_peers, sizeof(char*) * ctx->world));
    CK(cudaMemcpy(ctx->d_peers, ctx->peer_ptrs.data(), sizeof(char*) * ctx->world, cudaMemcpyHostToDevice));
  }
  return DVQLS_OK;
}

namespace {
// dvqls_create, or (plan_bytes != NULL) only the planning part of it: everything up to the
// device allocations runs as in a real create, then the total workspace size is returned and the
// context is released (dvqls_workspace_size).
int create_impl(dvqls_ctx** out, int n, int layers, int L, const char* paulis, const double* coeffs,
                const dvqls_bprep* bprep, const dvqls_opts* opts, size_t* plan_bytes) {
  g_create_err.clear();
  dvqls_ctx* ctx = nullptr;
  auto early = [&](int code, const char* msg) {
    g_create_err = msg;
    return code;
  };
  if (!out) return early(DVQLS_E_ARG, "out is NULL");
  *out = nullptr;
  if (n < 1 || n > 24) return early(DVQLS_E_ARG, "n_qubits must be in [1, 24]");
  if (layers < 1) return early(DVQLS_E_ARG, "layers must be >= 1");
  if (L < 1) return early(DVQLS_E_ARG, "n_terms must be >= 1");
  if (!paulis || !coeffs) return early(DVQLS_E_ARG, "pauli_terms / coeffs is NULL");
  if (n > kMaxQubits) return early(DVQLS_E_UNSUPPORTED, "this build evaluates n <= 24");
  if (n > 12 && bprep && bprep->kind == DVQLS_B_AMPLITUDES)
    return early(DVQLS_E_UNSUPPORTED, "amplitude b (Householder U_b) is implemented for n <= 12");

  ctx = new dvqls_ctx();
  ctx->n = n; ctx->layers = layers; ctx->L = L; ctx->P = 3 * n * layers; ctx->N = 1 << n;
  if (opts) {
    ctx->device = opts->device; ctx->rank = opts->rank; ctx->world = opts->world;
    ctx->entangler = opts->entangler; ctx->timing = opts->timing; ctx->mode = opts->mode;
    if (opts->max_batch > 0) ctx->max_batch = opts->max_batch;
  } else {
    ctx->device = -1; ctx->rank = 0; ctx->world = 1;
  }
  auto bail = [&](int code) {
    g_create_err = ctx->err;
    release(ctx);
    delete ctx;
    return code;
  };
  if (ctx->world < 1 || ctx->rank < 0 || ctx->rank >= ctx->world) {
    fail(ctx, DVQLS_E_ARG, "rank/world out of range");
    return bail(DVQLS_E_ARG);
  }
  if (ctx->mode != DVQLS_MODE_CIRCUITS && ctx->mode != DVQLS_MODE_PAULI) {
    fail(ctx, DVQLS_E_ARG, "mode must be DVQLS_MODE_CIRCUITS or DVQLS_MODE_PAULI");
    return bail(DVQLS_E_ARG);
  }
  if (ctx->mode == DVQLS_MODE_PAULI && bprep && bprep->kind != DVQLS_B_UNIFORM) {
    fail(ctx, DVQLS_E_UNSUPPORTED, "the Pauli fast path needs uniform b (U_b Z_j U_b^+ = X_j)");
    return bail(DVQLS_E_UNSUPPORTED);
  }
  if (ctx->entangler != 0 && ctx->entangler != 1) {
    fail(ctx, DVQLS_E_ARG, "entangler must be 0 (CNOT ring) or 1 (CZ ring)");
    return bail(DVQLS_E_ARG);
  }
  if (ctx->world > 1 && !plan_bytes && !(opts && opts->nccl_unique_id)) {
    fail(ctx, DVQLS_E_ARG, "world > 1 requires opts.nccl_unique_id");
    return bail(DVQLS_E_ARG);
  }

  // ---- a1: Pauli strings -> (x_mask, z_mask, n_Y), big-endian (reading 9) ----
  std::vector<PauliTerm> tab(L);
  std::set<std::string> seen;
  for (int l = 0; l < L; ++l) {
    std::string s(paulis + size_t(l) * n, size_t(n));
    if (!seen.insert(s).second) {
      fail(ctx, DVQLS_E_PAULI, "duplicate Pauli string %s (term %d)", s.c_str(), l);
      return bail(DVQLS_E_PAULI);
    }
    PauliTerm t{0, 0, 0, 0u};
    for (int q = 0; q < n; ++q) {
      const uint32_t bit = 1u << (n - 1 - q);
      switch (s[q]) {
        case 'I': break;
        case 'X': t.xm |= bit; break;
        case 'Y': t.xm |= bit; t.zm |= bit; t.ny += 1; break;
        case 'Z': t.zm |= bit; break;
        default:
          fail(ctx, DVQLS_E_PAULI, "bad Pauli character 0x%02x in term %d", (unsigned char)s[q], l);
          return bail(DVQLS_E_PAULI);
      }
    }
    // register-part sign word: bit r = popcount(r & (zm >> TB)) & 1, TB = n/2 (kernels.cuh Shape)
    const uint32_t zh = t.zm >> (n / 2);
    for (int r = 0; r < 32; ++r) t.wpar |= uint32_t(__builtin_popcount(uint32_t(r) & zh) & 1) << r;
    tab[l] = t;
  }
  std::vector<double2> coef(L);
  for (int l = 0; l < L; ++l) coef[l] = make_double2(coeffs[2 * l], coeffs[2 * l + 1]);

  // ---- U_b: uniform (H^{(x)n}) or Householder vector (reading 5) -------------
  std::vector<double2> hv;
  if (bprep) ctx->bkind = bprep->kind;
  if (ctx->bkind == DVQLS_B_AMPLITUDES) {
    if (!bprep->amps) {
      fail(ctx, DVQLS_E_BPREP, "AMPLITUDES b_prep needs amps");
      return bail(DVQLS_E_BPREP);
    }
    const int N = ctx->N;
    std::vector<std::complex<double>> b(N);
    double nn = 0;
    for (int i = 0; i < N; ++i) {
      b[i] = {bprep->amps[2 * i], bprep->amps[2 * i + 1]};
      nn += std::norm(b[i]);
    }
    if (std::fabs(std::sqrt(nn) - 1.0) > 1e-8) {
      fail(ctx, DVQLS_E_BPREP, "| ||b|| - 1 | = %.3e > 1e-8", std::fabs(std::sqrt(nn) - 1.0));
      return bail(DVQLS_E_BPREP);
    }
    const std::complex<double> w = std::abs(b[0]) > 0 ? b[0] / std::abs(b[0]) : std::complex<double>(1, 0);
    hv.resize(N);
    double vv = 0;
    for (int i = 0; i < N; ++i) {
      std::complex<double> v = (i == 0 ? 1.0 : 0.0) - std::conj(w) * b[i];
      hv[i] = make_double2(v.real(), v.imag());
      vv += std::norm(v);
    }
    ctx->hv_scale = vv > 0 ? 2.0 / vv : 0.0;
  } else if (ctx->bkind != DVQLS_B_UNIFORM) {
    fail(ctx, DVQLS_E_BPREP, "unknown b_prep kind %d", ctx->bkind);
    return bail(DVQLS_E_BPREP);
  }

  // ---- device, stream, kernel configuration ---------------------------------
  if ((ctx->device >= 0 && cudaSetDevice(ctx->device) != cudaSuccess) ||
      cudaGetDevice(&ctx->device) != cudaSuccess) {
    fail(ctx, DVQLS_E_CUDA, "no CUDA device");
    return bail(DVQLS_E_CUDA);
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, ctx->device) != cudaSuccess || prop.major != 10) {
    fail(ctx, DVQLS_E_CUDA, "libdvqls is built for sm_100a only (device cc %d.%d)", prop.major, prop.minor);
    return bail(DVQLS_E_CUDA);
  }
  if (opts && opts->cuda_stream) {
    ctx->stream = (cudaStream_t)opts->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      fail(ctx, DVQLS_E_CUDA, "cudaStreamCreate failed");
      return bail(DVQLS_E_CUDA);
    }
    ctx->own_stream = true;
  }
  ctx->tile_path = n > kMaxRegQubits;
  if (!ctx->tile_path) {
    ctx->kc = ctx->bkind == DVQLS_B_AMPLITUDES ? cfg_for<true>(n) : cfg_for<false>(n);
  } else {
    const bool hh = ctx->bkind == DVQLS_B_AMPLITUDES;
    ctx->tile_bits = n == 11 ? 11 : 12;
    if (ctx->tile_bits == 11)
      ctx->kc.fn = hh ? (const void*)&stream::stream_hadamard_kernel<11, true>
                      : (const void*)&stream::stream_hadamard_kernel<11, false>;
    else
      ctx->kc.fn = hh ? (const void*)&stream::stream_hadamard_kernel<12, true>
                      : (const void*)&stream::stream_hadamard_kernel<12, false>;
    ctx->kc.warps = (1 << ctx->tile_bits) / 16 / 32;
    ctx->kc.gpw = 1;
    ctx->kc.groups = 1;
    ctx->kc.smem = sizeof(double2) * (size_t(1) << ctx->tile_bits);
    // uniform b: the real-plane kernel (half the registers per thread, 3 CTAs/SM instead of 2);
    // DVQLS_PLANE=0 selects the complex kernel (A/B comparison knob)
    const char* pe = getenv("DVQLS_PLANE");
    if (!hh && !(pe && atoi(pe) == 0) && ctx->mode == DVQLS_MODE_CIRCUITS) {
      ctx->pstream = true;
      ctx->kc.fn = ctx->tile_bits == 11 ? (const void*)&streamp::stream_plane_kernel<11>
                                        : (const void*)&streamp::stream_plane_kernel<12>;
      ctx->kc.smem = ctx->tile_bits == 11 ? streamp::tile_smem<11>() : streamp::tile_smem<12>();
      // n >= 16 (scratch no longer L2-resident): TMA bulk-copy staging of the last-pass and
      // large-run mid-pass tiles (measured +1-3 % at n = 16..20, -5 % at n = 14 where the scratch
      // stays in L2; DVQLS_STAGE=0 keeps direct register loads + L2 prefetch, =1 forces it from n = 13)
      const char* se = getenv("DVQLS_STAGE");
      const int stage_from = se && atoi(se) == 1 ? 13 : 16;
      if (n >= stage_from && ctx->tile_bits == 12 && !(se && atoi(se) == 0)) {
        ctx->kc.fn = (const void*)&streamp::stream_plane_kernel<12, true>;
        ctx->kc.smem = streamp::staged_smem<12>();
      }
      // n = 11, 12 (one tile): the 2-exchange kernel with 64 doubles per thread (DVQLS_ONCHIP=0:
      // keep the 4-exchange tile kernel, A/B knob)
      const char* oe = getenv("DVQLS_ONCHIP");
      if (n <= 12 && !(oe && atoi(oe) == 0)) {
        ctx->pstream = false;
        ctx->onchip = true;
        ctx->kc.fn = n == 11 ? (const void*)&onchip::onchip_plane_kernel<11>
                             : (const void*)&onchip::onchip_plane_kernel<12>;
        ctx->kc.warps = onchip::WARPS;
        ctx->kc.groups = n == 11 ? onchip::Sh<11>::NG : onchip::Sh<12>::NG;
        ctx->kc.smem = n == 11 ? onchip::smem_bytes<11>() : onchip::smem_bytes<12>();
      }
    }
  }
  if (cudaFuncSetAttribute(ctx->kc.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ctx->kc.smem)) !=
      cudaSuccess) {
    fail(ctx, DVQLS_E_CUDA, "cannot reserve %zu B of shared memory", ctx->kc.smem);
    return bail(DVQLS_E_CUDA);
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ctx->kc.fn, ctx->kc.warps * 32, ctx->kc.smem);
  if (occ < 1) {
    fail(ctx, DVQLS_E_CUDA, "hadamard kernel cannot be resident (smem %zu B)", ctx->kc.smem);
    return bail(DVQLS_E_CUDA);
  }

  ctx->C = 2 * int64_t(n + 1) * L * L;
  dvqls_shard_range(ctx->C, ctx->rank, ctx->world, &ctx->c0, &ctx->c1);
  if (ctx->world == 1 && getenv("DVQLS_SLICE")) {
    // measurement knob (weak-scaling reference, SURVEY §8(d) cfg 4): evaluate only rank r's block
    // of a W-way split on this one GPU ("r/W"); costs then cover that block only
    int r = 0, W = 1;
    if (sscanf(getenv("DVQLS_SLICE"), "%d/%d", &r, &W) == 2 && W >= 1 && r >= 0 && r < W)
      dvqls_shard_range(ctx->C, r, W, &ctx->c0, &ctx->c1);
  }
  ctx->chunk = (ctx->C + ctx->world - 1) / ctx->world;
  if (ctx->c1 - ctx->c0 > int64_t(INT32_MAX)) {  // the kernels index a rank's circuits with 32-bit ints
    fail(ctx, DVQLS_E_UNSUPPORTED, "%lld circuits on one rank (more than 2^31 - 1): use more ranks",
         (long long)(ctx->c1 - ctx->c0));
    return bail(DVQLS_E_UNSUPPORTED);
  }
  const int64_t Cloc = ctx->c1 - ctx->c0;
  const bool flat_grid = !ctx->tile_path || ctx->onchip;  // one 1-D grid over the K x C work
  const int64_t groups_per_cta = flat_grid ? int64_t(ctx->kc.groups) : 1;
  int64_t want = int64_t(prop.multiProcessorCount) * occ;
  if (ctx->tile_path && n > ctx->tile_bits) {  // each CTA owns a 2^n-amplitude global scratch
    const int64_t cap = int64_t(kScratchBudget / ((ctx->pstream ? sizeof(double) : sizeof(double2)) * size_t(ctx->N)));
    want = std::max<int64_t>(1, std::min(want, cap));
  }
  if (ctx->tile_path) {
    const char* e = getenv("DVQLS_STREAM_GRID");  // tuning knob: CTAs of the n >= 11 path
    if (e && atoi(e) > 0) want = std::min<int64_t>(want, atoi(e));
  }
  const int64_t need = (Cloc + groups_per_cta - 1) / groups_per_cta;
  ctx->grid = int(std::max<int64_t>(1, std::min(want, need)));
  ctx->grid_cap = int(std::max<int64_t>(1, want));
  ctx->NG = std::max<int64_t>(int64_t(ctx->grid) * groups_per_cta, flat_grid ? ctx->grid_cap : 0);
  // Team mode is opt-in (DVQLS_TEAM=1): measured on B200 it cuts DRAM reads ~10x but the team
  // barriers cost as much as they save (cfg5 n=16: 210 vs 217 ms, n=18: 1218 vs 1123 ms, K=2).
  if (ctx->tile_path && n >= 15 && ctx->mode == DVQLS_MODE_CIRCUITS && getenv("DVQLS_TEAM") &&
      atoi(getenv("DVQLS_TEAM")) == 1) {
    // team mode: T = smallest power of two with (G / T) branches of 2^n x 16 B in <= 80 MB (L2)
    const void* tf = (const void*)&stream::stream_team_kernel<12>;
    if (cudaFuncSetAttribute(tf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(sizeof(double2) * stream::TS<12>::TN)) != cudaSuccess) {
      fail(ctx, DVQLS_E_CUDA, "team kernel smem");
      return bail(DVQLS_E_CUDA);
    }
    int tocc = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, tf, stream::TS<12>::THREADS,
                                                  sizeof(double2) * stream::TS<12>::TN);
    const int64_t G = int64_t(prop.multiProcessorCount) * std::max(1, tocc);
    const char* mb = getenv("DVQLS_TEAM_L2_MB");  // tuning knob: L2 budget of the in-flight branches
    const double budget = double(size_t(mb && atoi(mb) > 0 ? atoi(mb) : 80) << 20);
    const double ratio = double(G) * double(ctx->N) * 16.0 / budget;
    int64_t T = 1;
    while (T < ratio && T * 2 <= G) T *= 2;
    T = std::min<int64_t>(T, int64_t(ctx->N >> 12));  // at most one tile per member and pass
    if (T >= 2) {
      ctx->pstream = false;  // team mode runs the complex kernel
      ctx->team = int(T);
      ctx->nteams = int(G / T);
      ctx->grid = ctx->nteams * ctx->team;
      ctx->NG = std::max<int64_t>(ctx->NG, ctx->nteams);
    }
  }

  // ---- NEXT-2: symbolic task observables, dedup, folded weights (pauli.cuh) ---------------
  std::vector<pauli::Obs> obs;
  std::vector<double2> wE, wP;
  std::vector<uint32_t> task;
  if (ctx->mode == DVQLS_MODE_PAULI) {
    const int64_t T = ctx->C / 2;
    if (T > (int64_t(1) << 30)) {
      fail(ctx, DVQLS_E_UNSUPPORTED, "too many tasks for the Pauli fast path");
      return bail(DVQLS_E_UNSUPPORTED);
    }
    std::unordered_map<uint64_t, uint32_t> index;
    task.resize(size_t(T));
    for (int64_t t = 0; t < T; ++t) {
      const int s_ = int(t % (n + 1));
      const int64_t lk = t / (n + 1);
      const int k = int(lk % L), l = int(lk / L);
      const PauliOp B = task_observable(n, tab[l], tab[k], s_);
      const uint64_t key = (uint64_t(B.m) << 32) | B.z;
      auto it = index.find(key);
      uint32_t d;
      if (it == index.end()) {
        d = uint32_t(obs.size());
        index.emplace(key, d);
        obs.push_back(pauli::Obs{B.m, B.z});
        wE.push_back(make_double2(0.0, 0.0));
        wP.push_back(make_double2(0.0, 0.0));
      } else {
        d = it->second;
      }
      task[size_t(t)] = (d << 2) | uint32_t(B.q);
      // weight c_l^* c_k i^q (E = sum w <x|B|x> = sum w i^q e)
      const std::complex<double> w = std::conj(std::complex<double>(coef[l].x, coef[l].y)) *
                                     std::complex<double>(coef[k].x, coef[k].y) *
                                     std::pow(std::complex<double>(0.0, 1.0), B.q);
      double2& acc = s_ == 0 ? wP[d] : wE[d];
      acc.x += w.real();
      acc.y += w.imag();
    }
    ctx->D = int64_t(obs.size());
    dvqls_shard_range(ctx->D, ctx->rank, ctx->world, &ctx->d0, &ctx->d1);
    ctx->pauli_smem = ctx->N <= 8192 ? sizeof(double2) * size_t(ctx->N) : 0;
    if (cudaFuncSetAttribute((const void*)&pauli::pauli_expect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(ctx->pauli_smem)) != cudaSuccess) {
      fail(ctx, DVQLS_E_CUDA, "pauli kernel smem");
      return bail(DVQLS_E_CUDA);
    }
    int pocc = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pocc, (const void*)&pauli::pauli_expect_kernel,
                                                  pauli::WARPS * 32, ctx->pauli_smem);
    const int64_t pw = int64_t(prop.multiProcessorCount) * std::max(1, pocc);
    const int64_t pneed = (ctx->D + pauli::WARPS - 1) / pauli::WARPS;  // terms launches cover all D
    ctx->pgrid = int(std::max<int64_t>(1, std::min(pw, pneed)));
    ctx->NG = std::max<int64_t>(ctx->NG, ctx->pgrid);
  }

  {
    const char* e = getenv("DVQLS_PREFIX_RB");  // tuning knob: register-phase prefix for n <= 10
    ctx->prefix_rb = e ? std::min(std::max(1, std::min(3, atoi(e))), n) : (n <= 10 ? 0 : std::min(3, n));
  }
  {  // PDL behind the register prefix (n <= 12, 1-D Hadamard grid); off while the per-kernel
     // timing events sit between the two launches.  DVQLS_PDL=0 disables it (A/B knob).
    const char* e = getenv("DVQLS_PDL");
    ctx->pdl = n <= 12 && !ctx->timing && !(e && e[0] == '0');
  }
  if (n > 12) {
    ctx->prefix_rb = -1;  // global-memory multi-pass prefix (tile.cuh)
    ctx->prefix_fn = nullptr;
    if (cudaFuncSetAttribute((const void*)&tile::prefix_gate_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(sizeof(double2) * tile::TN)) != cudaSuccess) {
      fail(ctx, DVQLS_E_CUDA, "prefix_gate_pass smem");
      return bail(DVQLS_E_CUDA);
    }
  } else if (ctx->prefix_rb == 0 && n >= 7) {  // 4 amplitudes per thread, shuffles + 2 transposes/layer
    static const void* quads[11] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                    (const void*)&prefix_quad_kernel<7>, (const void*)&prefix_quad_kernel<8>,
                                    (const void*)&prefix_quad_kernel<9>, (const void*)&prefix_quad_kernel<10>};
    ctx->prefix_fn = quads[n];
    ctx->prefix_threads = std::max(32, ctx->N / 4);
    ctx->prefix_smem = sizeof(double2) * (2 * size_t(ctx->N) + 2 * size_t(n) * layers) + sizeof(int) * ctx->N;
  } else if (ctx->prefix_rb == 0) {  // one amplitude per thread, shuffles + 2 transposes per layer
    static const void* lanes[11] = {nullptr,
                                    (const void*)&prefix_lanes_kernel<1>, (const void*)&prefix_lanes_kernel<2>,
                                    (const void*)&prefix_lanes_kernel<3>, (const void*)&prefix_lanes_kernel<4>,
                                    (const void*)&prefix_lanes_kernel<5>, (const void*)&prefix_lanes_kernel<6>,
                                    (const void*)&prefix_lanes_kernel<7>, (const void*)&prefix_lanes_kernel<8>,
                                    (const void*)&prefix_lanes_kernel<9>, (const void*)&prefix_lanes_kernel<10>};
    ctx->prefix_fn = lanes[n];
    ctx->prefix_threads = std::max(32, ctx->N);
    ctx->prefix_smem = sizeof(double2) * (size_t(ctx->N) + 4 * size_t(n) * layers) + sizeof(int) * ctx->N;
  } else {
    ctx->prefix_fn = ctx->prefix_rb == 3 ? (const void*)&prefix_kernel<3>
                     : ctx->prefix_rb == 2 ? (const void*)&prefix_kernel<2> : (const void*)&prefix_kernel<1>;
    const int T = ctx->N >> ctx->prefix_rb;
    ctx->prefix_threads = std::min(512, std::max(32, (T + 31) / 32 * 32));
    ctx->prefix_smem = sizeof(double2) * (2 * size_t(ctx->N) + 2 * size_t(n) * layers) + sizeof(int) * ctx->N;
  }
  if (ctx->prefix_fn && cudaFuncSetAttribute(ctx->prefix_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(ctx->prefix_smem)) != cudaSuccess) {
    fail(ctx, DVQLS_E_CUDA, "prefix kernel smem %zu B", ctx->prefix_smem);
    return bail(DVQLS_E_CUDA);
  }
  // The prefix and the Hadamard-test kernel run back to back every call: give both the maximum
  // SMEM carveout so the SMs do not repartition L1/SMEM between them (DVQLS_CARVEOUT=0: driver
  // default, A/B knob)
  if (!(getenv("DVQLS_CARVEOUT") && atoi(getenv("DVQLS_CARVEOUT")) == 0)) {
    if (ctx->prefix_fn)
      cudaFuncSetAttribute(ctx->prefix_fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                           int(cudaSharedmemCarveoutMaxShared));
    cudaFuncSetAttribute(ctx->kc.fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
    cudaGetLastError();
  }

  // ---- device buffers: cudaMalloc'd once here, or carved from the caller's workspace -----
  const int KB = ctx->max_batch;
  std::vector<std::pair<void**, size_t>> req;
  auto buffer = [&](bool cond, void* p, size_t bytes) {
    if (cond) req.emplace_back(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 16));
  };
  // Pauli mode: a plan has no strings, so it sizes for one observable per task (the bound)
  const size_t nobs = plan_bytes ? size_t(ctx->C / 2) : obs.size();
  const size_t ntask = plan_bytes ? size_t(ctx->C / 2) : task.size();
  buffer(true, &ctx->d_tab, sizeof(PauliTerm) * L);
  buffer(true, &ctx->d_coef, sizeof(double2) * L);
  buffer(true, &ctx->d_hv, sizeof(double2) * ctx->N);
  buffer(true, &ctx->d_theta, sizeof(double) * KB * ctx->P);
  buffer(true, &ctx->d_x, sizeof(double2) * KB * ctx->N);
  buffer(true, &ctx->d_terms, sizeof(double) * KB * ctx->chunk);
  buffer(true, &ctx->d_partials, sizeof(double) * KB * ctx->NG * 4);
  buffer(true, &ctx->d_ep, sizeof(double) * KB * 4);
  buffer(true, &ctx->d_out, sizeof(double) * KB * 5);
  buffer(ctx->world > 1, &ctx->d_gather, sizeof(double) * ctx->world * ctx->chunk);
  buffer(true, &ctx->d_counter, sizeof(unsigned) * KB);
  buffer(true, &ctx->d_gcounter, sizeof(unsigned) * KB);
  buffer(true, &ctx->d_beta, sizeof(double) * 2 * KB * size_t(L));
  buffer(true, &ctx->d_out6, sizeof(double) * 6 * KB);
  buffer(ctx->bkind == DVQLS_B_AMPLITUDES, &ctx->d_b, sizeof(double2) * ctx->N);
  buffer(n > 12 && ctx->mode == DVQLS_MODE_CIRCUITS, &ctx->d_scratch,
       (ctx->pstream ? sizeof(double) : sizeof(double2)) * size_t(ctx->team ? ctx->nteams : ctx->grid) * ctx->N);
  buffer(ctx->pstream, &ctx->d_xp, sizeof(double2) * KB * ctx->N);
  // onchip: every theta's 4N-double x block aligned to its size (XOR addressing); slack for the round-up
  buffer(ctx->onchip, &ctx->d_xq, sizeof(double) * 4 * (size_t(KB) + 1) * ctx->N);
  buffer(ctx->team, &ctx->d_team_acc, sizeof(double) * 2 * size_t(ctx->nteams) * ctx->team);
  buffer(ctx->team, &ctx->d_team_ctr, sizeof(unsigned) * (size_t(ctx->nteams) + 1));
  const bool pm = ctx->mode == DVQLS_MODE_PAULI;
  buffer(pm, &ctx->d_obs, sizeof(pauli::Obs) * nobs);
  buffer(pm, &ctx->d_wE, sizeof(double2) * nobs);
  buffer(pm, &ctx->d_wP, sizeof(double2) * nobs);
  buffer(pm, &ctx->d_task, sizeof(uint32_t) * ntask);
  buffer(pm, &ctx->d_e, sizeof(double2) * nobs);
  buffer(n > 12, &ctx->d_x2, sizeof(double2) * size_t(ctx->N));
  buffer(n > 12, &ctx->d_gates, sizeof(double2) * 2 * size_t(n) * layers);
  size_t total = 0;
  for (auto& r : req) total += (r.second + 255) & ~size_t(255);
  if (plan_bytes) {
    *plan_bytes = total;
    release(ctx);
    delete ctx;
    return DVQLS_OK;
  }
  if (opts && opts->workspace_dev) {
    if ((reinterpret_cast<uintptr_t>(opts->workspace_dev) & 255u) || opts->workspace_bytes < total) {
      fail(ctx, DVQLS_E_ARG, "workspace: %zu bytes at %p, need %zu bytes 256-byte aligned", opts->workspace_bytes,
           opts->workspace_dev, total);
      return bail(DVQLS_E_ARG);
    }
    char* base = static_cast<char*>(opts->workspace_dev);
    for (auto& r : req) {
      *r.first = base;
      ctx->carved.push_back(r.first);
      base += (r.second + 255) & ~size_t(255);
    }
  } else {
    for (auto& r : req)
      if (cudaMalloc(r.first, r.second) != cudaSuccess) {
        fail(ctx, DVQLS_E_CUDA, "cudaMalloc failed");
        return bail(DVQLS_E_CUDA);
      }
  }
  ctx->h_stage_bytes = sizeof(double) * std::max<size_t>(size_t(KB) * (ctx->P + 5), 64);
  if (cudaMallocHost((void**)&ctx->h_stage, ctx->h_stage_bytes) != cudaSuccess) {
    fail(ctx, DVQLS_E_CUDA, "cudaMallocHost failed");
    return bail(DVQLS_E_CUDA);
  }
  if (cudaMemset(ctx->d_counter, 0, sizeof(unsigned) * KB) || cudaMemset(ctx->d_gcounter, 0, sizeof(unsigned) * KB) ||
      (ctx->team && cudaMemset(ctx->d_team_ctr, 0, sizeof(unsigned) * (size_t(ctx->nteams) + 1))) ||
      (ctx->bkind == DVQLS_B_AMPLITUDES &&
       cudaMemcpy(ctx->d_b, bprep->amps, sizeof(double2) * ctx->N, cudaMemcpyHostToDevice)) ||
      cudaMemcpy(ctx->d_tab, tab.data(), sizeof(PauliTerm) * L, cudaMemcpyHostToDevice) ||
      cudaMemcpy(ctx->d_coef, coef.data(), sizeof(double2) * L, cudaMemcpyHostToDevice) ||
      (!hv.empty() && cudaMemcpy(ctx->d_hv, hv.data(), sizeof(double2) * ctx->N, cudaMemcpyHostToDevice)) ||
      (!obs.empty() &&
       (cudaMemcpy(ctx->d_obs, obs.data(), sizeof(pauli::Obs) * obs.size(), cudaMemcpyHostToDevice) ||
        cudaMemcpy(ctx->d_wE, wE.data(), sizeof(double2) * obs.size(), cudaMemcpyHostToDevice) ||
        cudaMemcpy(ctx->d_wP, wP.data(), sizeof(double2) * obs.size(), cudaMemcpyHostToDevice) ||
        cudaMemcpy(ctx->d_task, task.data(), sizeof(uint32_t) * task.size(), cudaMemcpyHostToDevice)))) {
    fail(ctx, DVQLS_E_CUDA, "table upload failed");
    return bail(DVQLS_E_CUDA);
  }
  if (ctx->timing)
    for (auto& e : ctx->ev)
      if (cudaEventCreate(&e) != cudaSuccess) {
        fail(ctx, DVQLS_E_CUDA, "cudaEventCreate failed");
        return bail(DVQLS_E_CUDA);
      }

  // ---- NCCL communicator (a10) -------------------------------------------------
  if (ctx->world > 1) {
    if (!nccl().ok) {
      fail(ctx, DVQLS_E_NCCL, "libnccl.so.2 not loadable");
      return bail(DVQLS_E_NCCL);
    }
    ncclUniqueId id;
    std::memcpy(&id, opts->nccl_unique_id, sizeof id);
    ncclResult_t r = nccl().CommInitRank(&ctx->comm, ctx->world, id, ctx->rank);
    if (r != ncclSuccess) {
      fail(ctx, DVQLS_E_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
      ctx->comm = nullptr;
      return bail(DVQLS_E_NCCL);
    }
  }
  if (ctx->world > 1) {
    const char* e = getenv("DVQLS_ALLREDUCE");  // "nccl" forces the NCCL baseline
    if (!(e && std::string(e) == "nccl")) {
      int rc = setup_p2p(ctx);
      if (rc) return bail(rc);
    }
  }
  *out = ctx;
  return DVQLS_OK;
}
}  // namespace

extern "C" {

int dvqls_create(dvqls_ctx** out, int n, int layers, int L, const char* paulis, const double* coeffs,
                 const dvqls_bprep* bprep, const dvqls_opts* opts) {
  return create_impl(out, n, layers, L, paulis, coeffs, bprep, opts, nullptr);
}

size_t dvqls_workspace_size(int n, int layers, int L, const dvqls_opts* opts) {
  if (n < 1 || n > 24 || layers < 1 || L < 1 || double(L) > std::pow(4.0, n)) return 0;
  // L distinct placeholder strings (base-4 digits of l); only sizes are planned
  std::string ps(size_t(L) * n, 'I');
  for (int l = 0; l < L; ++l) {
    int64_t v = l;
    for (int q = n - 1; q >= 0 && v; --q, v >>= 2) ps[size_t(l) * n + q] = "IXYZ"[v & 3];
  }
  std::vector<double> co(2 * size_t(L), 0.0);
  co[0] = 1.0;
  size_t best = 0;
  const int mode = opts ? opts->mode : DVQLS_MODE_CIRCUITS;
  for (int kind : {DVQLS_B_UNIFORM, DVQLS_B_AMPLITUDES}) {  // the size for either U_b
    if (kind == DVQLS_B_AMPLITUDES && (n > 12 || mode != DVQLS_MODE_CIRCUITS)) continue;
    std::vector<double> amps;
    dvqls_bprep bp{kind, nullptr};
    if (kind == DVQLS_B_AMPLITUDES) {
      amps.assign(2 * (size_t(1) << n), 0.0);
      amps[0] = 1.0;
      bp.amps = amps.data();
    }
    size_t b = 0;
    dvqls_ctx* dummy = nullptr;
    if (create_impl(&dummy, n, layers, L, ps.data(), co.data(), &bp, opts, &b) != DVQLS_OK) return 0;
    best = std::max(best, b);
  }
  return best;
}

void dvqls_destroy(dvqls_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  release(ctx);
  delete ctx;
}

int dvqls_cost_dev(dvqls_ctx* ctx, int K, const double* thetas_dev, double* out_dev) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (K < 1 || K > ctx->max_batch) return fail(ctx, DVQLS_E_ARG, "K=%d outside [1, max_batch=%d]", K, ctx->max_batch);
  if (!thetas_dev || !out_dev) return fail(ctx, DVQLS_E_ARG, "NULL device pointer");
  return launch_eval(ctx, K, thetas_dev, true, out_dev);
}

int dvqls_terms_local_dev(dvqls_ctx* ctx, const double* theta_dev, double* out_dev) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (!theta_dev || !out_dev) return fail(ctx, DVQLS_E_ARG, "NULL device pointer");
  int rc = launch_eval(ctx, 1, theta_dev, false, nullptr);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out_dev, ctx->d_terms, sizeof(double) * (ctx->c1 - ctx->c0), cudaMemcpyDeviceToDevice,
                     ctx->stream));
  return DVQLS_OK;
}

int dvqls_costs_dev(dvqls_ctx* ctx, int K, const double* thetas_dev, double* out6_dev, double* beta_dev) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (K < 1 || K > ctx->max_batch) return fail(ctx, DVQLS_E_ARG, "K=%d outside [1, max_batch=%d]", K, ctx->max_batch);
  if (!thetas_dev || !out6_dev) return fail(ctx, DVQLS_E_ARG, "NULL device pointer");
  int rc = launch_eval(ctx, K, thetas_dev, true, ctx->d_out);
  if (rc) return rc;
  glob::overlap_kernel<<<dim3(ctx->L, K), glob::THREADS, 0, ctx->stream>>>(
      ctx->d_x, ctx->n, ctx->d_tab, ctx->d_coef, ctx->d_b, ctx->L, ctx->d_out, beta_dev ? beta_dev : ctx->d_beta,
      out6_dev, ctx->d_gcounter);
  CK(cudaGetLastError());
  return DVQLS_OK;
}

int dvqls_global_cost(dvqls_ctx* ctx, const double* theta, double* out6, double* out_beta) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (!theta || !out6) return fail(ctx, DVQLS_E_ARG, "NULL host pointer");
  std::memcpy(ctx->h_stage, theta, sizeof(double) * ctx->P);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, sizeof(double) * ctx->P, cudaMemcpyHostToDevice, ctx->stream));
  int rc = dvqls_costs_dev(ctx, 1, ctx->d_theta, ctx->d_out6, ctx->d_beta);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out6, ctx->d_out6, sizeof(double) * 6, cudaMemcpyDeviceToHost, ctx->stream));
  if (out_beta)
    CK(cudaMemcpyAsync(out_beta, ctx->d_beta, sizeof(double) * 2 * ctx->L, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (!(out6[3] > 1e-12)) return fail(ctx, DVQLS_E_DEGENERATE, "Re Psi <= 1e-12 (singular A on the ansatz state)");
  return DVQLS_OK;
}

int dvqls_cost_batch(dvqls_ctx* ctx, int K, const double* thetas, double* out_costs, double* out_E_Psi) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (K < 1 || K > ctx->max_batch) return fail(ctx, DVQLS_E_ARG, "K=%d outside [1, max_batch=%d]", K, ctx->max_batch);
  if (!thetas || !out_costs) return fail(ctx, DVQLS_E_ARG, "NULL host pointer");
  const size_t tb = sizeof(double) * size_t(K) * ctx->P;
  std::memcpy(ctx->h_stage, thetas, tb);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, tb, cudaMemcpyHostToDevice, ctx->stream));
  int rc = launch_eval(ctx, K, ctx->d_theta, true, ctx->d_out);
  if (rc) return rc;
  double* h_out = ctx->h_stage + size_t(K) * ctx->P;
  CK(cudaMemcpyAsync(h_out, ctx->d_out, sizeof(double) * 5 * K, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  bool degenerate = false;
  for (int k = 0; k < K; ++k) {
    out_costs[k] = h_out[5 * k];
    if (out_E_Psi)
      for (int j = 0; j < 4; ++j) out_E_Psi[4 * k + j] = h_out[5 * k + 1 + j];
    if (!(h_out[5 * k + 3] > 1e-12)) degenerate = true;
  }
  if (degenerate) return fail(ctx, DVQLS_E_DEGENERATE, "Re Psi <= 1e-12 (singular A on the ansatz state)");
  return DVQLS_OK;
}

int dvqls_cost(dvqls_ctx* ctx, const double* theta, double* out_cost, double* out_E_Psi) {
  return dvqls_cost_batch(ctx, 1, theta, out_cost, out_E_Psi);
}

int dvqls_terms(dvqls_ctx* ctx, const double* theta, double* out) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (!theta || !out) return fail(ctx, DVQLS_E_ARG, "NULL host pointer");
  std::memcpy(ctx->h_stage, theta, sizeof(double) * ctx->P);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, sizeof(double) * ctx->P, cudaMemcpyHostToDevice, ctx->stream));
  int rc = launch_eval(ctx, 1, ctx->d_theta, false, nullptr);
  if (rc) return rc;
  if (ctx->world == 1) {
    CK(cudaMemcpyAsync(out, ctx->d_terms, sizeof(double) * ctx->C, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    CKN(nccl().AllGather(ctx->d_terms, ctx->d_gather, size_t(ctx->chunk), ncclDouble, ctx->comm, ctx->stream));
    for (int r = 0; r < ctx->world; ++r) {
      const int64_t a = ctx->C * r / ctx->world, b = ctx->C * (r + 1) / ctx->world;
      CK(cudaMemcpyAsync(out + a, ctx->d_gather + size_t(r) * ctx->chunk, sizeof(double) * (b - a),
                         cudaMemcpyDeviceToHost, ctx->stream));
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DVQLS_OK;
}

int dvqls_state(dvqls_ctx* ctx, const double* theta, double* out_state) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (!theta || !out_state) return fail(ctx, DVQLS_E_ARG, "NULL host pointer");
  std::memcpy(ctx->h_stage, theta, sizeof(double) * ctx->P);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, sizeof(double) * ctx->P, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->prefix_rb < 0) {
    int rc = launch_prefix_global(ctx, 1, ctx->d_theta);
    if (rc) return rc;
  } else if (ctx->prefix_rb == 0) {
    void* args[] = {(void*)&ctx->layers, (void*)&ctx->entangler, (void*)&ctx->d_theta, (void*)&ctx->d_x};
    CK(cudaLaunchKernel(ctx->prefix_fn, dim3(1), dim3(ctx->prefix_threads), args, ctx->prefix_smem, ctx->stream));
  } else {
    void* args[] = {(void*)&ctx->n, (void*)&ctx->layers, (void*)&ctx->entangler, (void*)&ctx->d_theta,
                    (void*)&ctx->d_x};
    CK(cudaLaunchKernel(ctx->prefix_fn, dim3(1), dim3(ctx->prefix_threads), args, ctx->prefix_smem, ctx->stream));
  }
  CK(cudaMemcpyAsync(out_state, ctx->d_x, sizeof(double2) * ctx->N, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DVQLS_OK;
}

int dvqls_terms_subset(dvqls_ctx* ctx, const double* theta, const int64_t* idx, int64_t count, double* out) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (!theta || !out || (count > 0 && !idx) || count < 0) return fail(ctx, DVQLS_E_ARG, "bad subset arguments");
  for (int64_t i = 0; i < count; ++i)
    if (idx[i] < 0 || idx[i] >= ctx->C) return fail(ctx, DVQLS_E_ARG, "circuit index %lld out of range", (long long)idx[i]);
  if (count == 0) return DVQLS_OK;
  if (!ctx->tile_path || ctx->onchip || ctx->world > 1 || ctx->mode == DVQLS_MODE_PAULI) {  // all, pick
    std::vector<double> all(size_t(ctx->C));
    int rc = dvqls_terms(ctx, theta, all.data());
    if (rc) return rc;
    for (int64_t i = 0; i < count; ++i) out[i] = all[size_t(idx[i])];
    return DVQLS_OK;
  }
  if (count > ctx->sub_cap) {
    cudaFree(ctx->d_cidx); cudaFree(ctx->d_sub);
    ctx->d_cidx = nullptr; ctx->d_sub = nullptr; ctx->sub_cap = 0;
    CK(cudaMalloc((void**)&ctx->d_cidx, sizeof(int64_t) * count));
    CK(cudaMalloc((void**)&ctx->d_sub, sizeof(double) * count));
    ctx->sub_cap = count;
  }
  std::memcpy(ctx->h_stage, theta, sizeof(double) * ctx->P);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, sizeof(double) * ctx->P, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_cidx, idx, sizeof(int64_t) * count, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->prefix_rb < 0) {
    int rc = launch_prefix_global(ctx, 1, ctx->d_theta);
    if (rc) return rc;
  } else {
    void* args[] = {(void*)&ctx->n, (void*)&ctx->layers, (void*)&ctx->entangler, (void*)&ctx->d_theta,
                    (void*)&ctx->d_x};
    CK(cudaLaunchKernel(ctx->prefix_fn, dim3(1), dim3(ctx->prefix_threads), args, ctx->prefix_smem, ctx->stream));
  }
  const int grid = int(std::min<int64_t>(ctx->team ? ctx->nteams : ctx->grid, count));  // scratch slots
  int rc = launch_hadamard(ctx, 1, 0, count, ctx->d_cidx, ctx->d_sub, grid);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out, ctx->d_sub, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DVQLS_OK;
}

}  // extern "C"

// ---- NEXT-4: Pauli decomposition + pruning (decomp.cuh) ---------------------------------------
namespace {
struct DecompBufs {
  double2* A = nullptr;
  double2* B = nullptr;
  double2* C = nullptr;
  double* sq = nullptr;
  double* norm = nullptr;
  double* thr0 = nullptr;
  double* fro = nullptr;
  unsigned long long* count = nullptr;
  unsigned long long* outL = nullptr;
  uint64_t* idx = nullptr;
  double2* oc = nullptr;
  char* os = nullptr;
  cudaStream_t st = nullptr;
  ~DecompBufs() {
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(sq); cudaFree(norm); cudaFree(count); cudaFree(idx); cudaFree(oc); cudaFree(os);
    cudaFree(thr0); cudaFree(fro); cudaFree(outL);
    if (st) cudaStreamDestroy(st);
  }
};
thread_local std::string g_decomp_err;

int decomp_fail(int code, const char* msg) {
  g_decomp_err = msg;
  return code;
}

// NEXT-4 device pass over B (XOR diagonals of A as rows; n < 5: straight from A).
// MODE 0: all coefficients into C;  MODE 1: candidates + per-row |c|^2 (decomp.cuh).
template <int NB, int MODE>
int launch_rows_reg(DecompBufs& b, uint64_t cap) {
  const void* fn = (const void*)&decomp::fwht_rows_reg_kernel<NB, MODE>;
  const int smem = int(sizeof(double2) << NB);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
    return decomp_fail(DVQLS_E_CUDA, "fwht_rows_reg_kernel smem");
  decomp::fwht_rows_reg_kernel<NB, MODE><<<1u << NB, 1u << (NB - 4), smem, b.st>>>(b.B, b.C, b.sq, b.thr0, cap,
                                                                                  b.count, b.idx);
  return DVQLS_OK;
}
template <int MODE>
int launch_rows(DecompBufs& b, int n, uint64_t cap) {
  switch (n) {
    case 9: return launch_rows_reg<9, MODE>(b, cap);
    case 10: return launch_rows_reg<10, MODE>(b, cap);
    case 11: return launch_rows_reg<11, MODE>(b, cap);
    case 12: return launch_rows_reg<12, MODE>(b, cap);
    case 13: return launch_rows_reg<13, MODE>(b, cap);
    default: break;
  }
  const unsigned N = 1u << n;
  const int direct = n < 5 ? 1 : 0;
  if (cudaFuncSetAttribute((const void*)&decomp::fwht_rows_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(sizeof(double2) << n)))
    return decomp_fail(DVQLS_E_CUDA, "fwht_rows_kernel smem");
  decomp::fwht_rows_kernel<MODE><<<N, decomp::THREADS, sizeof(double2) * N, b.st>>>(
      direct ? b.A : b.B, n, b.C, b.sq, b.thr0, cap, b.count, b.idx, direct);
  return DVQLS_OK;
}

// A -> device, XOR-diagonal transposition (+ |A|^2 tile sums); write_c: every coefficient into C,
// else: Parseval candidate bound, one candidate pass, exact norm (decomp.cuh)
int decomp_transform(DecompBufs& b, int n, const double* A_host, int device, bool write_c, double eps = 0.0,
                     cudaEvent_t* ev0 = nullptr) {
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return decomp_fail(DVQLS_E_CUDA, "cudaSetDevice");
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10)
    return decomp_fail(DVQLS_E_CUDA, "libdvqls is built for sm_100a only");
  const size_t N = size_t(1) << n, NN = N * N;
  // transposition CTAs (persistent over the (N/32)^2 tiles; one |A|^2 partial each)
  const size_t nfro = n >= 5 ? std::min<size_t>((N >> 5) * (N >> 5), size_t(prop.multiProcessorCount) * 8) : 1;
  const uint64_t cap = decomp::SORT_MAX;
  if (cudaStreamCreateWithFlags(&b.st, cudaStreamNonBlocking) || cudaMalloc((void**)&b.A, sizeof(double2) * NN) ||
      cudaMalloc((void**)&b.C, sizeof(double2) * (write_c ? NN : size_t(cap))) ||
      cudaMalloc((void**)&b.sq, sizeof(double) * N) || cudaMalloc((void**)&b.norm, sizeof(double)) ||
      cudaMalloc((void**)&b.thr0, sizeof(double)) || cudaMalloc((void**)&b.fro, sizeof(double) * nfro) ||
      cudaMalloc((void**)&b.count, sizeof(unsigned long long)) ||
      cudaMalloc((void**)&b.outL, sizeof(unsigned long long)))
    return decomp_fail(DVQLS_E_CUDA, "cudaMalloc failed (decomposition)");
  if (!write_c && (cudaMalloc((void**)&b.idx, sizeof(uint64_t) * cap) ||
                   cudaMalloc((void**)&b.oc, sizeof(double2) * cap) || cudaMalloc((void**)&b.os, size_t(cap) * n)))
    return decomp_fail(DVQLS_E_CUDA, "cudaMalloc failed (pruning)");
  if (cudaMemcpyAsync(b.A, A_host, sizeof(double2) * NN, cudaMemcpyHostToDevice, b.st))
    return decomp_fail(DVQLS_E_CUDA, "copy of A failed");
  if (n >= 5 && cudaMalloc((void**)&b.B, sizeof(double2) * NN)) return decomp_fail(DVQLS_E_CUDA, "cudaMalloc B");
  if (ev0 && (cudaEventCreate(ev0) || cudaEventRecord(*ev0, b.st))) return decomp_fail(DVQLS_E_CUDA, "event");
  if (n >= 5)
    decomp::xor_transpose_kernel<<<unsigned(nfro), 256, 0, b.st>>>(b.A, n, b.B, b.fro);  // persistent
  else
    decomp::fro_small_kernel<<<1, 256, 0, b.st>>>(b.A, uint32_t(NN), b.fro);
  int rc;
  if (write_c) {
    rc = launch_rows<0>(b, n, 0);
  } else {
    decomp::prenorm_kernel<<<1, 256, 0, b.st>>>(b.fro, uint32_t(nfro), uint32_t(N), eps, b.thr0, b.count);
    rc = launch_rows<1>(b, n, cap);  // the exact norm is formed inside sort_emit_kernel
  }
  if (rc) return rc;
  if (cudaGetLastError()) return decomp_fail(DVQLS_E_CUDA, "decomposition kernel launch failed");
  return DVQLS_OK;
}
}  // namespace

extern "C" {

int dvqls_pauli_coefficients(int n, const double* A, double* out_coeffs, int device) {
  g_decomp_err.clear();
  if (n < 1 || n > 13 || !A || !out_coeffs) return decomp_fail(DVQLS_E_ARG, "n must be in [1, 13], non-NULL buffers");
  DecompBufs b;
  int rc = decomp_transform(b, n, A, device, true);
  if (rc) return rc;
  const size_t NN = (size_t(1) << n) * (size_t(1) << n);
  if (cudaMemcpyAsync(out_coeffs, b.C, sizeof(double2) * NN, cudaMemcpyDeviceToHost, b.st) ||
      cudaStreamSynchronize(b.st))
    return decomp_fail(DVQLS_E_CUDA, "decomposition failed");
  return DVQLS_OK;
}

int dvqls_decompose(int n, const double* A, double eps, int64_t max_terms, char* out_paulis, double* out_coeffs,
                    int64_t* out_L, double* out_norm, int device, float* out_ms) {
  g_decomp_err.clear();
  if (n < 1 || n > 13 || !A || !out_L || (max_terms > 0 && (!out_paulis || !out_coeffs)) || max_terms < 0 ||
      !(eps >= 0.0 && eps < 1.0))
    return decomp_fail(DVQLS_E_ARG, "n in [1, 13], 0 <= eps < 1, non-NULL outputs");
  DecompBufs b;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = decomp_transform(b, n, A, device, false, eps, out_ms ? &e0 : nullptr);
  if (rc) return rc;
  if (cudaFuncSetAttribute((const void*)&decomp::sort_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(decomp::SORT_SMEM)))
    return decomp_fail(DVQLS_E_CUDA, "sort kernel smem");
  decomp::sort_emit_kernel<<<1, decomp::THREADS, decomp::SORT_SMEM, b.st>>>(b.C, n, b.idx, b.count, b.sq, b.norm,
                                                                             eps, b.oc, b.os, b.outL);
  if (out_ms && (cudaEventCreate(&e1) || cudaEventRecord(e1, b.st)))
    return decomp_fail(DVQLS_E_CUDA, "event");
  unsigned long long cand = 0, L = 0;
  double norm = 0.0;
  if (cudaGetLastError() || cudaMemcpyAsync(&cand, b.count, sizeof cand, cudaMemcpyDeviceToHost, b.st) ||
      cudaMemcpyAsync(&L, b.outL, sizeof L, cudaMemcpyDeviceToHost, b.st) ||
      cudaMemcpyAsync(&norm, b.norm, sizeof norm, cudaMemcpyDeviceToHost, b.st) || cudaStreamSynchronize(b.st))
    return decomp_fail(DVQLS_E_CUDA, "pruning failed");
  if (out_norm) *out_norm = norm;
  if (cand > decomp::SORT_MAX) {
    *out_L = int64_t(cand);
    return decomp_fail(DVQLS_E_UNSUPPORTED, "more than 4096 terms survive the pruning");
  }
  *out_L = int64_t(L);
  if (int64_t(L) > max_terms) return decomp_fail(DVQLS_E_ARG, "max_terms too small (*out_L holds the count)");
  if (L > 0 && (cudaMemcpyAsync(out_coeffs, b.oc, sizeof(double2) * L, cudaMemcpyDeviceToHost, b.st) ||
                cudaMemcpyAsync(out_paulis, b.os, size_t(L) * n, cudaMemcpyDeviceToHost, b.st) ||
                cudaStreamSynchronize(b.st)))
    return decomp_fail(DVQLS_E_CUDA, "sort/emit failed");
  if (out_ms) {  // device time from after the H2D copy of A to the end of sort/emit
    cudaEventElapsedTime(out_ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return DVQLS_OK;
}

const char* dvqls_decompose_error(void) { return g_decomp_err.c_str(); }

const char* dvqls_last_error(const dvqls_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

int64_t dvqls_num_circuits(const dvqls_ctx* ctx) { return ctx ? ctx->C : -1; }

int dvqls_local_range(const dvqls_ctx* ctx, int64_t* c0, int64_t* c1) {
  if (!ctx || !c0 || !c1) return DVQLS_E_ARG;
  *c0 = ctx->c0;
  *c1 = ctx->c1;
  return DVQLS_OK;
}

void* dvqls_stream(const dvqls_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int dvqls_launch_grid(const dvqls_ctx* ctx) {
  if (!ctx) return DVQLS_E_ARG;
  return ctx->mode == DVQLS_MODE_PAULI ? ctx->pgrid : ctx->grid;
}

int64_t dvqls_num_observables(const dvqls_ctx* ctx) {
  if (!ctx) return DVQLS_E_ARG;
  return ctx->mode == DVQLS_MODE_PAULI ? ctx->D : 0;
}

int dvqls_task_observable(int n, const char* pauli_l, const char* pauli_k, int s, uint32_t* x_mask,
                          uint32_t* z_mask, int* phase) {
  if (n < 1 || n > 24 || !pauli_l || !pauli_k || s < 0 || s > n || !x_mask || !z_mask || !phase) return DVQLS_E_ARG;
  PauliTerm T[2] = {{0, 0, 0, 0u}, {0, 0, 0, 0u}};
  const char* str[2] = {pauli_l, pauli_k};
  for (int a = 0; a < 2; ++a)
    for (int q = 0; q < n; ++q) {
      const uint32_t bit = 1u << (n - 1 - q);
      switch (str[a][q]) {
        case 'I': break;
        case 'X': T[a].xm |= bit; break;
        case 'Y': T[a].xm |= bit; T[a].zm |= bit; T[a].ny += 1; break;
        case 'Z': T[a].zm |= bit; break;
        default: return DVQLS_E_PAULI;
      }
    }
  const PauliOp B = task_observable(n, T[0], T[1], s);
  *x_mask = B.m;
  *z_mask = B.z;
  *phase = B.q;
  return DVQLS_OK;
}

int dvqls_launches_per_call(const dvqls_ctx* ctx) {
  if (!ctx) return DVQLS_E_ARG;
  // prefix (1, or 2 + layers*(groups+1) for the global n > 12 prefix), hadamard (+ fused
  // reduction) [, finalize]  (+ NCCL's own allreduce kernel when world > 1)
  const int pre = ctx->prefix_rb < 0 ? 2 + ctx->layers * ((ctx->n <= 21 ? 2 : 3) + 1) : 1;
  return pre + 1 + ((ctx->pstream || ctx->onchip) ? 1 : 0) + ((ctx->world == 1 || ctx->p2p) ? 0 : 1);
}

int dvqls_last_timings(const dvqls_ctx* c, float* ms) {
  dvqls_ctx* ctx = const_cast<dvqls_ctx*>(c);
  if (!ctx || !ms || !ctx->timing || !ctx->timed_once) return DVQLS_E_ARG;
  CK(cudaEventSynchronize(ctx->ev[3]));
  CK(cudaEventElapsedTime(&ms[0], ctx->ev[0], ctx->ev[1]));
  CK(cudaEventElapsedTime(&ms[1], ctx->ev[1], ctx->ev[2]));
  CK(cudaEventElapsedTime(&ms[2], ctx->ev[2], ctx->ev[3]));
  CK(cudaEventElapsedTime(&ms[3], ctx->ev[0], ctx->ev[3]));
  return DVQLS_OK;
}

int dvqls_nccl_unique_id(void* out128) {
  if (!out128) return DVQLS_E_ARG;
  if (!nccl().ok) return DVQLS_E_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return DVQLS_E_NCCL;
  std::memcpy(out128, &id, sizeof id);
  return DVQLS_OK;
}

int dvqls_shard_range(int64_t n_circuits, int rank, int world, int64_t* c0, int64_t* c1) {
  if (n_circuits < 0 || world < 1 || rank < 0 || rank >= world || !c0 || !c1) return DVQLS_E_ARG;
  *c0 = n_circuits * rank / world;
  *c1 = n_circuits * (rank + 1) / world;
  return DVQLS_OK;
}

const char* dvqls_build_info(void) {
  return "libdvqls sm_100a; register-resident Hadamard-test path n=1..10, SMEM-tile path n=11..12, "
         "global streaming path n=13..24; fp64 (complex128); NCCL via dlopen";
}

}  // extern "C"
