// dvqls_api.cu - the C ABI of libdvqls.so (declared and documented in include/dvqls.h).
//
// Host side of the hot path: context build, launch of the sm_100a kernels
// (k_*.cu through launch.h), the cross-rank reduction (a10, "Global Reduction", Alg. 1 Step
// 4c P:461-463) fused into the kernels over NVLink peer memory or over a library-owned NCCL
// communicator, CUDA-graph capture of the per-call launch sequence, and marshalling of host
// buffers.  No arithmetic of the method runs here: the host validates inputs, precomputes the
// Householder vector of U_b, multiplies Pauli strings symbolically for the flagged NEXT-2 path
// and moves bytes.  Compiled as plain host C++ by nvcc (no device code in this file).

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dvqls.h"
#include "launch.h"
#include "nccl_dl.h"

using namespace dvqls;

namespace {

constexpr int kMaxRegQubits = 10;                    // register-resident path (one circuit per warp or less)
constexpr int kMaxQubits = 24;                       // streaming path up to n = 24
constexpr size_t kScratchBudget = size_t(48) << 30;  // bytes of per-CTA branch scratch (n > 12)
constexpr int64_t kSubCap = 4096;                    // circuits per dvqls_terms_subset launch
constexpr int kGraphCache = 16;                      // instantiated graphs kept per context

// Path of the Hadamard-test kernel
enum class Path {
  reg,       // n <= 10: hadamard_kernel (complex) or plane_kernel (n = 10, uniform b); 1-D flat grid
  onchip,    // n = 11, 12 uniform b: onchip_plane_kernel (1-D flat grid) + planar x copy
  pstream,   // n >= 13 uniform b: stream_plane_kernel (grid (G, K)) + planar x copy
  hh_tile,   // Householder b: n = 11, 12 stream_hadamard_kernel, n >= 13 stream_hh_kernel (grid (G, K))
};

struct GraphEntry {
  int kind = 0, K = 0;
  const void* a = nullptr;
  const void* b = nullptr;
  cudaGraphExec_t exec = nullptr;
  unsigned long long last_use = 0;
};

}  // namespace

struct dvqls_ctx {
  int n = 0, layers = 0, L = 0, P = 0, N = 0;
  int bkind = DVQLS_B_UNIFORM, entangler = 0;
  int device = 0, rank = 0, world = 1, max_batch = 16, timing = 0;
  int vrank = 0, vworld = 1;  // virtual rank (single-GPU sharding, opts.virtual_*)
  int64_t C = 0, c0 = 0, c1 = 0, chunk = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  int (*host_allgather)(void*, const void*, void*, size_t) = nullptr;
  void* host_user = nullptr;

  Path path = Path::reg;
  KernelCfg kc;
  int grid = 0;      // CTAs per theta (grid (G, K) kernels) / for one theta (flat-grid kernels)
  int grid_cap = 0;  // flat-grid kernels: resident CTAs (SMs x occupancy), the cap of a K-theta launch
  int64_t NG = 0;    // partial quadruples per theta
  PrefixCfg pc;      // n <= 12 SMEM prefix (pc.fn == nullptr: global-memory prefix, n >= 13)
  bool pdl = false;  // Hadamard kernel launched as a programmatic dependent of the prefix
  bool use_graphs = false;
  double hv_scale = 0.0;

  PauliTerm* d_tab = nullptr;
  double2* d_coef = nullptr;
  double2* d_hv = nullptr;
  double* d_theta = nullptr;     // max_batch * P
  double2* d_x = nullptr;        // max_batch * N
  double* d_terms = nullptr;     // max_batch * chunk
  double* d_partials = nullptr;  // max_batch * NG * 4
  double* d_ep = nullptr;        // max_batch * 4 (NCCL allreduce buffer)
  double* d_outbuf = nullptr;    // 1 + max_batch * 5: [error word | (C, E, Psi) per theta]
  double* d_out = nullptr;       // d_outbuf + 1
  unsigned* d_err = nullptr;     // (unsigned*)d_outbuf: sticky fused-allreduce timeout flag
  unsigned long long* d_epochs = nullptr;  // max_batch fused-allreduce epochs
  double* d_gather = nullptr;    // world * chunk (NCCL terms allgather)
  double* h_stage = nullptr;     // pinned staging (mapped: h_stage_dev is its device alias)
  double* h_stage_dev = nullptr;
  size_t h_stage_bytes = 0;
  unsigned* d_counter = nullptr; // last-CTA tickets, one per theta slot
  // fused NVLink allreduce (world > 1): own symmetric buffer + IPC-mapped peer buffers
  bool p2p = false;
  bool broken = false;           // a peer timed out: evaluations refused
  unsigned long long p2p_timeout_ns = 60ull * 1000000000ull;
  char* d_sym = nullptr;
  std::vector<char*> peer_ptrs;
  char** d_peers = nullptr;
  double2* d_scratch = nullptr;  // grid * N doubles (n > 12, uniform b)
  double* d_xq = nullptr;        // onchip: [K][x_re | -x_re | x_im | -x_im]
  double* d_xp = nullptr;        // pstream: planar copy of x [K][re N | im N]
  std::vector<void**> carved;    // device buffers carved from a caller workspace (not freed)
  double2* d_x2 = nullptr;       // ring ping-pong buffer (n > 12 prefix)
  double2* d_gates = nullptr;    // fused-gate table (n > 12 prefix)
  int64_t* d_cidx = nullptr;     // circuit subset (dvqls_terms_subset), kSubCap
  double* d_sub = nullptr;       // kSubCap
  // parameter-shift gradient (dvqls_cost_grad)
  double* d_gtheta = nullptr;    // (2P + 1) * P
  double* d_gres = nullptr;      // (2P + 1) * 5
  double* d_gout = nullptr;      // 1 + P + 4

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

  std::vector<GraphEntry> graphs;
  unsigned long long graph_clock = 0;
  int graphs_built = 0;
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
  P2PArgs p2p{1, 0, ctx->max_batch, ctx->d_epochs, nullptr, ctx->p2p_timeout_ns, ctx->d_err};
  if (red_out && with_cost && ctx->p2p) {
    p2p.world = ctx->world;
    p2p.rank = ctx->rank;
    p2p.peers = ctx->d_peers;
  }
  return p2p;
}

bool flat_grid(const dvqls_ctx* ctx) { return ctx->path == Path::reg || ctx->path == Path::onchip; }

// NEXT-2: distinct observables [d0, d1) of every theta; e -> out_e (nullable), fused reduction
int launch_pauli(dvqls_ctx* ctx, int K, int64_t d0, int64_t d1, double2* out_e, int grid, double* red_out,
                 int with_cost) {
  P2PArgs p2p = make_p2p(ctx, red_out, with_cost);
  const int stage = ctx->pauli_smem > 0 ? 1 : 0;
  void* args[] = {(void*)&ctx->d_x, (void*)&ctx->n, (void*)&ctx->d_obs, (void*)&ctx->d_wE, (void*)&ctx->d_wP,
                  (void*)&d0, (void*)&d1, (void*)&ctx->D, (void*)&out_e, (void*)&ctx->d_partials,
                  (void*)&with_cost, (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p, (void*)&stage};
  CK(cudaLaunchKernel(pauli_expect_fn(), dim3(grid, K), dim3(pauli_warps() * 32), args, ctx->pauli_smem,
                      ctx->stream));
  return DVQLS_OK;
}

// Hadamard-test kernel over circuits [c0, c0 + C) (or the list cidx[0..C)) of every theta.
// red_out != NULL: the kernel's last CTA per theta also performs the fixed-order reduction
// (with_cost 1: 5 doubles C, E, Psi per theta; 2: the same with C = NaN (virtual rank);
//  0: 4 doubles E, Psi for the NCCL allreduce).
int launch_hadamard(dvqls_ctx* ctx, int K, int64_t c0, int64_t C, const int64_t* cidx, double* terms, int grid,
                    double* red_out = nullptr, int with_cost = 0) {
  P2PArgs p2p = make_p2p(ctx, red_out, with_cost);
  const dim3 block(ctx->kc.warps * 32);
  if (flat_grid(ctx)) {
    // one persistent 1-D grid over the flattened K x C work: enough CTAs for all K thetas'
    // circuits, up to one resident wave
    const int g1 = int(std::max<int64_t>(
        1, std::min<int64_t>(ctx->grid_cap, (int64_t(K) * C + ctx->kc.groups - 1) / std::max(1, ctx->kc.groups))));
    if (ctx->path == Path::onchip) {  // [x_re | -x_re | x_im | -x_im], each theta's block aligned to its size
      const size_t blk = sizeof(double) * 4 * size_t(ctx->N);
      double* xq = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ctx->d_xq) + blk - 1) & ~uintptr_t(blk - 1));
      launch_to_planar4(ctx->d_x, uint32_t(ctx->N), uint32_t(K), xq, ctx->stream);
      void* args[] = {(void*)&xq, (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->L, (void*)&c0,
                      (void*)&C, (void*)&K, (void*)&terms, (void*)&ctx->d_partials, (void*)&with_cost,
                      (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p};
      CK(cudaLaunchKernel(ctx->kc.fn, dim3(g1), block, args, ctx->kc.smem, ctx->stream));
      return DVQLS_OK;
    }
    void* args[] = {(void*)&ctx->d_x,      (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->d_hv,
                    (void*)&ctx->hv_scale, (void*)&ctx->L,     (void*)&c0,          (void*)&C,
                    (void*)&K,             (void*)&terms,      (void*)&ctx->d_partials, (void*)&with_cost,
                    (void*)&red_out,       (void*)&ctx->d_counter, (void*)&p2p};
    if (ctx->pdl) {  // scheduled while the prefix runs; the kernel's griddepcontrol.wait orders the reads
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(g1);
      lc.blockDim = block;
      lc.dynamicSmemBytes = ctx->kc.smem;
      lc.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      CK(cudaLaunchKernelExC(&lc, ctx->kc.fn, args));
    } else {
      CK(cudaLaunchKernel(ctx->kc.fn, dim3(g1), block, args, ctx->kc.smem, ctx->stream));
    }
    return DVQLS_OK;
  }
  // grid (G, K) kernels: one circuit per CTA at a time
  if (ctx->n > 12) grid = std::max(1, grid / K);  // n > 12 uniform b: `grid` CTAs share the scratch in total
  const dim3 g(grid, K);
  if (ctx->path == Path::pstream) {  // planar x, then the real-plane streaming kernel
    launch_to_planar(ctx->d_x, uint32_t(ctx->N), uint32_t(K), ctx->d_xp, ctx->stream);
    double* scr = reinterpret_cast<double*>(ctx->d_scratch);
    void* args[] = {(void*)&ctx->d_xp, (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->L, (void*)&ctx->n,
                    (void*)&c0, (void*)&C, (void*)&cidx, (void*)&scr, (void*)&terms, (void*)&ctx->d_partials,
                    (void*)&with_cost, (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p};
    CK(cudaLaunchKernel(ctx->kc.fn, g, block, args, ctx->kc.smem, ctx->stream));
  } else {  // Householder b (stream.cuh)
    void* args[] = {(void*)&ctx->d_x, (void*)&ctx->d_tab, (void*)&ctx->d_coef, (void*)&ctx->d_hv,
                    (void*)&ctx->hv_scale, (void*)&ctx->L, (void*)&ctx->n, (void*)&c0, (void*)&C,
                    (void*)&cidx, (void*)&ctx->d_scratch, (void*)&terms, (void*)&ctx->d_partials,
                    (void*)&with_cost, (void*)&red_out, (void*)&ctx->d_counter, (void*)&p2p};
    CK(cudaLaunchKernel(ctx->kc.fn, g, block, args, ctx->kc.smem, ctx->stream));
  }
  return DVQLS_OK;
}

// a2: x_k = V(theta_k)|0> for the K thetas
int launch_prefix(dvqls_ctx* ctx, int K, const double* thetas_dev) {
  if (!ctx->pc.fn) {
    const int e = launch_prefix_global(ctx->n, ctx->layers, ctx->entangler, K, thetas_dev, ctx->d_x, ctx->d_x2,
                                       ctx->d_gates, ctx->stream);
    if (e) return fail(ctx, DVQLS_E_CUDA, "global prefix: %s", cudaGetErrorString(cudaError_t(e)));
    return DVQLS_OK;
  }
  if (ctx->pc.cluster > 0) {  // thread-block cluster of pc.cluster CTAs per theta (prefix_cluster.cuh)
    void* args[] = {(void*)&ctx->layers, (void*)&ctx->entangler, (void*)&thetas_dev, (void*)&ctx->d_x};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(ctx->pc.cluster, K);
    lc.blockDim = dim3(ctx->pc.threads);
    lc.dynamicSmemBytes = ctx->pc.smem;
    lc.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ctx->pc.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelExC(&lc, ctx->pc.fn, args));
  } else if (ctx->pc.with_n) {
    void* args[] = {(void*)&ctx->n, (void*)&ctx->layers, (void*)&ctx->entangler, (void*)&thetas_dev,
                    (void*)&ctx->d_x};
    CK(cudaLaunchKernel(ctx->pc.fn, dim3(K), dim3(ctx->pc.threads), args, ctx->pc.smem, ctx->stream));
  } else {
    void* args[] = {(void*)&ctx->layers, (void*)&ctx->entangler, (void*)&thetas_dev, (void*)&ctx->d_x};
    CK(cudaLaunchKernel(ctx->pc.fn, dim3(K), dim3(ctx->pc.threads), args, ctx->pc.smem, ctx->stream));
  }
  return DVQLS_OK;
}

// One evaluation of the hot path for K thetas (a2-a10).  want_cost: (C, E, Psi) per theta into
// out_dev (5 doubles each); else the terms of this rank's block into d_terms.
int launch_eval(dvqls_ctx* ctx, int K, const double* thetas_dev, bool want_cost, double* out_dev) {
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  int rc = launch_prefix(ctx, K, thetas_dev);
  if (rc) return rc;
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  const int64_t Cloc = ctx->c1 - ctx->c0;
  // a9 (+ a10 on one rank / over peer memory) fused into the kernel tail
  const bool direct = ctx->world == 1 || ctx->p2p;  // kernel writes the final (C, E, Psi)
  double* red = want_cost ? (direct ? out_dev : ctx->d_ep) : nullptr;
  const int wc = direct ? (ctx->vworld > 1 ? 2 : 1) : 0;
  if (ctx->mode == DVQLS_MODE_PAULI) {
    if (want_cost) {
      rc = launch_pauli(ctx, K, ctx->d0, ctx->d1, nullptr, ctx->pgrid, red, wc);
    } else {  // terms: every observable on every rank (cheap), then this rank's circuit block
      rc = launch_pauli(ctx, K, 0, ctx->D, ctx->d_e, ctx->pgrid, nullptr, 0);
      if (!rc) {
        launch_pauli_scatter(ctx->d_e, ctx->d_task, ctx->c0, Cloc, ctx->d_terms, ctx->stream);
        CK(cudaGetLastError());
      }
    }
  } else {
    rc = launch_hadamard(ctx, K, ctx->c0, Cloc, nullptr, ctx->d_terms, ctx->grid, red, wc);
  }
  if (rc) return rc;
  if (ctx->timing) CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  if (want_cost && !direct) {
    CKN(nccl().AllReduce(ctx->d_ep, ctx->d_ep, size_t(4) * K, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    launch_finalize(ctx->d_ep, K, ctx->n, out_dev, ctx->stream);
    CK(cudaGetLastError());
  }
  if (ctx->timing) {
    CK(cudaEventRecord(ctx->ev[3], ctx->stream));
    ctx->timed_once = true;
  }
  return DVQLS_OK;
}

// Parameter-shift gradient (shift.cuh): 2P + 1 thetas, evaluated in batches of max_batch
int launch_grad(dvqls_ctx* ctx, const double* theta_dev, double* out_dev) {
  const int R = 2 * ctx->P + 1;
  launch_shift_thetas(theta_dev, ctx->P, ctx->d_gtheta, ctx->stream);
  CK(cudaGetLastError());
  for (int r0 = 0; r0 < R; r0 += ctx->max_batch) {
    const int K = std::min(ctx->max_batch, R - r0);
    int rc = launch_eval(ctx, K, ctx->d_gtheta + size_t(r0) * ctx->P, true, ctx->d_gres + size_t(r0) * 5);
    if (rc) return rc;
  }
  launch_shift_grad(ctx->d_gres, ctx->P, ctx->n, out_dev, ctx->stream);
  CK(cudaGetLastError());
  return DVQLS_OK;
}

// Run `body` (device work on ctx->stream) directly, or as a CUDA graph captured on first use for
// this (kind, K, a, b) and replayed afterwards (opts.graphs; not with timing events or NCCL).
template <class F>
int run_graph(dvqls_ctx* ctx, int kind, int K, const void* a, const void* b, F&& body) {
  if (!ctx->use_graphs) return body();
  GraphEntry* hit = nullptr;
  for (auto& g : ctx->graphs)
    if (g.kind == kind && g.K == K && g.a == a && g.b == b) hit = &g;
  if (!hit) {
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    int rc = body();
    cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess) return fail(ctx, DVQLS_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    cudaGraphExec_t exec = nullptr;
    ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return fail(ctx, DVQLS_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    if (int(ctx->graphs.size()) >= kGraphCache) {  // evict the least recently used
      auto lru = std::min_element(ctx->graphs.begin(), ctx->graphs.end(),
                                  [](const GraphEntry& x, const GraphEntry& y) { return x.last_use < y.last_use; });
      cudaGraphExecDestroy(lru->exec);
      ctx->graphs.erase(lru);
    }
    ctx->graphs.push_back(GraphEntry{kind, K, a, b, exec, 0});
    ++ctx->graphs_built;
    hit = &ctx->graphs.back();
  }
  hit->last_use = ++ctx->graph_clock;
  CK(cudaGraphLaunch(hit->exec, ctx->stream));
  return DVQLS_OK;
}

int check_usable(dvqls_ctx* ctx) {
  if (ctx->broken)
    return fail(ctx, DVQLS_E_NCCL,
                "a peer of the fused allreduce timed out earlier: the context is unusable (destroy and recreate)");
  return DVQLS_OK;
}

// error word copied back with the results: nonzero = a peer timed out
int check_err_word(dvqls_ctx* ctx, unsigned word) {
  if (word) {
    ctx->broken = true;
    return fail(ctx, DVQLS_E_NCCL, "fused allreduce: a peer did not publish within %llu ms (p2p_timeout_ms)",
                (unsigned long long)(ctx->p2p_timeout_ns / 1000000ull));
  }
  return DVQLS_OK;
}

int all_gather_host(dvqls_ctx* ctx, const void* send, void* recv, size_t bytes) {
  if (!ctx->host_allgather || ctx->host_allgather(ctx->host_user, send, recv, bytes) != 0)
    return fail(ctx, DVQLS_E_NCCL, "host_allgather failed");
  return DVQLS_OK;
}

void release(dvqls_ctx* c) {
  if (!c) return;
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  for (void** p : c->carved) *p = nullptr;  // owned by the caller's workspace
  for (int q = 0; q < int(c->peer_ptrs.size()); ++q)
    if (q != c->rank && c->peer_ptrs[q]) cudaIpcCloseMemHandle(c->peer_ptrs[q]);
  cudaFree(c->d_sym); cudaFree(c->d_peers);
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  void* bufs[] = {c->d_tab, c->d_coef, c->d_hv, c->d_theta, c->d_x, c->d_terms, c->d_partials, c->d_ep,
                  c->d_outbuf, c->d_epochs, c->d_gather, c->d_obs, c->d_wE, c->d_wP, c->d_task, c->d_e,
                  c->d_b, c->d_beta, c->d_out6, c->d_gcounter, c->d_counter, c->d_scratch, c->d_xp, c->d_xq,
                  c->d_x2, c->d_gates, c->d_cidx, c->d_sub, c->d_gtheta, c->d_gres, c->d_gout};
  for (void* p : bufs) cudaFree(p);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (auto& e : c->ev) if (e) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
}

// Symmetric buffers for the fused allreduce: allocate, exchange IPC handles (NCCL allgather or the
// caller's host allgather, create-time only), map every peer's buffer.  All ranks agree on the
// outcome; without a mapping the context falls back to ncclAllReduce, or fails without NCCL.
int setup_p2p(dvqls_ctx* ctx) {
  const size_t bytes = size_t(2) * ctx->world * ctx->max_batch * (32 + 8);
  CK(cudaMalloc((void**)&ctx->d_sym, bytes));
  CK(cudaMemsetAsync(ctx->d_sym, 0, bytes, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->d_sym));
  std::vector<cudaIpcMemHandle_t> all(ctx->world);
  if (ctx->comm) {
    char* d_h = nullptr;
    CK(cudaMalloc((void**)&d_h, sizeof(h) * (ctx->world + 1)));
    CK(cudaMemcpyAsync(d_h, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
    ncclResult_t r = nccl().AllGather(d_h, d_h + sizeof(h), sizeof(h), ncclChar, ctx->comm, ctx->stream);
    if (r != ncclSuccess) {
      cudaFree(d_h);
      return fail(ctx, DVQLS_E_NCCL, "handle allgather: %s", nccl().GetErrorString(r));
    }
    CK(cudaMemcpyAsync(all.data(), d_h + sizeof(h), sizeof(h) * ctx->world, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(d_h);
  } else {
    int rc = all_gather_host(ctx, &h, all.data(), sizeof(h));
    if (rc) return rc;
  }
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
  // every rank must agree: fall back together if any rank could not map
  int all_ok = 0;
  if (ctx->comm) {
    int flag = ok ? 1 : 0;
    int* d_f = nullptr;
    CK(cudaMalloc((void**)&d_f, sizeof(int)));
    CK(cudaMemcpyAsync(d_f, &flag, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    ncclResult_t r2 = nccl().AllReduce(d_f, d_f, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream);
    if (r2 != ncclSuccess) { cudaFree(d_f); return fail(ctx, DVQLS_E_NCCL, "p2p agreement"); }
    CK(cudaMemcpyAsync(&all_ok, d_f, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(d_f);
  } else {
    int flag = ok ? 1 : 0;
    std::vector<int> flags(ctx->world, 0);
    int rc = all_gather_host(ctx, &flag, flags.data(), sizeof(int));
    if (rc) return rc;
    all_ok = *std::min_element(flags.begin(), flags.end());
  }
  ctx->p2p = all_ok == 1;
  if (ctx->p2p) {
    CK(cudaMalloc((void**)&ctx->d_peers, sizeof(char*) * ctx->world));
    CK(cudaMemcpyAsync(ctx->d_peers, ctx->peer_ptrs.data(), sizeof(char*) * ctx->world, cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  } else if (!ctx->comm) {
    return fail(ctx, DVQLS_E_NCCL, "peer buffers could not be mapped on every rank and no NCCL communicator exists");
  }
  return DVQLS_OK;
}

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

  ctx = new dvqls_ctx();
  ctx->n = n; ctx->layers = layers; ctx->L = L; ctx->P = 3 * n * layers; ctx->N = 1 << n;
  dvqls_opts o{};
  if (opts) o = *opts;
  else o.device = -1, o.world = 1;
  ctx->device = o.device; ctx->rank = o.rank; ctx->world = o.world;
  ctx->entangler = o.entangler; ctx->timing = o.timing; ctx->mode = o.mode;
  if (o.max_batch > 0) ctx->max_batch = o.max_batch;
  if (o.virtual_world > 1) { ctx->vworld = o.virtual_world; ctx->vrank = o.virtual_rank; }
  if (o.p2p_timeout_ms > 0) ctx->p2p_timeout_ns = (unsigned long long)o.p2p_timeout_ms * 1000000ull;
  ctx->host_allgather = o.host_allgather;
  ctx->host_user = o.host_allgather_user;
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
  if (o.virtual_world > 1 && (ctx->world != 1 || o.virtual_rank < 0 || o.virtual_rank >= o.virtual_world)) {
    fail(ctx, DVQLS_E_ARG, "virtual ranks need world == 1 and 0 <= virtual_rank < virtual_world");
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
  if (o.prefix < 0 || o.prefix > 1) {
    fail(ctx, DVQLS_E_ARG, "prefix must be 0 or 1");
    return bail(DVQLS_E_ARG);
  }
  if (o.variant < 0 || o.variant > 2) {
    fail(ctx, DVQLS_E_ARG, "variant must be 0, 1 or 2");
    return bail(DVQLS_E_ARG);
  }
  if (o.allreduce != DVQLS_ALLREDUCE_P2P && o.allreduce != DVQLS_ALLREDUCE_NCCL) {
    fail(ctx, DVQLS_E_ARG, "allreduce must be DVQLS_ALLREDUCE_P2P or DVQLS_ALLREDUCE_NCCL");
    return bail(DVQLS_E_ARG);
  }
  if (ctx->world > 1 && !plan_bytes && !o.nccl_unique_id && !o.host_allgather) {
    fail(ctx, DVQLS_E_ARG, "world > 1 requires opts.nccl_unique_id or opts.host_allgather");
    return bail(DVQLS_E_ARG);
  }
  if (ctx->world > 1 && !o.nccl_unique_id && o.allreduce == DVQLS_ALLREDUCE_NCCL) {
    fail(ctx, DVQLS_E_ARG, "allreduce = NCCL needs opts.nccl_unique_id");
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
  const bool hh = ctx->bkind == DVQLS_B_AMPLITUDES;
  if (hh) {
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
  if (o.cuda_stream) {
    ctx->stream = (cudaStream_t)o.cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      fail(ctx, DVQLS_E_CUDA, "cudaStreamCreate failed");
      return bail(DVQLS_E_CUDA);
    }
    ctx->own_stream = true;
  }
  if (n <= kMaxRegQubits) {
    ctx->path = Path::reg;
    if (n == 10 && !hh)
      ctx->kc = o.variant == 1 ? plane_cfg() : plane2_cfg();  // default: two circuits per warp
    else
      ctx->kc = n <= 6 ? reg_cfg_lo(n, hh) : reg_cfg_hi(n, hh);
  } else if (hh) {
    ctx->path = Path::hh_tile;
    ctx->kc = stream_hh_cfg(n);
  } else if (n <= 12) {
    ctx->path = Path::onchip;
    // n = 12: x staged in SMEM (measured 5.86e7 vs 5.00e7 circuits/s at cfg5, K=2); n = 11: x from L2
    // (10 warps with x in SMEM measured no faster: profiles/r2_onchip/)
    ctx->kc = onchip_cfg(n, n == 12);
  } else {
    ctx->path = Path::pstream;
    // n >= 16 (scratch no longer L2-resident): TMA bulk-copy staging of the last-pass and large-run
    // mid-pass tiles (measured +1-3 % at n = 16..20, -5 % at n = 14 where the scratch stays in L2)
    const int stage_from = o.stage == 1 ? 13 : 16;
    ctx->kc = stream_plane_cfg(o.stage != -1 && n >= stage_from);
  }
  if (!ctx->kc.fn) {
    fail(ctx, DVQLS_E_UNSUPPORTED, "no Hadamard-test kernel for n = %d", n);
    return bail(DVQLS_E_UNSUPPORTED);
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
  if (ctx->vworld > 1)
    dvqls_shard_range(ctx->C, ctx->vrank, ctx->vworld, &ctx->c0, &ctx->c1);
  else
    dvqls_shard_range(ctx->C, ctx->rank, ctx->world, &ctx->c0, &ctx->c1);
  ctx->chunk = 0;  // the largest rank block (terms buffer and allgather slot)
  for (int r = 0; r < std::max(ctx->world, ctx->vworld); ++r) {
    int64_t a, b;
    dvqls_shard_range(ctx->C, r, std::max(ctx->world, ctx->vworld), &a, &b);
    ctx->chunk = std::max(ctx->chunk, b - a);
  }
  if (ctx->c1 - ctx->c0 > int64_t(INT32_MAX)) {  // the kernels index a rank's circuits with 32-bit ints
    fail(ctx, DVQLS_E_UNSUPPORTED, "%lld circuits on one rank (more than 2^31 - 1): use more ranks",
         (long long)(ctx->c1 - ctx->c0));
    return bail(DVQLS_E_UNSUPPORTED);
  }
  const int64_t Cloc = ctx->c1 - ctx->c0;
  const int64_t groups_per_cta = flat_grid(ctx) ? int64_t(ctx->kc.groups) : 1;
  int64_t want = int64_t(prop.multiProcessorCount) * occ;
  const bool scratch = ctx->path == Path::pstream;  // per-CTA 2^n-double branch scratch
  if (scratch) want = std::max<int64_t>(1, std::min<int64_t>(want, int64_t(kScratchBudget / (8 * size_t(ctx->N)))));
  if (!flat_grid(ctx) && o.stream_grid > 0) want = std::min<int64_t>(want, o.stream_grid);
  const int64_t need = (Cloc + groups_per_cta - 1) / groups_per_cta;
  ctx->grid = int(std::max<int64_t>(1, std::min(want, need)));
  ctx->grid_cap = int(std::max<int64_t>(1, want));
  ctx->NG = std::max<int64_t>(int64_t(ctx->grid) * groups_per_cta, flat_grid(ctx) ? ctx->grid_cap : 0);

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
    if (ctx->vworld > 1)
      dvqls_shard_range(ctx->D, ctx->vrank, ctx->vworld, &ctx->d0, &ctx->d1);
    else
      dvqls_shard_range(ctx->D, ctx->rank, ctx->world, &ctx->d0, &ctx->d1);
    ctx->pauli_smem = ctx->N <= 8192 ? sizeof(double2) * size_t(ctx->N) : 0;
    if (cudaFuncSetAttribute(pauli_expect_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, int(ctx->pauli_smem)) !=
        cudaSuccess) {
      fail(ctx, DVQLS_E_CUDA, "pauli kernel smem");
      return bail(DVQLS_E_CUDA);
    }
    int pocc = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pocc, pauli_expect_fn(), pauli_warps() * 32, ctx->pauli_smem);
    const int64_t pw = int64_t(prop.multiProcessorCount) * std::max(1, pocc);
    const int64_t pneed = (ctx->D + pauli_warps() - 1) / pauli_warps();  // terms launches cover all D
    ctx->pgrid = int(std::max<int64_t>(1, std::min(pw, pneed)));
    ctx->NG = std::max<int64_t>(ctx->NG, ctx->pgrid);
  }

  // ---- prefix (a2) ----------------------------------------------------------------------
  if (n <= 12) {
    ctx->pc = prefix_cfg(n, layers, o.prefix == 1);
    if (!ctx->pc.fn || cudaFuncSetAttribute(ctx->pc.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(ctx->pc.smem)) != cudaSuccess) {
      fail(ctx, DVQLS_E_CUDA, "prefix kernel smem %zu B", ctx->pc.smem);
      return bail(DVQLS_E_CUDA);
    }
    // the prefix and the Hadamard-test kernel run back to back every call: the maximum SMEM
    // carveout for both keeps the SMs from repartitioning L1/SMEM between them
    cudaFuncSetAttribute(ctx->pc.fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
  }
  cudaFuncSetAttribute(ctx->kc.fn, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared));
  cudaGetLastError();
  // PDL behind the SMEM prefix for the register path (n <= 10, 1-D grid; the kernels there execute
  // griddepcontrol.wait).  Off while per-kernel timing events sit between the two launches.
  ctx->pdl = n <= kMaxRegQubits && !ctx->timing && o.pdl != -1;

  // ---- device buffers: cudaMalloc'd once here, or carved from the caller's workspace -----
  const int KB = ctx->max_batch;
  const size_t R = size_t(2 * ctx->P + 1);  // parameter-shift rows
  std::vector<std::pair<void**, size_t>> req;
  auto buffer = [&](bool cond, void* p, size_t bytes) {
    if (cond) req.emplace_back(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 16));
  };
  // Pauli mode: a plan has no strings, so it sizes for one observable per task (the bound)
  const size_t nobs = plan_bytes ? size_t(ctx->C / 2) : obs.size();
  const size_t ntask = plan_bytes ? size_t(ctx->C / 2) : task.size();
  const bool subset = !flat_grid(ctx) && ctx->mode == DVQLS_MODE_CIRCUITS;
  buffer(true, &ctx->d_tab, sizeof(PauliTerm) * L);
  buffer(true, &ctx->d_coef, sizeof(double2) * L);
  buffer(true, &ctx->d_hv, sizeof(double2) * ctx->N);
  buffer(true, &ctx->d_theta, sizeof(double) * KB * ctx->P);
  buffer(true, &ctx->d_x, sizeof(double2) * KB * ctx->N);
  buffer(true, &ctx->d_terms, sizeof(double) * KB * ctx->chunk);
  buffer(true, &ctx->d_partials, sizeof(double) * KB * ctx->NG * 4);
  buffer(true, &ctx->d_ep, sizeof(double) * KB * 4);
  buffer(true, &ctx->d_outbuf, sizeof(double) * (size_t(KB) * 5 + 1));
  buffer(true, &ctx->d_epochs, sizeof(unsigned long long) * KB);
  buffer(ctx->world > 1, &ctx->d_gather, sizeof(double) * ctx->world * ctx->chunk);
  buffer(true, &ctx->d_counter, sizeof(unsigned) * KB);
  buffer(true, &ctx->d_gcounter, sizeof(unsigned) * KB);
  buffer(true, &ctx->d_beta, sizeof(double) * 2 * KB * size_t(L));
  buffer(true, &ctx->d_out6, sizeof(double) * 6 * KB);
  buffer(true, &ctx->d_gtheta, sizeof(double) * R * ctx->P);
  buffer(true, &ctx->d_gres, sizeof(double) * R * 5);
  buffer(true, &ctx->d_gout, sizeof(double) * (size_t(ctx->P) + 5));
  buffer(hh, &ctx->d_b, sizeof(double2) * ctx->N);
  buffer(scratch && ctx->mode == DVQLS_MODE_CIRCUITS, &ctx->d_scratch, sizeof(double) * size_t(ctx->grid) * ctx->N);
  buffer(ctx->path == Path::pstream, &ctx->d_xp, sizeof(double2) * KB * ctx->N);
  // onchip: every theta's 4N-double x block aligned to its size (XOR addressing); slack for the round-up
  buffer(ctx->path == Path::onchip, &ctx->d_xq, sizeof(double) * 4 * (size_t(KB) + 1) * ctx->N);
  buffer(subset, &ctx->d_cidx, sizeof(int64_t) * kSubCap);
  buffer(subset, &ctx->d_sub, sizeof(double) * kSubCap);
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
  if (o.workspace_dev) {
    if ((reinterpret_cast<uintptr_t>(o.workspace_dev) & 255u) || o.workspace_bytes < total) {
      fail(ctx, DVQLS_E_ARG, "workspace: %zu bytes at %p, need %zu bytes 256-byte aligned", o.workspace_bytes,
           o.workspace_dev, total);
      return bail(DVQLS_E_ARG);
    }
    char* base = static_cast<char*>(o.workspace_dev);
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
  ctx->d_out = ctx->d_outbuf + 1;
  ctx->d_err = reinterpret_cast<unsigned*>(ctx->d_outbuf);
  ctx->h_stage_bytes = sizeof(double) * std::max<size_t>({size_t(KB) * (ctx->P + 5) + 1, 2 * size_t(ctx->P) + 6, 64});
  if (cudaHostAlloc((void**)&ctx->h_stage, ctx->h_stage_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&ctx->h_stage_dev, ctx->h_stage, 0) != cudaSuccess) {
    fail(ctx, DVQLS_E_CUDA, "cudaHostAlloc (mapped) failed");
    return bail(DVQLS_E_CUDA);
  }
  // tables and counters are written on the context stream (the stream every later call uses)
  // and create waits for them, so no call can race the uploads
  cudaStream_t st = ctx->stream;
  if (cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned) * KB, st) ||
      cudaMemsetAsync(ctx->d_gcounter, 0, sizeof(unsigned) * KB, st) ||
      cudaMemsetAsync(ctx->d_outbuf, 0, sizeof(double) * (size_t(KB) * 5 + 1), st) ||
      cudaMemsetAsync(ctx->d_epochs, 0, sizeof(unsigned long long) * KB, st) ||
      (hh && cudaMemcpyAsync(ctx->d_b, bprep->amps, sizeof(double2) * ctx->N, cudaMemcpyHostToDevice, st)) ||
      cudaMemcpyAsync(ctx->d_tab, tab.data(), sizeof(PauliTerm) * L, cudaMemcpyHostToDevice, st) ||
      cudaMemcpyAsync(ctx->d_coef, coef.data(), sizeof(double2) * L, cudaMemcpyHostToDevice, st) ||
      (!hv.empty() && cudaMemcpyAsync(ctx->d_hv, hv.data(), sizeof(double2) * ctx->N, cudaMemcpyHostToDevice, st)) ||
      (!obs.empty() &&
       (cudaMemcpyAsync(ctx->d_obs, obs.data(), sizeof(pauli::Obs) * obs.size(), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(ctx->d_wE, wE.data(), sizeof(double2) * obs.size(), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(ctx->d_wP, wP.data(), sizeof(double2) * obs.size(), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(ctx->d_task, task.data(), sizeof(uint32_t) * task.size(), cudaMemcpyHostToDevice, st))) ||
      cudaStreamSynchronize(st)) {
    fail(ctx, DVQLS_E_CUDA, "table upload failed");
    return bail(DVQLS_E_CUDA);
  }
  if (ctx->timing)
    for (auto& e : ctx->ev)
      if (cudaEventCreate(&e) != cudaSuccess) {
        fail(ctx, DVQLS_E_CUDA, "cudaEventCreate failed");
        return bail(DVQLS_E_CUDA);
      }

  // ---- cross-rank reduction (a10): NCCL communicator and/or the fused peer-memory path -------
  if (ctx->world > 1 && o.nccl_unique_id) {
    if (!nccl().ok) {
      fail(ctx, DVQLS_E_NCCL, "libnccl.so.2 not loadable");
      return bail(DVQLS_E_NCCL);
    }
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_unique_id, sizeof id);
    ncclResult_t r = nccl().CommInitRank(&ctx->comm, ctx->world, id, ctx->rank);
    if (r != ncclSuccess) {
      fail(ctx, DVQLS_E_NCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
      ctx->comm = nullptr;
      return bail(DVQLS_E_NCCL);
    }
  }
  if (ctx->world > 1 && o.allreduce == DVQLS_ALLREDUCE_P2P) {
    int rc = setup_p2p(ctx);
    if (rc) return bail(rc);
  }
  ctx->use_graphs = o.graphs != -1 && !ctx->timing && (ctx->world == 1 || ctx->p2p);
  *out = ctx;
  return DVQLS_OK;
}

// host copy of the error word + K result rows, then the error / degeneracy checks
// after the results (error word + K rows) were copied to h_stage + K P: checks and unpacking
int finish_host_cost(dvqls_ctx* ctx, int K, double* out_costs, double* out_E_Psi) {
  double* h = ctx->h_stage + size_t(K) * ctx->P;
  CK(cudaStreamSynchronize(ctx->stream));
  unsigned word;
  std::memcpy(&word, h, sizeof word);
  int rc = check_err_word(ctx, word);
  if (rc) return rc;
  const double* r = h + 1;
  bool degenerate = false;
  for (int k = 0; k < K; ++k) {
    out_costs[k] = r[5 * k];
    if (out_E_Psi)
      for (int j = 0; j < 4; ++j) out_E_Psi[4 * k + j] = r[5 * k + 1 + j];
    if (ctx->vworld <= 1 && !(r[5 * k + 3] > 1e-12)) degenerate = true;
  }
  if (degenerate) return fail(ctx, DVQLS_E_DEGENERATE, "Re Psi <= 1e-12 (singular A on the ansatz state)");
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
    if (kind == DVQLS_B_AMPLITUDES && mode != DVQLS_MODE_CIRCUITS) continue;
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
  if (int rc = check_usable(ctx)) return rc;
  if (K < 1 || K > ctx->max_batch) return fail(ctx, DVQLS_E_ARG, "K=%d outside [1, max_batch=%d]", K, ctx->max_batch);
  if (!thetas_dev || !out_dev) return fail(ctx, DVQLS_E_ARG, "NULL device pointer");
  return run_graph(ctx, 0, K, thetas_dev, out_dev, [&] { return launch_eval(ctx, K, thetas_dev, true, out_dev); });
}

int dvqls_cost_grad_dev(dvqls_ctx* ctx, const double* theta_dev, double* out_dev) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (int rc = check_usable(ctx)) return rc;
  if (!theta_dev || !out_dev) return fail(ctx, DVQLS_E_ARG, "NULL device pointer");
  if (ctx->vworld > 1) return fail(ctx, DVQLS_E_ARG, "the gradient needs the global sums (not a virtual rank)");
  return run_graph(ctx, 1, 1, theta_dev, out_dev, [&] { return launch_grad(ctx, theta_dev, out_dev); });
}

int dvqls_cost_grad(dvqls_ctx* ctx, const double* theta, double* out_cost, double* out_grad, double* out_E_Psi) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (!theta || !out_cost || !out_grad) return fail(ctx, DVQLS_E_ARG, "NULL host pointer");
  if (int rc = check_usable(ctx)) return rc;
  std::memcpy(ctx->h_stage, theta, sizeof(double) * ctx->P);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, sizeof(double) * ctx->P, cudaMemcpyHostToDevice, ctx->stream));
  int rc = dvqls_cost_grad_dev(ctx, ctx->d_theta, ctx->d_gout);
  if (rc) return rc;
  double* h = ctx->h_stage + ctx->P;
  CK(cudaMemcpyAsync(h, ctx->d_gout, sizeof(double) * (size_t(ctx->P) + 5), cudaMemcpyDeviceToHost, ctx->stream));
  unsigned* hw = reinterpret_cast<unsigned*>(h + ctx->P + 5);
  CK(cudaMemcpyAsync(hw, ctx->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if ((rc = check_err_word(ctx, *hw))) return rc;
  *out_cost = h[0];
  std::memcpy(out_grad, h + 1, sizeof(double) * ctx->P);
  if (out_E_Psi) std::memcpy(out_E_Psi, h + 1 + ctx->P, sizeof(double) * 4);
  if (!(h[1 + ctx->P + 2] > 1e-12)) return fail(ctx, DVQLS_E_DEGENERATE, "Re Psi <= 1e-12 at theta");
  return DVQLS_OK;
}

int dvqls_check(dvqls_ctx* ctx) {
  if (!ctx) return DVQLS_E_ARG;
  if (int rc = check_usable(ctx)) return rc;
  unsigned word = 0;
  CK(cudaMemcpyAsync(ctx->h_stage, ctx->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  std::memcpy(&word, ctx->h_stage, sizeof word);
  return check_err_word(ctx, word);
}

int dvqls_terms_local_dev(dvqls_ctx* ctx, const double* theta_dev, double* out_dev) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (int rc = check_usable(ctx)) return rc;
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
  if (int rc = check_usable(ctx)) return rc;
  if (K < 1 || K > ctx->max_batch) return fail(ctx, DVQLS_E_ARG, "K=%d outside [1, max_batch=%d]", K, ctx->max_batch);
  if (!thetas_dev || !out6_dev) return fail(ctx, DVQLS_E_ARG, "NULL device pointer");
  if (ctx->vworld > 1) return fail(ctx, DVQLS_E_ARG, "the global cost needs the global sums (not a virtual rank)");
  double* beta = beta_dev ? beta_dev : ctx->d_beta;
  return run_graph(ctx, 2, K, thetas_dev, out6_dev, [&] {
    int rc = launch_eval(ctx, K, thetas_dev, true, ctx->d_out);
    if (rc) return rc;
    launch_overlap(dim3(ctx->L, K), ctx->d_x, ctx->n, ctx->d_tab, ctx->d_coef, ctx->d_b, ctx->L, ctx->d_out, beta,
                   out6_dev, ctx->d_gcounter, ctx->stream);
    CK(cudaGetLastError());
    return DVQLS_OK;
  });
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
  if ((rc = dvqls_check(ctx))) return rc;
  if (!(out6[3] > 1e-12)) return fail(ctx, DVQLS_E_DEGENERATE, "Re Psi <= 1e-12 (singular A on the ansatz state)");
  return DVQLS_OK;
}

int dvqls_cost_batch(dvqls_ctx* ctx, int K, const double* thetas, double* out_costs, double* out_E_Psi) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (K < 1 || K > ctx->max_batch) return fail(ctx, DVQLS_E_ARG, "K=%d outside [1, max_batch=%d]", K, ctx->max_batch);
  if (!thetas || !out_costs) return fail(ctx, DVQLS_E_ARG, "NULL host pointer");
  if (int rc = check_usable(ctx)) return rc;
  const size_t tb = sizeof(double) * size_t(K) * ctx->P;
  std::memcpy(ctx->h_stage, thetas, tb);
  double* h = ctx->h_stage + size_t(K) * ctx->P;
  if (ctx->world == 1 && ctx->vworld <= 1) {
    // zero copy: the prefix reads theta from the mapped pinned stage and the fused reduction writes
    // (C, E, Psi) straight into it -- one graph of two kernels, no copy nodes on the call path (the
    // error word is only ever set by the cross-rank reduction, so a single rank leaves it 0)
    std::memset(h, 0, sizeof(double));
    double* hd = ctx->h_stage_dev + size_t(K) * ctx->P;
    int rc = run_graph(ctx, 4, K, ctx->h_stage, h, [&] { return launch_eval(ctx, K, ctx->h_stage_dev, true, hd + 1); });
    if (rc) return rc;
    return finish_host_cost(ctx, K, out_costs, out_E_Psi);
  }
  // theta H2D from the pinned stage, the whole path, results D2H: one graph launch per call
  int rc = run_graph(ctx, 3, K, ctx->h_stage, h, [&] {
    CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, tb, cudaMemcpyHostToDevice, ctx->stream));
    int r = launch_eval(ctx, K, ctx->d_theta, true, ctx->d_out);
    if (r) return r;
    CK(cudaMemcpyAsync(h, ctx->d_outbuf, sizeof(double) * (1 + 5 * size_t(K)), cudaMemcpyDeviceToHost, ctx->stream));
    return DVQLS_OK;
  });
  if (rc) return rc;
  return finish_host_cost(ctx, K, out_costs, out_E_Psi);
}

int dvqls_cost(dvqls_ctx* ctx, const double* theta, double* out_cost, double* out_E_Psi) {
  return dvqls_cost_batch(ctx, 1, theta, out_cost, out_E_Psi);
}

int dvqls_terms(dvqls_ctx* ctx, const double* theta, double* out) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (int rc = check_usable(ctx)) return rc;
  if (!theta || !out) return fail(ctx, DVQLS_E_ARG, "NULL host pointer");
  std::memcpy(ctx->h_stage, theta, sizeof(double) * ctx->P);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, sizeof(double) * ctx->P, cudaMemcpyHostToDevice, ctx->stream));
  int rc = launch_eval(ctx, 1, ctx->d_theta, false, nullptr);
  if (rc) return rc;
  const int64_t Cloc = ctx->c1 - ctx->c0;
  if (ctx->world == 1) {  // (a virtual rank writes its block in place)
    CK(cudaMemcpyAsync(out + ctx->c0, ctx->d_terms, sizeof(double) * Cloc, cudaMemcpyDeviceToHost, ctx->stream));
  } else if (ctx->comm) {
    CKN(nccl().AllGather(ctx->d_terms, ctx->d_gather, size_t(ctx->chunk), ncclDouble, ctx->comm, ctx->stream));
    for (int r = 0; r < ctx->world; ++r) {
      int64_t a, b;
      dvqls_shard_range(ctx->C, r, ctx->world, &a, &b);
      CK(cudaMemcpyAsync(out + a, ctx->d_gather + size_t(r) * ctx->chunk, sizeof(double) * (b - a),
                         cudaMemcpyDeviceToHost, ctx->stream));
    }
  } else {  // host allgather of the term slices (chunk doubles per rank)
    std::vector<double> mine(size_t(ctx->chunk), 0.0), all(size_t(ctx->chunk) * ctx->world);
    CK(cudaMemcpyAsync(mine.data(), ctx->d_terms, sizeof(double) * Cloc, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if ((rc = all_gather_host(ctx, mine.data(), all.data(), sizeof(double) * ctx->chunk))) return rc;
    for (int r = 0; r < ctx->world; ++r) {
      int64_t a, b;
      dvqls_shard_range(ctx->C, r, ctx->world, &a, &b);
      std::memcpy(out + a, all.data() + size_t(r) * ctx->chunk, sizeof(double) * (b - a));
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
  int rc = launch_prefix(ctx, 1, ctx->d_theta);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out_state, ctx->d_x, sizeof(double2) * ctx->N, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DVQLS_OK;
}

int dvqls_terms_subset(dvqls_ctx* ctx, const double* theta, const int64_t* idx, int64_t count, double* out) {
  if (!ctx) return DVQLS_E_ARG;
  ctx->err.clear();
  if (int rc = check_usable(ctx)) return rc;
  if (!theta || !out || (count > 0 && !idx) || count < 0) return fail(ctx, DVQLS_E_ARG, "bad subset arguments");
  const int64_t lo = ctx->vworld > 1 ? ctx->c0 : 0, hi = ctx->vworld > 1 ? ctx->c1 : ctx->C;
  for (int64_t i = 0; i < count; ++i)
    if (idx[i] < lo || idx[i] >= hi)
      return fail(ctx, DVQLS_E_ARG, "circuit index %lld outside [%lld, %lld)", (long long)idx[i], (long long)lo,
                  (long long)hi);
  if (count == 0) return DVQLS_OK;
  if (!ctx->d_cidx || ctx->world > 1) {  // evaluate all, pick
    std::vector<double> all(size_t(ctx->C));
    int rc = dvqls_terms(ctx, theta, all.data());
    if (rc) return rc;
    for (int64_t i = 0; i < count; ++i) out[i] = all[size_t(idx[i])];
    return DVQLS_OK;
  }
  std::memcpy(ctx->h_stage, theta, sizeof(double) * ctx->P);
  CK(cudaMemcpyAsync(ctx->d_theta, ctx->h_stage, sizeof(double) * ctx->P, cudaMemcpyHostToDevice, ctx->stream));
  int rc = launch_prefix(ctx, 1, ctx->d_theta);
  if (rc) return rc;
  for (int64_t i0 = 0; i0 < count; i0 += kSubCap) {
    const int64_t m = std::min(kSubCap, count - i0);
    CK(cudaMemcpyAsync(ctx->d_cidx, idx + i0, sizeof(int64_t) * m, cudaMemcpyHostToDevice, ctx->stream));
    const int grid = int(std::min<int64_t>(ctx->grid, m));  // scratch slots
    rc = launch_hadamard(ctx, 1, 0, m, ctx->d_cidx, ctx->d_sub, grid);
    if (rc) return rc;
    CK(cudaMemcpyAsync(out + i0, ctx->d_sub, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // d_cidx / d_sub reused by the next chunk
  }
  return DVQLS_OK;
}

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

int dvqls_num_graphs(const dvqls_ctx* ctx) { return ctx ? ctx->graphs_built : DVQLS_E_ARG; }

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
  // prefix (1, or the global n > 12 prefix's passes), [planar copy of x], Hadamard kernel (+ fused
  // reduction) [, finalize after NCCL] (+ NCCL's own allreduce kernel when world > 1 without p2p)
  const int pre = ctx->pc.fn ? 1 : prefix_global_launches(ctx->n, ctx->layers);
  const bool planar = ctx->path == Path::onchip || ctx->path == Path::pstream;
  return pre + 1 + (planar ? 1 : 0) + ((ctx->world == 1 || ctx->p2p) ? 0 : 1);
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
  const int64_t T = n_circuits / 2;  // whole tasks (Re, Im circuit pairs)
  *c0 = 2 * (T * rank / world);
  *c1 = rank + 1 == world ? n_circuits : 2 * (T * (rank + 1) / world);
  return DVQLS_OK;
}

const char* dvqls_build_info(void) {
  return "libdvqls sm_100a; register-resident Hadamard-test path n=1..10, on-chip path n=11..12, "
         "global streaming path n=13..24 (uniform and Householder b); fp64 (complex128); NCCL via dlopen";
}

}  // extern "C"
