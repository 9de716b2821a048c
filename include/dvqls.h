/*
 * dvqls.h - C ABI of libdvqls.so, the B200 (sm_100a) hot path of D-VQLS
 * (arXiv 2604.14435): per cost call, evaluate all 2(n+1)L^2 Hadamard-test
 * circuits of the LCU-expanded local VQLS cost, reduce them
 * coefficient-weighted into (E, Psi), allreduce across ranks and return
 *     C = 1/2 - 1/2 * Re E / (n * Re Psi).
 *
 * Citations are PAPER.md line numbers (P:n) with section / equation /
 * algorithm, and SURVEY.md sections (§n) for readings of the paper.
 *
 *   A = sum_l c_l A_l, A_l Pauli strings            P:372-375 (Eq. 3, §II-B)
 *   E   = sum_j sum_{l,k} c_l^* c_k <x|A_l U_b Z_j U_b^+ A_k|x>
 *   Psi =       sum_{l,k} c_l^* c_k <x|A_l A_k|x>    P:380-385 (Eq. 4)
 *   each expectation = two Hadamard tests (Re, Im)
 *   x = V(theta)|0>, hardware-efficient ansatz
 *   local aggregation, Allreduce, C formula         P:389-398, Alg. 1
 *
 * Conventions (SURVEY §8(c) readings; listed in DESIGN.md):
 *   - big-endian: qubit 0 = most significant index bit; Pauli string
 *     character q acts on qubit q (reading 9);
 *   - V(theta): `layers` layers; per qubit Ry(t0), Rz(t1), Ry(t2) with
 *     t_r = theta[(layer*n + q)*3 + r]; then a CNOT ring q -> (q+1) mod n in
 *     ascending q (none for n = 1), or a CZ ring (readings 6-8);
 *     Ry(t) = exp(-i t Y/2), Rz(t) = exp(-i t Z/2);
 *   - P_j = Z_j on system qubit j; U_b applied in the numerator (readings 1-2);
 *   - Im circuit uses S^dagger after the first ancilla H: <Z_anc> = +Im (reading 10);
 *   - task t = ((l*L + k)*(n+1) + s), s = 0 denominator, s = 1+j numerator j;
 *     circuit c = 2t + part, part 0 = Re, 1 = Im (reading 17).
 *
 * Threading: a context is not thread-safe; calls on one context must be
 * serialised by the caller.  All calls return 0 on success or a negative
 * DVQLS_E_* code; the first error aborts the call and its message is
 * available from dvqls_last_error().  No CPU fallback exists: without a
 * usable sm_100 device dvqls_create fails with DVQLS_E_CUDA.
 */
#ifndef DVQLS_H
#define DVQLS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define DVQLS_OK 0
#define DVQLS_E_ARG (-1)         /* bad size, null pointer, out-of-range option          */
#define DVQLS_E_PAULI (-2)       /* Pauli character not in {I,X,Y,Z}, or duplicate string */
#define DVQLS_E_BPREP (-3)       /* | ||b|| - 1 | > 1e-8, or unknown b kind              */
#define DVQLS_E_DEGENERATE (-4)  /* Re Psi <= 1e-12 (SURVEY §8(c) reading 13)            */
#define DVQLS_E_CUDA (-5)        /* CUDA runtime error / no sm_100 device                */
#define DVQLS_E_NCCL (-6)        /* NCCL unavailable or NCCL call failed                 */
#define DVQLS_E_UNSUPPORTED (-7) /* size this build cannot evaluate                       */

/* ---- b-state preparation U_b ("fixed unitary U_b|0> = |b>") ------ */
#define DVQLS_B_UNIFORM 0    /* U_b = H^{(x)n}; |b> = uniform superposition          */
#define DVQLS_B_AMPLITUDES 1 /* U_b = w (I - 2 v v^+ / v^+ v), v = e_0 - conj(w) b,
                                w = b_0/|b_0| (1 if b_0 = 0); U_b = w I if v = 0
                                (SURVEY §8(c) reading 5).  C depends on this choice. */
typedef struct dvqls_bprep {
  int kind;            /* DVQLS_B_UNIFORM or DVQLS_B_AMPLITUDES                       */
  const double* amps;  /* AMPLITUDES: 2*2^n doubles, interleaved (re, im), host memory;
                          copied at create.  Ignored for UNIFORM.                       */
} dvqls_bprep;

/* ---- evaluation mode (dvqls_opts.mode) --------------------------------- */
#define DVQLS_MODE_CIRCUITS 0 /* every Hadamard-test circuit simulated on its own (the
                                 method as stated; the headline path)          */
#define DVQLS_MODE_PAULI 1    /* NEXT-2 algebraic fast path, FLAGGED: uniform b only.
                                 U_b Z_j U_b^+ = X_j (P:382 with U_b = H^n), every term is
                                 i^q <x|P|x> of one Pauli string P = A_l X_j A_k (or
                                 A_l A_k); each distinct P is evaluated once per theta and
                                 Re/Im share it.  Same outputs as CIRCUITS up to rounding;
                                 never reported as circuits/s.                             */

/* ---- options (all fields optional: pass NULL for defaults) ------------- */
typedef struct dvqls_opts {
  int device;                  /* CUDA device ordinal; -1 = current device              */
  int rank;                    /* this process's rank in [0, world)                      */
  int world;                   /* number of ranks (1 = single GPU)                       */
  const void* nccl_unique_id;  /* 128-byte ncclUniqueId, identical on all ranks; required
                                  when world > 1 (see dvqls_nccl_unique_id)              */
  int entangler;               /* 0 = CNOT ring (default), 1 = CZ ring                   */
  void* cuda_stream;           /* cudaStream_t for all device work; NULL = library-owned */
  int timing;                  /* nonzero: record CUDA events around each kernel         */
  int max_batch;               /* largest K accepted by the *_batch calls (default 16)   */
  int mode;                    /* DVQLS_MODE_CIRCUITS (0, default) or DVQLS_MODE_PAULI   */
  void* workspace_dev;         /* NULL: the library cudaMallocs its device tables once, in
                                  dvqls_create.  Else: caller-owned device memory (e.g. a
                                  torch tensor) of workspace_bytes >= dvqls_workspace_size(),
                                  256-byte aligned; every per-context device buffer is carved
                                  from it (the IPC-shared 4-double-per-theta allreduce buffer
                                  of world > 1 is the one exception: IPC needs its own
                                  allocation).  It must outlive the context.               */
  size_t workspace_bytes;      /* size of workspace_dev                                   */
  /* ---- fields below: zero selects the default ------------------------------------------- */
  int virtual_rank;            /* with virtual_world > 1 (and world == 1): evaluate only block
                                  virtual_rank of a virtual_world-way split of the circuits on
                                  this one GPU (the sharding of P:394 / SURVEY §8(e) run as one
                                  virtual rank; the single-GPU weak-scaling reference).  Cost
                                  calls then return this block's PARTIAL (E, Psi) and C = NaN (no
                                  DVQLS_E_DEGENERATE); the caller sums the partials in rank order.
                                  dvqls_terms writes only out[c0, c1).                         */
  int virtual_world;           /* 0 or 1: off                                                  */
  int allreduce;               /* world > 1: DVQLS_ALLREDUCE_P2P (0, default): the fused NVLink
                                  reduction in the Hadamard kernel's tail (falls back to NCCL if a
                                  peer buffer cannot be mapped and a communicator exists);
                                  DVQLS_ALLREDUCE_NCCL (1): ncclAllReduce + a finalize kernel     */
  int p2p_timeout_ms;          /* fused reduction: how long a rank waits for its peers (0 =
                                  60000).  On expiry the call returns DVQLS_E_NCCL and the context
                                  refuses further evaluations (destroy and recreate it).        */
  int (*host_allgather)(void* user, const void* send, void* recv, size_t bytes);
                               /* world > 1 WITHOUT nccl_unique_id: the caller's allgather of
                                  `bytes` bytes per rank (recv = world * bytes, rank order; return 0
                                  on success), e.g. over torch.distributed/gloo.  Used only at
                                  create (IPC handles of the fused reduction; every rank must map
                                  every peer, else DVQLS_E_NCCL) and by dvqls_terms (term slices).
                                  No NCCL communicator is created; ranks may share one GPU.     */
  void* host_allgather_user;   /* passed back to host_allgather                                */
  int graphs;                  /* 0: capture each (K, buffers) launch sequence of the cost path in
                                  a CUDA graph on first use and replay it (default, only when
                                  timing == 0 and the reduction is not NCCL); -1: plain launches */
  int pdl;                     /* 0: programmatic dependent launch of the n <= 10 Hadamard kernel
                                  behind the prefix (default, timing == 0 only); -1: off       */
  int stage;                   /* n >= 13 uniform b: TMA staging of streaming tiles. 0 = from
                                  n = 16 (default), -1 = off, 1 = from n = 13                   */
  int stream_grid;             /* n >= 11: cap on the CTAs of the streaming kernels (0 = one wave) */
  int variant;                 /* kernel variant for n = 10, uniform b: 0 = default (= 2), 1 = one
                                  circuit per warp (plane_kernel), 2 = two circuits in flight per
                                  warp, skewed phases (plane2_kernel; measured 0.6-1.5 % faster).
                                  Bitwise-identical terms; (E, Psi) equal to rounding.          */
  int prefix;                  /* V(theta)|0> for 7 <= n <= 10: 0 = one CTA per theta (default);
                                  1 = a thread-block cluster of 2^(n-7) CTAs per theta joined by
                                  DSMEM (measured no faster on B200: DESIGN.md §6)              */
} dvqls_opts;

#define DVQLS_ALLREDUCE_P2P 0
#define DVQLS_ALLREDUCE_NCCL 1

typedef struct dvqls_ctx dvqls_ctx;

/* Device bytes a context with these parameters carves from opts->workspace_dev (SURVEY §8(b):
 * the workspace is allocated by the caller, e.g. torch, so the library does no cudaMalloc
 * for its tables).  Same rules as dvqls_create for n, layers, n_terms and opts (rank, world,
 * max_batch, mode, device); for DVQLS_MODE_PAULI the bound assumes every task has its own
 * observable.  Needs the device (kernel occupancy decides grid-sized buffers).  Returns 0 on
 * invalid arguments or without a usable device. */
size_t dvqls_workspace_size(int n_qubits, int layers, int n_terms, const dvqls_opts* opts);

/* Build a context: parse the L Pauli strings into
 * (x_mask, z_mask, n_Y), copy coefficients, build U_b data, allocate device
 * buffers (the only cudaMalloc calls of the library; none when opts->workspace_dev
 * supplies the memory, see dvqls_workspace_size), pick this rank's
 * contiguous block of whole tasks [c0, c1) (dvqls_shard_range) of the
 * C = 2(n+1)L^2 circuits ("strided workload allocation"; a contiguous
 * block balances equally) and, for world > 1, create the NCCL
 * communicator.  Collective over all ranks when world > 1.
 *   n_qubits    system qubits n, 1 <= n <= 24 (n <= 10: register path; 11..12: SMEM
 *               tile path; 13..24: global streaming path; both U_b kinds at every n)
 *   layers      ansatz depth d >= 1; theta has P = 3*n*layers doubles
 *   n_terms     L >= 1
 *   pauli_terms L*n characters, row-major (term l at pauli_terms + l*n)
 *   coeffs      2*L doubles, interleaved (re, im) of c_l
 * Inputs are copied; the caller may free them on return. */
int dvqls_create(dvqls_ctx** out, int n_qubits, int layers, int n_terms,
                 const char* pauli_terms, const double* coeffs,
                 const dvqls_bprep* b_prep, const dvqls_opts* opts);

/* Free all device and host resources (safe on NULL). */
void dvqls_destroy(dvqls_ctx* ctx);

/* Term expectations of one theta (host buffers; synchronous).
 *   theta        P doubles (host)
 *   out_expvals  2(n+1)L^2 doubles (host), canonical order, index 2t + part;
 *                every rank receives the full array (allgather over NCCL). */
int dvqls_terms(dvqls_ctx* ctx, const double* theta, double* out_expvals);

/* Cost of one theta (host buffers; synchronous): the whole hot path
 * (prefix -> circuits -> weighted reduction -> allreduce -> C).
 *   out_cost   1 double
 *   out_E_Psi  NULL or 4 doubles: Re E, Im E, Re Psi, Im Psi (global sums)
 * Returns DVQLS_E_DEGENERATE (out_cost = NaN) if Re Psi <= 1e-12. */
int dvqls_cost(dvqls_ctx* ctx, const double* theta, double* out_cost, double* out_E_Psi);

/* K independent thetas in one pass (FD / parameter-shift points), host buffers.
 *   thetas     K*P doubles, row-major;  1 <= K <= opts.max_batch
 *   out_costs  K doubles;  out_E_Psi NULL or 4*K doubles
 * Degenerate entries get NaN and the call returns DVQLS_E_DEGENERATE.
 * One CUDA graph launch per call: the inputs are copied into the context's mapped pinned stage;
 * on a single rank the kernels read theta from it and write the results into it (no copy
 * nodes), across ranks theta goes H2D and the results (with the error word) D2H inside the
 * graph.  dvqls_cost is this call with K = 1. */
int dvqls_cost_batch(dvqls_ctx* ctx, int K, const double* thetas, double* out_costs,
                     double* out_E_Psi);

/* Parameter-shift gradient (NEXT-1 with 2P shift points; SURVEY §8(c) reading 23): every
 * parameter enters V(theta) through one exp(-i theta sigma/2), so each Hadamard-test value, and
 * Re E, Re Psi, satisfy df/dtheta_p = [f(theta + pi/2 e_p) - f(theta - pi/2 e_p)] / 2 exactly;
 *     dC/dtheta_p = -(dReE_p Re Psi - Re E dRePsi_p) / (2 n Re Psi^2).
 * The 2P shifted thetas and theta are built on the device and evaluated through the circuit path
 * in batches of max_batch (every circuit simulated: 2P + 1 cost evaluations per gradient).
 *   theta      P doubles (host)
 *   out_cost   1 double: C(theta);  out_grad P doubles;  out_E_Psi NULL or 4 doubles at theta
 * Returns DVQLS_E_DEGENERATE (NaN outputs) if Re Psi(theta) <= 1e-12. */
int dvqls_cost_grad(dvqls_ctx* ctx, const double* theta, double* out_cost, double* out_grad, double* out_E_Psi);

/* Device-resident parameter-shift gradient, asynchronous on the context stream.
 *   theta_dev  P doubles (device);  out_dev 1 + P + 4 doubles (device): C, dC/dtheta[P], E, Psi */
int dvqls_cost_grad_dev(dvqls_ctx* ctx, const double* theta_dev, double* out_dev);

/* Synchronise the context stream and report asynchronous failures of the _dev calls: returns
 * DVQLS_E_NCCL if a fused-allreduce peer timed out (the context is then unusable), DVQLS_E_CUDA on
 * a CUDA error, else DVQLS_OK. */
int dvqls_check(dvqls_ctx* ctx);

/* Device-resident variant: asynchronous on the context stream, no host sync.
 *   thetas_dev  K*P doubles in device memory
 *   out_dev     5*K doubles in device memory: per theta (C, Re E, Im E, Re Psi, Im Psi);
 *               C = NaN when Re Psi <= 1e-12.
 * Caller synchronises the stream (dvqls_stream) before reading out_dev. */
int dvqls_cost_dev(dvqls_ctx* ctx, int K, const double* thetas_dev, double* out_dev);

/* NEXT-3: local AND global cost (Eq. 1) of K thetas, device-resident, async.
 * C_G = 1 - |sum_l c_l beta_l|^2 / Re Psi with beta_l = <b|A_l|x> from the 2L overlap
 * Hadamard tests (ancilla-controlled V, A_l, U_b^+; Re and Im circuits) and Re Psi the
 * local cost's denominator sum (global over ranks) of the same call.
 *   out6_dev  6*K doubles: per theta (C_L, Re E, Im E, Re Psi, Im Psi, C_G); C = NaN when
 *             Re Psi <= 1e-12
 *   beta_dev  NULL or 2*L*K doubles: per theta and l, (Re, Im) beta_l */
int dvqls_costs_dev(dvqls_ctx* ctx, int K, const double* thetas_dev, double* out6_dev, double* beta_dev);

/* Host-buffer variant of dvqls_costs_dev for one theta (synchronous).
 *   out6      6 doubles (C_L, Re E, Im E, Re Psi, Im Psi, C_G)
 *   out_beta  NULL or 2*L doubles
 * Returns DVQLS_E_DEGENERATE if Re Psi <= 1e-12. */
int dvqls_global_cost(dvqls_ctx* ctx, const double* theta, double* out6, double* out_beta);

/* Device-resident terms of THIS rank's block [c0, c1) for one theta (async).
 *   out_dev  (c1 - c0) doubles in device memory */
int dvqls_terms_local_dev(dvqls_ctx* ctx, const double* theta_dev, double* out_dev);

/* Solution state |x(theta)> = V(theta)|0> (Alg. 1 Step 5), computed by the
 * prefix kernel and copied to the host.
 *   out_state  2*2^n doubles, interleaved (re, im), big-endian index order. */
int dvqls_state(dvqls_ctx* ctx, const double* theta, double* out_state);

/* Term expectations of a subset of circuits (testing at large n, where evaluating all
 * 2(n+1)L^2 circuits takes minutes).  Synchronous; single-rank contexts of the streaming path
 * (n >= 13, or Householder b at n = 11, 12) evaluate only the listed circuits (in launches of at
 * most 4096, from buffers planned in the workspace), other contexts evaluate all and select.
 * Virtual-rank contexts accept only indices inside their block.
 *   idx   count circuit indices in [0, 2(n+1)L^2), host memory
 *   out   count doubles, out[i] = <Z_anc> of circuit idx[i] */
int dvqls_terms_subset(dvqls_ctx* ctx, const double* theta, const int64_t* idx, int64_t count, double* out);

/* ---- NEXT-4: Pauli decomposition + pruning on the GPU (no context) ------
 * Alg. 1 Steps 1-2 (FWHT-based decomposition P:379, pruning below 1 % of the l2
 * norm P:490):  c_P = tr(P A)/2^n for all 4^n Pauli strings P, then keep |c| >= 1e-14 and
 * |c| >= eps * ||c||_2 (inclusive), ordered by descending |c| (magnitudes within
 * 1e-12 * ||c||_2 tie) then lexicographically with I < X < Y < Z (SURVEY §8(c) reading 15).
 *   n            1..13 (A is 2^n x 2^n; 1 GB of complex128 at n = 13)
 *   A            2^n * 2^n complex, row-major, interleaved (re, im), HOST memory (copied)
 *   eps          0 <= eps < 1
 *   max_terms    capacity of out_paulis (max_terms*n chars) and out_coeffs (2*max_terms doubles)
 *   out_L        number of surviving terms (set even when it exceeds max_terms: DVQLS_E_ARG)
 *   out_norm     NULL or ||c||_2
 *   device       CUDA device ordinal, -1 = current
 *   out_ms       NULL or device milliseconds of transform + pruning + sort (CUDA events,
 *                after the host-to-device copy of A; ||A||_F^2 is summed chunk by chunk during
 *                that copy and is not in out_ms)
 * The output feeds dvqls_create (pauli_terms, coeffs) directly.  Synchronous; allocates its
 * own device buffers (16 * 4^n bytes for A, plus the candidates).  One pass over the XOR
 * diagonals of A: candidates above eps * ||A||_F / 2^{n/2} * (1 - 1e-9) (Parseval) are kept, then
 * filtered with the exact ||c||_2 = sqrt(sum |c|^2) and ordered in one CTA (<= 4096 candidates)
 * or, beyond that, by a second candidate pass into buffers of the counted size and a global
 * bitonic sort (same order).
 * Errors: dvqls_decompose_error(). */
int dvqls_decompose(int n, const double* A, double eps, int64_t max_terms, char* out_paulis,
                    double* out_coeffs, int64_t* out_L, double* out_norm, int device, float* out_ms);
/* All 4^n coefficients, out_coeffs[2 * (m * 2^n + z) + {0,1}] = c_{P(m, z)} with x-mask m and
 * z-mask z (big-endian bits; character q <-> bit n-1-q), same transform as dvqls_decompose. */
int dvqls_pauli_coefficients(int n, const double* A, double* out_coeffs, int device);
const char* dvqls_decompose_error(void);

/* ---- introspection ------------------------------------------------------ */
const char* dvqls_last_error(const dvqls_ctx* ctx); /* "" if none; static text if ctx NULL */
int64_t dvqls_num_circuits(const dvqls_ctx* ctx);   /* 2(n+1)L^2 */
int dvqls_local_range(const dvqls_ctx* ctx, int64_t* c0, int64_t* c1);
void* dvqls_stream(const dvqls_ctx* ctx);           /* the cudaStream_t in use */
/* CTAs of the Hadamard-test kernel per theta (the n >= 13 streaming path: in total over the
 * batch, one 2^n-amplitude scratch each). */
int dvqls_launch_grid(const dvqls_ctx* ctx);
/* DVQLS_MODE_PAULI: number of distinct Pauli observables among the (n+1)L^2 tasks
 * (0 in CIRCUITS mode). */
int64_t dvqls_num_observables(const dvqls_ctx* ctx);
/* Pure host helper (no device access), NEXT-2 algebra: the observable of task (l, k, s) for
 * uniform b, B = A_l X_j A_k (s = 1 + j) or A_l A_k (s = 0), as
 *     B|i> = i^phase (-1)^{popcount(i & z_mask)} |i ^ x_mask>   (big-endian bits).
 *   pauli_l, pauli_k  n characters each from {I,X,Y,Z}
 * Returns DVQLS_E_ARG / DVQLS_E_PAULI on bad input. */
int dvqls_task_observable(int n, const char* pauli_l, const char* pauli_k, int s, uint32_t* x_mask,
                          uint32_t* z_mask, int* phase);
/* CUDA graphs instantiated so far by this context (one per (K, buffers) of the cost path). */
int dvqls_num_graphs(const dvqls_ctx* ctx);
/* Kernel launches per cost evaluation call (prefix + circuits + reduce [+ finalize]). */
int dvqls_launches_per_call(const dvqls_ctx* ctx);
/* With opts.timing: device milliseconds of the last call, measured with CUDA events
 * on the context stream: ms[0] prefix, ms[1] Hadamard-test kernel, ms[2] reduction
 * (+ allreduce + finalize), ms[3] whole call.  Returns DVQLS_E_ARG if timing is off. */
int dvqls_last_timings(const dvqls_ctx* ctx, float* ms4);
/* Pure host helper (no device access): the contiguous circuit block a rank evaluates, in whole
 * tasks (the Re and Im circuits 2t, 2t+1 of a task stay together; P:394 allocates tasks):
 *     [c0, c1) = [2 floor(T*rank/world), 2 floor(T*(rank+1)/world)),  T = floor(C/2),
 * the last rank also taking circuit C-1 when C is odd.  Blocks of consecutive ranks tile [0, C)
 * and differ in size by at most 2 (3 with an odd C). */
int dvqls_shard_range(int64_t n_circuits, int rank, int world, int64_t* c0, int64_t* c1);
/* Write a fresh 128-byte ncclUniqueId into out128 (rank 0 calls, then broadcasts). */
int dvqls_nccl_unique_id(void* out128);
/* Static build description (arch, supported n range). */
const char* dvqls_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* DVQLS_H */
