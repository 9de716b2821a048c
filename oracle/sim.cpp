// ORACLE - TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously correct CPU state-vector simulator of the D-VQLS
// Hadamard-test circuits (arXiv 2604.14435).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares no code with the CUDA product path (paper_2604_14435_b200/).
//
// What it computes, gate by gate, following SURVEY.md §8(c) "Plain definition":
//   register of n+1 qubits, ancilla = qubit 0 (most significant index bit),
//   system qubit q = register qubit q+1, big-endian (qubit 0 = MSB).
//   1. |0...0>
//   2. V(theta) on the system qubits: d layers; per qubit Ry, Rz, Ry with
//      theta[(layer*n + q)*3 + r]; then a CNOT ring q -> (q+1) mod n in
//      ascending q (none for n = 1) or a CZ ring (
//      SURVEY §8(c) readings 6-8).  Ry(t) = exp(-i t Y/2), Rz(t) = exp(-i t Z/2).
//   3. H(anc); for the Im circuit S^dagger(anc) (reading 10).
//   4. controlled A_k: one controlled X/Y/Z per non-identity factor.
//   5. numerator tasks (s >= 1): controlled U_b^dagger, controlled Z_j,
//      controlled U_b (Eq. 4; reading 2).  U_b = H^{(x)n} (uniform)
//      or the Householder completion U_b = w(I - 2 v v^+/v^+v) (reading 5), applied as the
//      dense 2^n x 2^n matrix for n <= 12 and, for n > 12 (a dense matrix would take
//      4^n * 16 B), from its definition as psi -> w (psi - 2 v (v^+ psi) / v^+ v), the same
//      operator (pinned against the dense matrix in tests/test_oracle_sim.py).
//   6. controlled A_l (A_l^dagger = A_l for Pauli strings).
//   7. H(anc); 8. <Z_anc> = sum|psi_{anc=0}|^2 - sum|psi_{anc=1}|^2.
// Task t = ((l*L + k)*(n+1) + s), s = 0 denominator, s = 1+j numerator j;
// circuit c = 2t + part, part 0 = Re, 1 = Im (SURVEY §8 notation, reading 17).
//
// Every gate is one full pass over the 2^(n+1) amplitudes; no fusion, no
// blocking, no SIMD intrinsics.  The only parallelism is independent circuits
// on std::thread workers.

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

using cplx = std::complex<double>;
using State = std::vector<cplx>;

struct Gate2 {
  cplx u00, u01, u10, u11;
};

// bit position of register qubit q in an m-qubit big-endian index
inline int bitpos(int m, int q) { return m - 1 - q; }

// single-qubit gate U on qubit q
void apply_1q(State& psi, int m, int q, const Gate2& U) {
  const size_t s = size_t(1) << bitpos(m, q);
  for (size_t i = 0; i < psi.size(); ++i) {
    if (i & s) continue;
    cplx a = psi[i], b = psi[i | s];
    psi[i] = U.u00 * a + U.u01 * b;
    psi[i | s] = U.u10 * a + U.u11 * b;
  }
}

// single-qubit gate U on qubit q, controlled on qubit c being |1>
void apply_c1q(State& psi, int m, int c, int q, const Gate2& U) {
  const size_t s = size_t(1) << bitpos(m, q);
  const size_t cm = size_t(1) << bitpos(m, c);
  for (size_t i = 0; i < psi.size(); ++i) {
    if ((i & s) || !(i & cm)) continue;
    cplx a = psi[i], b = psi[i | s];
    psi[i] = U.u00 * a + U.u01 * b;
    psi[i | s] = U.u10 * a + U.u11 * b;
  }
}

// single-qubit gate U on qubit q, controlled on qubits c1 and c2 both being |1>
void apply_cc1q(State& psi, int m, int c1, int c2, int q, const Gate2& U) {
  const size_t s = size_t(1) << bitpos(m, q);
  const size_t cm = (size_t(1) << bitpos(m, c1)) | (size_t(1) << bitpos(m, c2));
  for (size_t i = 0; i < psi.size(); ++i) {
    if ((i & s) || (i & cm) != cm) continue;
    cplx a = psi[i], b = psi[i | s];
    psi[i] = U.u00 * a + U.u01 * b;
    psi[i | s] = U.u10 * a + U.u11 * b;
  }
}

// controlled dense unitary U (2^n x 2^n, row-major) on system qubits 1..n,
// control = ancilla (qubit 0, the MSB): acts on the anc=1 half only.
void apply_c_dense(State& psi, int n, const std::vector<cplx>& U) {
  const size_t N = size_t(1) << n;
  std::vector<cplx> out(N);
  for (size_t r = 0; r < N; ++r) {
    cplx acc = 0;
    for (size_t c = 0; c < N; ++c) acc += U[r * N + c] * psi[N + c];
    out[r] = acc;
  }
  for (size_t r = 0; r < N; ++r) psi[N + r] = out[r];
}

const double kInvSqrt2 = 0.70710678118654752440;
const Gate2 kH{kInvSqrt2, kInvSqrt2, kInvSqrt2, -kInvSqrt2};
const Gate2 kX{0, 1, 1, 0};
const Gate2 kY{0, cplx(0, -1), cplx(0, 1), 0};
const Gate2 kZ{1, 0, 0, -1};
const Gate2 kSdg{1, 0, 0, cplx(0, -1)};

Gate2 Ry(double t) {
  double c = std::cos(t / 2), s = std::sin(t / 2);
  return Gate2{c, -s, s, c};
}
Gate2 Rz(double t) {
  return Gate2{std::exp(cplx(0, -t / 2)), 0, 0, std::exp(cplx(0, t / 2))};
}

struct Problem {
  int n = 0, layers = 0, L = 0, entangler = 0, bkind = 0;
  std::vector<std::string> paulis;  // L strings of n chars
  std::vector<cplx> Ub, Ubdg;       // dense U_b, U_b^dagger (amplitude b, dense form)
  std::vector<cplx> hv;             // Householder v = e_0 - conj(w) b (amplitude b)
  cplx hw = 1.0;                    // Householder phase w
  double hvv = 0.0;                 // v^+ v
  bool dense = true;                // U_b applied as the dense matrix (else from v, w)
};

// Householder form of the oracle (test hook): 0 = dense for n <= 12, definition form above;
// 1 = definition form at every n; 2 = dense at every n <= 12
int g_hh_form = 0;

// controlled U_b (or U_b^dagger) = w (I - 2 v v^+ / v^+ v) on the anc = 1 half, from its
// definition: psi_1 -> w' (psi_1 - (2 / v^+ v) v (v^+ psi_1)), w' = w (U_b) or conj(w) (U_b^dagger:
// the reflector is Hermitian).  U_b = w I when v = 0.
void apply_c_householder(State& psi, const Problem& P, bool dagger) {
  const size_t N = size_t(1) << P.n;
  const cplx wf = dagger ? std::conj(P.hw) : P.hw;
  cplx d = 0;
  for (size_t i = 0; i < N; ++i) d += std::conj(P.hv[i]) * psi[N + i];
  const cplx f = P.hvv > 0 ? 2.0 * d / P.hvv : cplx(0, 0);
  for (size_t i = 0; i < N; ++i) psi[N + i] = wf * (psi[N + i] - f * P.hv[i]);
}

// V(theta) on system qubits (register qubits offset+0 .. offset+n-1)
void apply_ansatz(State& psi, int m, int offset, const Problem& P, const double* theta) {
  const int n = P.n;
  for (int layer = 0; layer < P.layers; ++layer) {
    for (int q = 0; q < n; ++q) {
      const double* t = theta + (layer * n + q) * 3;
      apply_1q(psi, m, offset + q, Ry(t[0]));
      apply_1q(psi, m, offset + q, Rz(t[1]));
      apply_1q(psi, m, offset + q, Ry(t[2]));
    }
    if (n >= 2) {
      for (int q = 0; q < n; ++q) {
        int c = offset + q, tq = offset + (q + 1) % n;
        apply_c1q(psi, m, c, tq, P.entangler == 0 ? kX : kZ);
      }
    }
  }
}

// V(theta) on the system qubits (register qubits 1..n), every gate controlled on the ancilla
// (qubit 0): c-Ry, c-Rz, c-Ry per qubit, the ring as Toffoli (CNOT) or CCZ (CZ) gates.
void apply_controlled_ansatz(State& psi, const Problem& P, const double* theta) {
  const int n = P.n, m = n + 1;
  for (int layer = 0; layer < P.layers; ++layer) {
    for (int q = 0; q < n; ++q) {
      const double* t = theta + (layer * n + q) * 3;
      apply_c1q(psi, m, 0, q + 1, Ry(t[0]));
      apply_c1q(psi, m, 0, q + 1, Rz(t[1]));
      apply_c1q(psi, m, 0, q + 1, Ry(t[2]));
    }
    if (n >= 2)
      for (int q = 0; q < n; ++q) apply_cc1q(psi, m, 0, q + 1, (q + 1) % n + 1, P.entangler == 0 ? kX : kZ);
  }
}

const Gate2& pauli_gate(char ch) {
  switch (ch) {
    case 'X': return kX;
    case 'Y': return kY;
    default: return kZ;
  }
}

void apply_controlled_pauli_string(State& psi, int m, const std::string& p) {
  for (size_t q = 0; q < p.size(); ++q)
    if (p[q] != 'I') apply_c1q(psi, m, 0, int(q) + 1, pauli_gate(p[q]));
}

void apply_controlled_Ub(State& psi, const Problem& P, bool dagger) {
  const int m = P.n + 1;
  if (P.bkind == 0) {
    for (int q = 0; q < P.n; ++q) apply_c1q(psi, m, 0, q + 1, kH);
  } else if (P.dense) {
    apply_c_dense(psi, P.n, dagger ? P.Ubdg : P.Ub);
  } else {
    apply_c_householder(psi, P, dagger);
  }
}

double expect_z_anc(const State& psi) {
  const size_t half = psi.size() / 2;
  double p0 = 0, p1 = 0;
  for (size_t i = 0; i < half; ++i) p0 += std::norm(psi[i]);
  for (size_t i = half; i < psi.size(); ++i) p1 += std::norm(psi[i]);
  return p0 - p1;
}

// One Hadamard-test circuit (§8(c) steps 1-8).  `prefix`, if non-null, is the
// (n+1)-qubit state after step 2 (bitwise identical to recomputing it).
double hadamard_test(const Problem& P, const double* theta, const State* prefix, int64_t circuit) {
  const int n = P.n, m = n + 1, L = P.L;
  const int64_t t = circuit / 2;
  const int part = int(circuit % 2);
  const int s = int(t % (n + 1));
  const int k = int((t / (n + 1)) % L);
  const int l = int(t / (int64_t(n + 1) * L));

  State psi;
  if (prefix) {
    psi = *prefix;
  } else {
    psi.assign(size_t(1) << m, 0);
    psi[0] = 1;
    apply_ansatz(psi, m, 1, P, theta);
  }
  apply_1q(psi, m, 0, kH);
  if (part == 1) apply_1q(psi, m, 0, kSdg);
  apply_controlled_pauli_string(psi, m, P.paulis[k]);
  if (s >= 1) {
    const int j = s - 1;
    apply_controlled_Ub(psi, P, /*dagger=*/true);
    apply_c1q(psi, m, 0, j + 1, kZ);
    apply_controlled_Ub(psi, P, /*dagger=*/false);
  }
  apply_controlled_pauli_string(psi, m, P.paulis[l]);
  apply_1q(psi, m, 0, kH);
  return expect_z_anc(psi);
}

// Global-cost overlap Hadamard test (NEXT-3; Eq. 1): Re (part 0) or Im (part 1)
// of beta_l = <0| U_b^+ A_l V(theta) |0> = <b| A_l |x>, gate by gate on n+1 qubits:
// |0..0>, H(anc), [S^+(anc)], controlled V(theta), controlled A_l, controlled U_b^+, H(anc),
// <Z_anc>.  (The |0> branch keeps |0^n>; the |1> branch carries U_b^+ A_l V|0>.)
double overlap_test(const Problem& P, const double* theta, int l, int part) {
  const int n = P.n, m = n + 1;
  State psi(size_t(1) << m, 0);
  psi[0] = 1;
  apply_1q(psi, m, 0, kH);
  if (part == 1) apply_1q(psi, m, 0, kSdg);
  apply_controlled_ansatz(psi, P, theta);
  apply_controlled_pauli_string(psi, m, P.paulis[l]);
  apply_controlled_Ub(psi, P, /*dagger=*/true);
  apply_1q(psi, m, 0, kH);
  return expect_z_anc(psi);
}

// Dense U_b = w (I - 2 v v^+ / v^+ v), v = e_0 - conj(w) b, w = b_0/|b_0|
// (w = 1 if b_0 = 0; U_b = w I if v = 0).  SURVEY §8(c) reading 5.
void build_householder(Problem& P, const double* b_amps) {
  const size_t N = size_t(1) << P.n;
  std::vector<cplx> b(N);
  for (size_t i = 0; i < N; ++i) b[i] = cplx(b_amps[2 * i], b_amps[2 * i + 1]);
  cplx w = std::abs(b[0]) > 0 ? b[0] / std::abs(b[0]) : cplx(1, 0);
  std::vector<cplx> v(N);
  for (size_t i = 0; i < N; ++i) v[i] = (i == 0 ? cplx(1, 0) : cplx(0, 0)) - std::conj(w) * b[i];
  double vv = 0;
  for (size_t i = 0; i < N; ++i) vv += std::norm(v[i]);
  P.hv = v;
  P.hw = w;
  P.hvv = vv;
  P.dense = g_hh_form == 2 || (g_hh_form == 0 && P.n <= 12);
  if (!P.dense) return;
  P.Ub.assign(N * N, 0);
  P.Ubdg.assign(N * N, 0);
  for (size_t r = 0; r < N; ++r)
    for (size_t c = 0; c < N; ++c) {
      cplx h = (r == c ? cplx(1, 0) : cplx(0, 0));
      if (vv > 0) h -= 2.0 * v[r] * std::conj(v[c]) / vv;
      P.Ub[r * N + c] = w * h;
    }
  for (size_t r = 0; r < N; ++r)
    for (size_t c = 0; c < N; ++c) P.Ubdg[r * N + c] = std::conj(P.Ub[c * N + r]);
}

int build_problem(Problem& P, int n, int layers, int L, const char* paulis, int entangler,
                  int bkind, const double* b_amps) {
  if (n < 1 || n > 24 || layers < 1 || L < 1 || !paulis) return -1;
  if (bkind == 1 && !b_amps) return -1;
  if (bkind == 1 && g_hh_form == 2 && n > 12) return -1;
  P.n = n; P.layers = layers; P.L = L; P.entangler = entangler; P.bkind = bkind;
  P.paulis.resize(L);
  for (int l = 0; l < L; ++l) {
    P.paulis[l].assign(paulis + size_t(l) * n, size_t(n));
    for (char ch : P.paulis[l])
      if (ch != 'I' && ch != 'X' && ch != 'Y' && ch != 'Z') return -2;
  }
  if (bkind == 1) build_householder(P, b_amps);
  return 0;
}

}  // namespace

extern "C" {

// x = V(theta)|0^n>, written as 2*2^n interleaved doubles.
int oracle_ansatz_state(int n, int layers, int entangler, const double* theta, double* out) {
  Problem P;
  P.n = n; P.layers = layers; P.entangler = entangler;
  if (n < 1 || n > 24 || layers < 1) return -1;
  State psi(size_t(1) << n, 0);
  psi[0] = 1;
  apply_ansatz(psi, n, 0, P, theta);
  for (size_t i = 0; i < psi.size(); ++i) {
    out[2 * i] = psi[i].real();
    out[2 * i + 1] = psi[i].imag();
  }
  return 0;
}

// Expectation values <Z_anc> of the requested circuits (all 2(n+1)L^2 when
// idx == NULL, else idx[0..count)), in that order.
// mode 0 = faithful (V(theta) re-simulated per circuit, the paper's model);
// mode 1 = prefix-shared (the state after step 2 computed once and copied).
int oracle_terms(int n, int layers, int L, const char* paulis, int entangler, int bkind,
                 const double* b_amps, const double* theta, int mode, int nthreads,
                 const int64_t* idx, int64_t count, double* out) {
  Problem P;
  int rc = build_problem(P, n, layers, L, paulis, entangler, bkind, b_amps);
  if (rc) return rc;
  const int64_t total = 2 * int64_t(n + 1) * L * L;
  if (!idx) count = total;
  for (int64_t i = 0; idx && i < count; ++i)
    if (idx[i] < 0 || idx[i] >= total) return -3;

  State prefix;
  if (mode == 1) {
    const int m = n + 1;
    prefix.assign(size_t(1) << m, 0);
    prefix[0] = 1;
    apply_ansatz(prefix, m, 1, P, theta);
  }
  if (nthreads < 1) nthreads = int(std::thread::hardware_concurrency());
  if (nthreads < 1) nthreads = 1;
  if (int64_t(nthreads) > count) nthreads = int(count > 0 ? count : 1);
  std::vector<std::thread> pool;
  for (int w = 0; w < nthreads; ++w) {
    pool.emplace_back([&, w]() {
      const int64_t lo = count * w / nthreads, hi = count * (w + 1) / nthreads;
      for (int64_t i = lo; i < hi; ++i) {
        const int64_t c = idx ? idx[i] : i;
        out[i] = hadamard_test(P, theta, mode == 1 ? &prefix : nullptr, c);
      }
    });
  }
  for (auto& th : pool) th.join();
  return 0;
}

// NEXT-3: the 2L overlap Hadamard tests, out[2l + part] = Re / Im <b|A_l|x>.
int oracle_overlap_terms(int n, int layers, int L, const char* paulis, int entangler, int bkind,
                         const double* b_amps, const double* theta, int nthreads, double* out) {
  Problem P;
  int rc = build_problem(P, n, layers, L, paulis, entangler, bkind, b_amps);
  if (rc) return rc;
  const int64_t count = 2 * int64_t(L);
  if (nthreads < 1) nthreads = int(std::thread::hardware_concurrency());
  if (nthreads < 1) nthreads = 1;
  if (int64_t(nthreads) > count) nthreads = int(count);
  std::vector<std::thread> pool;
  for (int w = 0; w < nthreads; ++w) {
    pool.emplace_back([&, w]() {
      const int64_t lo = count * w / nthreads, hi = count * (w + 1) / nthreads;
      for (int64_t i = lo; i < hi; ++i) out[i] = overlap_test(P, theta, int(i / 2), int(i % 2));
    });
  }
  for (auto& th : pool) th.join();
  return 0;
}

// Dense U_b (row-major, interleaved complex) for inspection/tests.
int oracle_ub_matrix(int n, int bkind, const double* b_amps, double* out) {
  Problem P;
  P.n = n; P.bkind = bkind;
  const size_t N = size_t(1) << n;
  if (bkind == 1) {
    if (n > 12) return -1;
    const int keep = g_hh_form;
    g_hh_form = 2;
    build_householder(P, b_amps);
    g_hh_form = keep;
    for (size_t i = 0; i < N * N; ++i) {
      out[2 * i] = P.Ub[i].real();
      out[2 * i + 1] = P.Ub[i].imag();
    }
    return 0;
  }
  // H^{(x)n} via the simulator itself: column c = H^{(x)n}|c>
  for (size_t c = 0; c < N; ++c) {
    State psi(N, 0);
    psi[c] = 1;
    for (int q = 0; q < n; ++q) apply_1q(psi, n, q, kH);
    for (size_t r = 0; r < N; ++r) {
      out[2 * (r * N + c)] = psi[r].real();
      out[2 * (r * N + c) + 1] = psi[r].imag();
    }
  }
  return 0;
}

int oracle_hardware_threads(void) { return int(std::thread::hardware_concurrency()); }

// test hook: form of the Householder U_b (0 auto, 1 definition form, 2 dense); returns the old one
int oracle_set_householder_form(int form) {
  const int old = g_hh_form;
  if (form >= 0 && form <= 2) g_hh_form = form;
  return old;
}

}  // extern "C"
