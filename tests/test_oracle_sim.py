"""Pins for the gate-by-gate oracle simulator (oracle/sim.cpp) - CPU only.

Each Hadamard-test value is checked against something other than itself:
dense quadratic forms <x|B|x> with B = A_l U_b Z_j U_b^+ A_k built from full
matrices (Eq. 4), the closed-form Pauli expectation (uniform b:
U_b Z_j U_b^+ = X_j), SPEC.md worked examples and invariants.
"""

import numpy as np
import pytest

from dvqls_inputs import configs, seeds
from oracle import dense, sim


# --- ansatz V(theta) -------------------------------------

def test_ansatz_zero_params_is_identity():
    for n in (1, 2, 3, 5):
        x = sim.ansatz_state(n, 2, np.zeros(3 * n * 2))
        e0 = np.zeros(1 << n, complex)
        e0[0] = 1
        assert np.max(np.abs(x - e0)) < 1e-15


def test_ansatz_n1_pi_gives_one():
    """n=1, d=1, params (pi,0,0) -> |1> up to phase."""
    x = sim.ansatz_state(1, 1, np.array([np.pi, 0.0, 0.0]))
    assert abs(abs(x[1]) - 1) < 1e-15 and abs(x[0]) < 1e-15


def test_ry_half_pi_is_plus():
    x = sim.ansatz_state(1, 1, np.array([np.pi / 2, 0.0, 0.0]))
    assert np.allclose(x, [2 ** -0.5, 2 ** -0.5], atol=1e-15)


def test_cnot_big_endian():
    """CNOT(control 0, target 1)|10> = |11> (qubit 0 = MSB)."""
    C = dense.controlled_matrix(dense.X2, 0, 1, 2)
    v = np.zeros(4)
    v[0b10] = 1
    assert np.array_equal(C @ v, np.eye(4)[0b11])


@pytest.mark.parametrize("n,d,ent", [(1, 3, 0), (2, 2, 0), (3, 2, 0), (4, 3, 0), (5, 2, 0),
                                     (3, 2, 1), (4, 2, 1)])
def test_ansatz_matches_dense_matrix_product(n, d, ent):
    th = seeds.theta0(n, d, seed=n + 10 * d)
    x = sim.ansatz_state(n, d, th, ent)
    xd = dense.ansatz_state(n, d, th, ent)
    assert np.max(np.abs(x - xd)) < 1e-13
    assert abs(np.linalg.norm(x) - 1) < 1e-13


def test_cz_ring_n2_degeneracy():
    """SURVEY §8(c) reading 6 trap: CZ(0,1) CZ(1,0) = I, so the n=2 CZ ansatz is a product state."""
    th = seeds.theta0(2, 3, seed=5)
    x = sim.ansatz_state(2, 3, th, entangler=1).reshape(2, 2)
    sv = np.linalg.svd(x, compute_uv=False)
    assert sv[1] < 1e-13


# --- U_b (reading 5) ----------------------------------------------------

def test_ub_uniform_is_hadamard_power():
    assert np.max(np.abs(sim.ub_matrix(3, 0) - dense.kron_all([dense.H2] * 3))) < 1e-15


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_householder_ub_prepares_b_and_is_unitary(seed):
    n = 4
    b = seeds.random_b(n, seed)
    U = sim.ub_matrix(n, 1, b)
    assert np.max(np.abs(U[:, 0] - b)) < 1e-14
    assert np.max(np.abs(U.conj().T @ U - np.eye(16))) < 1e-13


def test_householder_trivial_b_is_identity():
    b = np.zeros(8, complex)
    b[0] = 1
    assert np.max(np.abs(sim.ub_matrix(3, 1, b) - np.eye(8))) < 1e-15


# --- Hadamard tests ------------------------------------------------------------

def _decode(c, n, L):
    t, part = divmod(c, 2)
    return t // ((n + 1) * L), (t // (n + 1)) % L, t % (n + 1), part


def test_identity_denominator_is_one_zero():
    """B = I -> Re = 1, Im = 0 (den task with A_l = A_k)."""
    w = configs.cfg1()
    T = sim.workload_terms(w)
    n, L = w.n, w.L
    for l in range(L):
        t = (l * L + l) * (n + 1)
        assert abs(T[2 * t] - 1) < 1e-14 and abs(T[2 * t + 1]) < 1e-14


def test_z0_at_theta0_is_plus_one():
    """B = Z_0, x = |0..0> -> +1.  U_b = I (b = e_0), A_l = A_k = I."""
    n = 3
    b = np.zeros(8, complex)
    b[0] = 1
    T = sim.terms(n, 1, b"III", np.zeros(3 * n), bkind=1, b=b)
    for j in range(n):
        assert abs(T[2 * (1 + j)] - 1) < 1e-15 and abs(T[2 * (1 + j) + 1]) < 1e-15


@pytest.mark.parametrize("mk", [configs.cfg1, configs.cfg2_velocity, configs.cfg2_pressure])
def test_paper_configs_match_dense_quadratic_forms(mk):
    w = mk()
    th = w.theta0()
    T = sim.workload_terms(w, th)
    x = dense.ansatz_state(w.n, w.layers, th, w.entangler)
    assert np.max(np.abs(dense.all_terms_dense(w, x) - T)) < 1e-12


@pytest.mark.parametrize("n,L,d,amp,ent", [(2, 5, 2, False, 0), (2, 4, 1, True, 0),
                                           (3, 6, 2, False, 1), (3, 5, 2, True, 0),
                                           (4, 4, 2, True, 1), (1, 3, 2, False, 0)])
def test_random_lcu_matches_dense_quadratic_forms(n, L, d, amp, ent):
    """SPEC A4: random (l,k,j,theta), both parts, vs the dense quadratic form <= 1e-10."""
    w = configs.random_workload(n, L, d, seed=n * 31 + L, amplitudes=amp, entangler=ent)
    th = w.theta0()
    T = sim.workload_terms(w, th)
    x = dense.ansatz_state(n, d, th, ent)
    assert np.max(np.abs(dense.all_terms_dense(w, x) - T)) < 1e-12


def test_closed_form_full_size_sample():
    """n = 10 (cfg 3): gate-by-gate values vs the O(2^n) closed-form Pauli expectation."""
    w = configs.cfg3()
    th = w.theta0()
    idx = np.arange(0, w.n_circuits, 173)
    T = sim.workload_terms(w, th, idx=idx)
    x = sim.ansatz_state(w.n, w.layers, th)
    assert abs(np.linalg.norm(x) - 1) < 1e-13
    for c, v in zip(idx, T):
        l, k, s, part = _decode(int(c), w.n, w.L)
        ref = dense.term_closed_form_uniform(x, w.terms[l][1], w.terms[k][1], s)
        assert abs((ref.real if part == 0 else ref.imag) - v) < 1e-12


def test_faithful_equals_prefix_shared_bitwise():
    w = configs.random_workload(5, 6, 3, seed=9, amplitudes=True)
    idx = np.arange(0, w.n_circuits, 7)
    a = sim.workload_terms(w, mode=0, idx=idx)
    b = sim.workload_terms(w, mode=1, idx=idx)
    assert np.array_equal(a, b)


def test_theta_zero_selection_rule():
    """x = |0>: <0|B|0> != 0 only if B's combined x-mask is 0 (uniform b: B = A_l X_j A_k)."""
    w = configs.cfg1()
    T = sim.workload_terms(w, np.zeros(w.n_params))
    n, L = w.n, w.L
    for c in range(w.n_circuits):
        l, k, s, part = _decode(c, n, L)
        ml, mk = dense.masks(w.terms[l][1])[0], dense.masks(w.terms[k][1])[0]
        xm = ml ^ mk ^ ((1 << (n - s)) if s else 0)
        if xm:
            assert abs(T[c]) < 1e-14


def test_pair_conjugacy_and_diagonal_im_zero():
    """term(k,l,j) = conj(term(l,k,j)) (B(k,l) = B(l,k)^+); Im = 0 when l = k."""
    w = configs.random_workload(3, 5, 2, seed=2, amplitudes=True)
    T = sim.workload_terms(w)
    n, L = w.n, w.L
    for l in range(L):
        for k in range(L):
            for s in range(n + 1):
                t1 = (l * L + k) * (n + 1) + s
                t2 = (k * L + l) * (n + 1) + s
                assert abs(T[2 * t1] - T[2 * t2]) < 1e-13
                assert abs(T[2 * t1 + 1] + T[2 * t2 + 1]) < 1e-13
                if l == k:
                    assert abs(T[2 * t1 + 1]) < 1e-13


# --- Householder U_b in definition form (n > 12; reading 5) ------------------------------------

@pytest.fixture
def hh_form():
    old = sim.set_householder_form(1)
    yield
    sim.set_householder_form(old)


@pytest.mark.parametrize("n,L,ent", [(3, 4, 0), (4, 3, 1), (5, 2, 0)])
def test_householder_definition_form_matches_dense_quadratic_forms(hh_form, n, L, ent):
    """The n > 12 form psi -> w(psi - 2 v (v^+ psi)/v^+v) vs the dense quadratic form x^+ B x with
    B = A_l U_b Z_j U_b^+ A_k built from explicit matrices (dense.py), every circuit."""
    w = configs.random_workload(n, L, 2, seed=400 + n, amplitudes=True, entangler=ent)
    th = w.theta0()
    T = sim.workload_terms(w, th)
    x = dense.ansatz_state(n, 2, th, ent)
    assert np.max(np.abs(dense.all_terms_dense(w, x) - T)) < 1e-12


def test_householder_definition_form_equals_dense_oracle():
    """Both oracle forms of the same operator agree to rounding (n = 6, all circuits)."""
    w = configs.random_workload(6, 3, 2, seed=77, amplitudes=True)
    th = w.theta0()
    old = sim.set_householder_form(2)
    try:
        a = sim.workload_terms(w, th)
        sim.set_householder_form(1)
        b = sim.workload_terms(w, th)
    finally:
        sim.set_householder_form(old)
    assert np.max(np.abs(a - b)) < 1e-13


def _pauli_apply(s, x):
    """(P x)[i] = i^{nY} (-1)^{popcount((i ^ m) & z)} x[i ^ m]  (P|j> = i^{nY} (-1)^{j.z} |j ^ m>)."""
    xm, zm, ny = dense.masks(s)
    i = np.arange(x.size)
    src = i ^ xm
    return (1j ** ny) * (1.0 - 2.0 * dense._parity(src & zm)) * x[src]


@pytest.mark.parametrize("m", [0, 5, 4097])
def test_householder_large_n_basis_b(m):
    """n = 13 (definition form by default), b = e_m: w = 1, v = e_0 - e_m, so U_b swaps e_0 and
    e_m (U_b = I for m = 0) and U_b Z_j U_b^+ is the diagonal sign of Z_j with entries 0 and m
    exchanged: every term is <A_l x| D_j |A_k x>, an O(2^n) closed form."""
    n = 13
    b = np.zeros(1 << n, complex)
    b[m] = 1.0
    strings = ["I" * n, "X" + "Y" * 5 + "I" * 6 + "Z", "Z" * 3 + "X" * 10]
    paulis = "".join(strings).encode()
    th = seeds.theta0(n, 1, 3)
    L = len(strings)
    idx = np.arange(0, 2 * (n + 1) * L * L, 7)
    T = sim.terms(n, 1, paulis, th, bkind=1, b=b, idx=idx)
    x = sim.ansatz_state(n, 1, th)
    i = np.arange(1 << n)
    for c, v in zip(idx, T):
        l, k, s, part = _decode(int(c), n, L)
        yl, yk = _pauli_apply(strings[l], x), _pauli_apply(strings[k], x)
        if s == 0:
            d = np.ones(1 << n)
        else:
            d = 1.0 - 2.0 * ((i >> (n - s)) & 1)
            d[[0, m]] = d[[m, 0]]
        ref = np.vdot(yl, d * yk)
        assert abs((ref.real if part == 0 else ref.imag) - v) < 1e-12
