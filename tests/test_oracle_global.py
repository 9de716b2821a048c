"""Pins for the NEXT-3 oracle (global cost C_G, Eq. 1) - CPU only.

oracle.sim.overlap_terms runs the overlap Hadamard test gate by gate (controlled V(theta),
controlled A_l, controlled U_b^+ on n+1 qubits).  It is pinned against
  * the dense textbook overlap <b|A_l|x> = b^+ (A_l x) (Pauli matrices, dense ansatz),
  * the closed form C_G = 1 - |<b|A|x>|^2 / <x|A^+A|x> (oracle/dense.global_cost),
  * the operator sandwich C_L <= C_G <= n C_L (SURVEY §8(c) cost pin iii),
  * special cases: A = I and b = |0> with x = |0> -> C_G = 0 and beta = 1;
    theta = 0 (x = |0>) with uniform b -> beta_l = 2^{-n/2} * (sum of A_l's column 0).
"""

import numpy as np
import pytest

from dvqls_inputs import configs
from oracle import cost, dense, sim


def _b_of(w):
    N = 1 << w.n
    return np.full(N, N ** -0.5, dtype=complex) if w.bkind == 0 else np.asarray(w.b, dtype=complex)


def _dense_overlaps(w, x):
    b = _b_of(w)
    out = []
    for _, s in w.terms:
        v = np.vdot(b, dense.pauli_matrix(s) @ x)
        out += [v.real, v.imag]
    return np.array(out)


@pytest.mark.parametrize("mk", [configs.cfg1, configs.cfg2_velocity, configs.cfg2_pressure])
def test_overlaps_equal_dense(mk):
    w = mk()
    for seed in range(2):
        th = w.theta0(seed)
        got = sim.workload_overlaps(w, th)
        x = dense.ansatz_state(w.n, w.layers, th)
        assert np.max(np.abs(got - _dense_overlaps(w, x))) < 1e-12


@pytest.mark.parametrize("n,amp,ent", [(2, False, 0), (3, True, 0), (4, False, 1), (5, True, 1)])
def test_random_non_hermitian(n, amp, ent):
    w = configs.random_workload(n, 4, 2, seed=40 + n, amplitudes=amp, entangler=ent)
    th = w.theta0()
    got = sim.workload_overlaps(w, th)
    x = dense.ansatz_state(w.n, w.layers, th, ent)
    assert np.max(np.abs(got - _dense_overlaps(w, x))) < 1e-12


@pytest.mark.parametrize("mk", [configs.cfg1, configs.cfg2_velocity, configs.cfg2_pressure])
def test_global_cost_closed_form_and_sandwich(mk):
    w = mk()
    b = _b_of(w)
    for seed in range(3):
        th = w.theta0(seed)
        T = sim.workload_terms(w, th)
        CL, E, Psi = cost.cost(T, cost.coeffs_of(w), w.n, w.L)
        CG = cost.global_cost(sim.workload_overlaps(w, th), cost.coeffs_of(w), Psi)
        x = dense.ansatz_state(w.n, w.layers, th)
        assert abs(CG - dense.global_cost(w.A, b, x)) < 1e-12
        assert 0.0 <= CG <= 1.0 + 1e-12
        assert CL <= CG + 1e-12 and CG <= w.n * CL + 1e-12


def test_special_cases():
    # theta = 0 -> x = |0>, uniform b: beta_l = <b|A_l|0> = 2^{-n/2} i^{ny} (-1)^{popcount(m & z)}
    w = configs.cfg1()
    got = sim.workload_overlaps(w, np.zeros(w.n_params))
    N = 1 << w.n
    for l, (_, s) in enumerate(w.terms):
        col0 = dense.pauli_matrix(s)[:, 0]
        ref = col0.sum() / np.sqrt(N)
        assert abs(got[2 * l] - ref.real) < 1e-14 and abs(got[2 * l + 1] - ref.imag) < 1e-14
    # A = I, b = |0>, x = |0>: C_G = 0, beta = 1
    n = 3
    b = np.zeros(1 << n, dtype=complex)
    b[0] = 1.0
    ov = sim.overlap_terms(n, 1, b"III", np.zeros(3 * n), 1, b)
    assert abs(ov[0] - 1.0) < 1e-14 and abs(ov[1]) < 1e-14
    assert abs(cost.global_cost(ov, [1.0], 1.0 + 0j)) < 1e-14
