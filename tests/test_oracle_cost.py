"""Pins for the oracle cost (Alg. 1 Steps 4b-4c) - CPU only.

The oracle's C = 1/2 - Re E / (2 n Re Psi) is checked against the dense local
cost written from Eq. 2 read with P_j = Z_j, the global cost Eq. 1
sandwich C_L <= C_G <= n C_L, special cases with known answers, and range.
"""

import numpy as np
import pytest

from conftest import golden
from dvqls_inputs import configs, problems, lcu
from oracle import cost, dense, sim


def _oracle_cost(w, th):
    T = sim.workload_terms(w, th)
    return cost.cost(T, cost.coeffs_of(w), w.n, w.L)


@pytest.mark.parametrize("mk", [configs.cfg1, configs.cfg2_velocity, configs.cfg2_pressure])
def test_cost_equals_dense_local_cost(mk):
    w = mk()
    for seed in range(3):
        th = w.theta0(seed)
        C, E, Psi = _oracle_cost(w, th)
        x = dense.ansatz_state(w.n, w.layers, th)
        Ub = dense.ub_dense(w.n, w.bkind, w.b)
        assert abs(C - dense.local_cost(w.A, Ub, x, w.n)) < 1e-12
        # Eq. 2 (with Z_j) = 2 x Alg. 1 form (reading 1)
        assert abs(dense.local_cost_eq2(w.A, Ub, x, w.n) - 2 * C) < 1e-12
        assert abs(1 - E.real / (w.n * Psi.real) - 2 * C) < 1e-12
        # Hermitian A, real b: imaginary residues vanish (reading 12)
        assert abs(E.imag) < 1e-12 and abs(Psi.imag) < 1e-12


def test_cost_range_and_global_sandwich():
    """0 <= C_L <= 1 and C_L <= C_G <= n C_L (operator inequality on Hamming weight)."""
    for n in (2, 3):
        A, rhs = problems.tridiag_toeplitz(n, 2.5)
        terms = lcu.decompose_pruned(A, 0.0)
        for amp in (False, True):
            b = problems.normalise(np.random.default_rng(n).standard_normal(1 << n)) if amp \
                else problems.normalise(rhs)
            w = configs.Workload("t", n, 2, terms, 1 if amp else 0, b if amp else None, A=A)
            for seed in range(6):
                th = w.theta0(seed)
                C, _, _ = _oracle_cost(w, th)
                x = dense.ansatz_state(n, 2, th)
                CG = dense.global_cost(A, b, x)
                assert -1e-12 <= C <= 1 + 1e-12
                assert C - 1e-12 <= CG <= n * C + 1e-12


def test_exact_solution_gives_zero_cost():
    """A = [[2,-1],[-1,2]], b uniform: x* = |+> = Ry(pi/2)|0>  ->  C = 0."""
    A, _ = problems.tridiag_toeplitz(1)
    w = configs.Workload("t", 1, 1, lcu.decompose_pruned(A, 0.0))
    C, _, _ = _oracle_cost(w, np.array([np.pi / 2, 0.0, 0.0]))
    assert abs(C) < 1e-15


def test_orthogonal_state_gives_cost_one():
    """A = I, b = |0>, x = |1>  ->  C = 1."""
    b = np.array([1, 0], dtype=complex)
    w = configs.Workload("t", 1, 1, [(1.0 + 0j, "I")], 1, b)
    C, _, _ = _oracle_cost(w, np.array([np.pi, 0.0, 0.0]))
    assert abs(C - 1) < 1e-15


def test_degenerate_denominator_raises():
    with pytest.raises(cost.DegenerateDenominator):
        cost.cost_from(0j, 0j, 3)


def test_convention_crosscheck_values():
    """SURVEY §8(c) convention cross-check values (NOT paper pins; drift detector)."""
    g = golden("convention_crosscheck.json")
    tol = g["tolerance"]
    mk = {"cfg1": configs.cfg1, "cfg2_pressure": configs.cfg2_pressure,
          "cfg2_velocity": configs.cfg2_velocity}
    for case in g["cases"]:
        w = mk[case["config"]]()
        C, E, Psi = _oracle_cost(w, w.theta0(0))
        assert abs(C - case["C"]) < tol
        if "E" in case:
            assert abs(E.real - case["E"]) < tol and abs(Psi.real - case["Psi"]) < tol
