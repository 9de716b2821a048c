"""Pins for the NEXT-4 oracle (oracle/pauli_decomp.py: Alg. 1 Steps 1-2) - CPU only.

* every coefficient equals the brute-force trace formula tr(P A)/2^n with dense Pauli matrices
  (oracle/dense.py, n <= 4) on random complex matrices;
* round trip: sum_P c_P P reconstructs A (n = 5, 6);
* Parseval: sum_P |c_P|^2 = ||A||_F^2 / 2^n;
* the pruned tridiagonal Toeplitz decomposition reproduces Table II's term counts L = 64 / 128
  at eps = 0.01 / 0.005 for n = 10 (golden table2.json) and the SPEC worked examples.
"""

import numpy as np
import pytest

from conftest import golden
from dvqls_inputs import problems
from oracle import dense, pauli_decomp


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_coefficients_equal_trace_formula(n):
    rng = np.random.default_rng(n)
    N = 1 << n
    A = rng.normal(size=(N, N)) + 1j * rng.normal(size=(N, N))
    C = pauli_decomp.coefficients(A)
    ref = dense.decompose_bruteforce(A)
    for m in range(N):
        for z in range(N):
            s = pauli_decomp.pauli_string(m, z, n)
            assert abs(C[m, z] - ref[s]) < 1e-12


@pytest.mark.parametrize("n", [5, 6])
def test_round_trip_and_parseval(n):
    rng = np.random.default_rng(10 + n)
    N = 1 << n
    A = rng.normal(size=(N, N)) + 1j * rng.normal(size=(N, N))
    C = pauli_decomp.coefficients(A)
    R = np.zeros_like(A)
    for m in range(N):
        for z in range(N):
            R += C[m, z] * dense.pauli_matrix(pauli_decomp.pauli_string(m, z, n))
    assert np.max(np.abs(R - A)) < 1e-11
    assert abs(np.sum(np.abs(C) ** 2) - np.sum(np.abs(A) ** 2) / N) < 1e-9


def test_table2_term_counts():
    """Table II: L = 64 at eps = 0.01 and 128 at eps = 0.005 (reading 4, a = 2)."""
    g = golden("table2.json")
    A, _ = problems.tridiag_toeplitz(g["n"], 2.0, -1.0, -1.0)
    for row in g["rows"]:
        if row["eps"] in (0.01, 0.005):
            terms, _ = pauli_decomp.decompose_pruned(A, row["eps"])
            assert len(terms) == row["L"]
            assert 2 * (g["n"] + 1) * len(terms) ** 2 == row["circuits"]


def test_ordering_rule():
    A, _ = problems.tridiag_toeplitz(4, 2.0, -1.0, -1.0)
    terms, norm = pauli_decomp.decompose_pruned(A, 0.01)
    mags = [abs(c) for c, _ in terms]
    assert all(mags[i] >= mags[i + 1] - 1e-12 * norm for i in range(len(mags) - 1))
    for i in range(len(terms) - 1):
        if abs(mags[i] - mags[i + 1]) < 1e-13:
            assert terms[i][1] < terms[i + 1][1]  # ASCII order of I<X<Y<Z is the lexicographic rule
    assert terms[0] == (2.0 + 0j, "IIII")


def test_single_coefficient_matches_full_transform():
    rng = np.random.default_rng(3)
    n = 6
    N = 1 << n
    A = rng.normal(size=(N, N)) + 1j * rng.normal(size=(N, N))
    C = pauli_decomp.coefficients(A)
    for m, z in [(0, 0), (5, 9), (63, 63), (17, 40)]:
        assert abs(pauli_decomp.coefficient(A, m, z) - C[m, z]) < 1e-12
