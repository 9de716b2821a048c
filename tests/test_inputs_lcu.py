"""Pins for the LCU / problem inputs (dvqls_inputs) - CPU only.

The FWHT decomposition is pinned against the DEFINITION c_P = tr(P A)/2^n
(oracle.dense.decompose_bruteforce), the reconstruction sum_l c_l P_l, SPEC.md
worked examples, and the paper's printed term counts (Table II).
"""

import numpy as np
import pytest

from conftest import golden
from dvqls_inputs import configs, lcu, problems
from oracle import dense


def _as_dict(terms):
    return {s: c for c, s in terms}


@pytest.mark.parametrize("case", golden("spec_examples.json")["decompose"])
def test_spec_decompose_examples(case):
    A = np.array(case["A"], dtype=float)
    got = _as_dict(lcu.decompose_pruned(A, 0.0))
    assert set(got) == set(case["terms"])
    for s, v in case["terms"].items():
        assert abs(got[s] - v) < 1e-15


@pytest.mark.parametrize("n", [1, 2, 3])
def test_fwht_equals_trace_formula(n):
    rng = np.random.default_rng(100 + n)
    for _ in range(20):
        N = 1 << n
        A = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
        coeffs, _ = lcu.decompose(A)
        brute = dense.decompose_bruteforce(A)
        for code, c in enumerate(coeffs):
            assert abs(c - brute[lcu.code_to_string(code, n)]) < 1e-12


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_round_trip(n):
    rng = np.random.default_rng(7 + n)
    N = 1 << n
    A = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    terms = lcu.decompose_pruned(A, 0.0)
    assert np.max(np.abs(dense.reconstruct(terms, n) - A)) < 1e-12


def test_hermitian_gives_real_coefficients():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
    H = M + M.conj().T
    coeffs, _ = lcu.decompose(H)
    assert np.max(np.abs(coeffs.imag)) < 1e-12


def test_pruning_monotone_and_ordered():
    A, _ = problems.tridiag_toeplitz(6)
    prev = None
    for eps in [0.0, 0.005, 0.01, 0.02, 0.05, 0.1]:
        t = lcu.decompose_pruned(A, eps)
        mags = [abs(c) for c, _ in t]
        assert all(mags[i] >= mags[i + 1] - 1e-12 for i in range(len(mags) - 1))
        s = {p for _, p in t}
        if prev is not None:
            assert s <= prev
        prev = s


def test_table2_term_counts_default_reading():
    """(a,b,c) = (2,-1,-1): eps 0.03/0.02/0.01/0.005 -> 16/32/64/128 (Table II)."""
    g = golden("table2.json")
    for row in g["rows"]:
        if row["eps"] in (0.1, 0.05):
            continue  # reading 4: 8/16 under (2,-1,-1); see next test
        assert len(configs._tridiag_terms(10, row["eps"])) == row["L"]
        assert 2 * (10 + 1) * row["L"] ** 2 == row["circuits"]


def test_table2_term_counts_a25_reading():
    """SURVEY §8(c) reading 4: a = 2.5 reproduces all six Table II L values."""
    for row in golden("table2.json")["rows"]:
        assert len(configs._tridiag_terms(10, row["eps"], 2.5)) == row["L"]


def test_pruning_claim_p490():
    """'2^n Pauli terms when n <= 6 ... saturates at 64 terms for n > 6'."""
    for n in range(2, 11):
        assert len(configs._tridiag_terms(n, 0.01)) == min(1 << n, 64)


def test_term_reduction_p269():
    g = golden("table2.json")["term_reduction"]
    assert 2 * 11 * (1 << 10) ** 2 == g["unpruned_circuits"]
    assert 2 * 11 * 64 ** 2 == g["pruned_circuits"]
    assert g["unpruned_circuits"] // g["pruned_circuits"] == 256


@pytest.mark.parametrize("n", [8, 9])
def test_identity_padding(n):
    """pruned(n >= 7, eps=0.01) == I-padded pruned(7) (used for cfg 5 inputs)."""
    full = {s: c for c, s in configs._tridiag_terms(n, 0.01)}
    pad = {s: c for c, s in lcu.identity_padded(list(configs._tridiag_terms(7, 0.01)), n - 7)}
    assert set(full) == set(pad)
    for s in full:
        assert abs(full[s] - pad[s]) < 1e-12


def test_hele_shaw_systems():
    """SPD systems; pressure linear in x, velocity parabolic (reading 21)."""
    Ap, rp = problems.hele_shaw_pressure()
    Au, ru = problems.hele_shaw_velocity()
    for A in (Ap, Au):
        assert np.array_equal(A, A.T)
        assert np.linalg.eigvalsh(A).min() > 0
    p = np.linalg.solve(Ap, rp).reshape(4, 4)
    assert np.allclose(p, np.tile([0.8, 0.6, 0.4, 0.2], (4, 1)), atol=1e-13)
    u = np.linalg.solve(Au, ru).reshape(4, 4)
    assert np.allclose(u, np.tile([[0.4], [0.6], [0.6], [0.4]], (1, 4)), atol=1e-13)
    assert np.allclose(ru, ru[0], atol=1e-15)  # uniform rhs -> U_b = H^{(x)4}
    assert configs.cfg2_velocity().L == 8 and configs.cfg2_pressure().L == 8


def test_tridiag_spectrum_closed_form():
    """eigenvalues of tridiag(2,-1,-1), N=4, are 2 - 2 cos(k pi/5)."""
    A, _ = problems.tridiag_toeplitz(2)
    ev = np.sort(np.linalg.eigvalsh(A))
    ref = np.sort([2 - 2 * np.cos(k * np.pi / 5) for k in range(1, 5)])
    assert np.allclose(ev, ref, atol=1e-14)
