"""GPU parity of NEXT-4 (dvqls_decompose / dvqls_pauli_coefficients, decomp.cuh) against the
definitional oracle (oracle/pauli_decomp.py): every coefficient <= 1e-12 * ||A||, the pruned
LCU identical (strings, order) with coefficients <= 1e-12; n = 13 by sampled coefficients and
sampled reconstruction of A."""

import numpy as np
import pytest

from dvqls_inputs import problems
from oracle import pauli_decomp as opd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_14435_b200 import build, dvqls
    build.build()
    return dvqls


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 9, 10])
def test_all_coefficients_random(dv, n):
    rng = np.random.default_rng(100 + n)
    N = 1 << n
    A = rng.normal(size=(N, N)) + 1j * rng.normal(size=(N, N))
    got = dv.pauli_coefficients(A)
    assert np.max(np.abs(got - opd.coefficients(A))) <= 1e-12 * max(1.0, np.abs(A).max())


@pytest.mark.parametrize("n,eps", [(4, 0.01), (6, 0.01), (8, 0.01), (9, 0.01), (10, 0.01), (10, 0.005),
                                   (11, 0.01), (12, 0.01)])
def test_pruned_tridiagonal(dv, n, eps):
    A, _ = problems.tridiag_toeplitz(n, 2.0, -1.0, -1.0)
    got, norm = dv.decompose(A, eps)
    ref, rnorm = opd.decompose_pruned(A, eps)
    assert abs(norm - rnorm) <= 1e-12 * rnorm
    assert [s for _, s in got] == [s for _, s in ref]
    assert max(abs(a - b) for (a, _), (b, _) in zip(got, ref)) <= 1e-12


@pytest.mark.parametrize("which", ["p", "u"])
def test_pruned_hele_shaw(dv, which):
    A, _ = problems.hele_shaw_pressure(4) if which == "p" else problems.hele_shaw_velocity(4)
    got, _ = dv.decompose(A, 0.01)
    ref, _ = opd.decompose_pruned(A, 0.01)
    assert [s for _, s in got] == [s for _, s in ref]
    assert max(abs(a - b) for (a, _), (b, _) in zip(got, ref)) <= 1e-12


@pytest.mark.parametrize("n,eps", [(7, 0.015), (9, 0.0055)])
def test_pruned_random_dense(dv, n, eps):
    """Dense random A: many coefficients near the threshold, so the Parseval candidate bound and
    the exact-norm filter of the one-pass pruning are both exercised."""
    rng = np.random.default_rng(5)
    N = 1 << n
    A = rng.normal(size=(N, N)) + 1j * rng.normal(size=(N, N))
    got, _ = dv.decompose(A, eps)
    ref, _ = opd.decompose_pruned(A, eps)
    assert len(got) == len(ref) > 0
    assert [s for _, s in got] == [s for _, s in ref]
    assert max(abs(a - b) for (a, _), (b, _) in zip(got, ref)) <= 1e-12


def test_n13_sampled(dv):
    """n = 13 (A is 1 GB): 64 sampled coefficients by the oracle's one-at-a-time definition and
    16 sampled entries of A rebuilt from the GPU's 4^13 coefficients."""
    n = 13
    N = 1 << n
    rng = np.random.default_rng(13)
    A = np.zeros((N, N), dtype=np.complex128)
    A[np.arange(N), np.arange(N)] = 2.5
    A[np.arange(N - 1), np.arange(1, N)] = -1.0 + 0.25j
    A[np.arange(1, N), np.arange(N - 1)] = -1.0 - 0.25j
    rows = rng.integers(0, N, 64)
    A[rows, rng.integers(0, N, 64)] += rng.normal(size=64)  # break the Toeplitz structure
    C = dv.pauli_coefficients(A)
    for m, z in zip(rng.integers(0, N, 64), rng.integers(0, N, 64)):
        assert abs(C[m, z] - opd.coefficient(A, int(m), int(z))) <= 1e-12
    zz = np.arange(N)
    for i, j in zip(rng.integers(0, N, 16), rng.integers(0, N, 16)):
        m = int(i) ^ int(j)
        pz = np.array([bin(int(v)).count("1") for v in (m & zz)]) % 4
        pj = np.array([bin(int(v)).count("1") for v in (int(j) & zz)]) % 2
        val = np.sum(C[m, :] * (1j) ** pz * np.where(pj == 1, -1.0, 1.0))
        assert abs(val - A[i, j]) <= 1e-10
    got, norm = dv.decompose(A, 0.01)
    assert abs(norm ** 2 - np.sum(np.abs(A) ** 2) / N) <= 1e-9 * norm ** 2  # Parseval
    assert len(got) > 0 and all(abs(c) >= 0.01 * norm for c, _ in got)


@pytest.mark.parametrize("n,eps", [(7, 0.001), (8, 0.002)])
def test_pruned_dense_beyond_the_one_cta_sort(dv, n, eps):
    """A dense random A keeps most of its 4^n coefficients: more than the 4,096 candidates of the
    one-CTA sort, so the global bitonic path orders them; strings and order identical to the
    oracle, coefficients <= 1e-12 * ||A||."""
    rng = np.random.default_rng(700 + n)
    N = 1 << n
    A = rng.normal(size=(N, N)) + 1j * rng.normal(size=(N, N))
    got, norm = dv.decompose(A, eps, max_terms=4 ** n)
    ref, rnorm = opd.decompose_pruned(A, eps)
    assert len(ref) > 4096
    assert len(got) == len(ref)
    assert [s for _, s in got] == [s for _, s in ref]
    assert max(abs(c - r) for (c, _), (r, _) in zip(got, ref)) <= 1e-12 * np.abs(A).max()
    assert abs(norm - rnorm) <= 1e-12 * rnorm
