"""NEXT-2 host algebra (dvqls_task_observable, pure host, no GPU): the observable of every
Hadamard-test task for uniform b is one Pauli string up to a phase,
    B = A_l U_b Z_j U_b^+ A_k = A_l X_j A_k   (U_b = H^n),  B = A_l A_k (denominator),
and the library's symbolic product (x_mask, z_mask, i^phase) must equal the dense matrix product
of the oracle's textbook Pauli and Hadamard matrices (oracle/dense.py), entry by entry."""

import itertools

import numpy as np
import pytest

from oracle import dense


def _matrix_of(n, m, z, q):
    N = 1 << n
    M = np.zeros((N, N), dtype=complex)
    for i in range(N):
        M[i ^ m, i] = (1j ** q) * (-1) ** bin(i & z).count("1")
    return M


def _lib():
    from paper_2604_14435_b200 import dvqls
    try:
        dvqls.load()
    except RuntimeError as e:  # library not built in this checkout
        pytest.skip(str(e))
    return dvqls


@pytest.mark.parametrize("n", [1, 2, 3])
def test_every_pair_and_s_matches_dense(n):
    dv = _lib()
    Ub = dense.ub_dense(n, 0)
    strings = ["".join(p) for p in itertools.product("IXYZ", repeat=n)]
    rng = np.random.default_rng(n)
    pairs = [(a, b) for a in strings for b in strings]
    if len(pairs) > 600:
        pairs = [pairs[i] for i in rng.choice(len(pairs), 600, replace=False)]
    for sl, sk in pairs:
        for s in range(n + 1):
            m, z, q = dv.task_observable(n, sl, sk, s)
            B = dense.term_operator(sl, sk, s, Ub)
            assert np.allclose(_matrix_of(n, m, z, q), B, atol=1e-12), (sl, sk, s, m, z, q)


def test_random_strings_n6():
    dv = _lib()
    n = 6
    Ub = dense.ub_dense(n, 0)
    rng = np.random.default_rng(7)
    for _ in range(40):
        sl = "".join(rng.choice(list("IXYZ"), n))
        sk = "".join(rng.choice(list("IXYZ"), n))
        s = int(rng.integers(0, n + 1))
        m, z, q = dv.task_observable(n, sl, sk, s)
        assert np.allclose(_matrix_of(n, m, z, q), dense.term_operator(sl, sk, s, Ub), atol=1e-12)


def test_errors():
    dv = _lib()
    with pytest.raises(dv.DvqlsError):
        dv.task_observable(2, "XQ", "II", 0)
    with pytest.raises(dv.DvqlsError):
        dv.task_observable(2, "XX", "II", 3)
