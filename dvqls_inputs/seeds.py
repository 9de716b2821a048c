"""Seeded random inputs (SURVEY.md §8(d) "Synthetic inputs").

* theta_0 ~ U[-pi, pi)^P with numpy.random.default_rng(seed) (Alg. 1 Step 3,
  P:448 "Initialize theta_0 randomly"); P = 3 n d (SURVEY.md §8(c) reading 6).
* robustness LCUs: L distinct random Pauli strings over {I,X,Y,Z}^n with complex
  N(0,1) coefficients (non-Hermitian A, so the Im Hadamard test is exercised);
* random normalised complex b (Householder U_b path, SURVEY.md §8(c) reading 5).
"""

from __future__ import annotations

import numpy as np


def n_params(n: int, layers: int) -> int:
    return 3 * n * layers


def theta0(n: int, layers: int, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-np.pi, np.pi, n_params(n, layers))


def thetas(n: int, layers: int, K: int, seed: int = 0) -> np.ndarray:
    """K independent parameter vectors, shape (K, P)."""
    return np.random.default_rng(seed).uniform(-np.pi, np.pi, (K, n_params(n, layers)))


def random_lcu(n: int, L: int, seed: int = 0, hermitian: bool = False):
    """L distinct random Pauli strings with complex N(0,1) (or real if hermitian) coefficients."""
    rng = np.random.default_rng(seed)
    if L > 4 ** n:
        raise ValueError("random_lcu: L > 4^n")
    seen = set()
    terms = []
    while len(terms) < L:
        s = "".join("IXYZ"[v] for v in rng.integers(0, 4, n))
        if s in seen:
            continue
        seen.add(s)
        re, im = rng.standard_normal(2)
        terms.append((complex(re, 0.0 if hermitian else im), s))
    return terms


def random_b(n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return v / np.linalg.norm(v)
