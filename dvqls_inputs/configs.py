"""BASELINE.json configurations as concrete synthetic inputs.

Every config yields a ``Workload``: n system qubits, ansatz layers d, the LCU
(list of (c_l, pauli_string)), the b-preparation kind and amplitudes, and the
seeded theta_0.  Nothing here evaluates the method.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import lcu, problems, seeds

B_UNIFORM = 0     # U_b = H^{(x)n}                      (SURVEY.md §8(c) reading 3)
B_AMPLITUDES = 1  # U_b = Householder completion of b    (SURVEY.md §8(c) reading 5)


@dataclass
class Workload:
    name: str
    n: int
    layers: int
    terms: list
    bkind: int = B_UNIFORM
    b: np.ndarray | None = None  # normalised complex b (AMPLITUDES), else None
    seed: int = 0
    entangler: int = 0           # 0 = CNOT ring (default), 1 = CZ ring
    A: np.ndarray | None = field(default=None, repr=False)    # dense A when small
    rhs: np.ndarray | None = field(default=None, repr=False)  # dense rhs when small

    @property
    def L(self) -> int:
        return len(self.terms)

    @property
    def n_params(self) -> int:
        return seeds.n_params(self.n, self.layers)

    @property
    def n_tasks(self) -> int:
        return (self.n + 1) * self.L * self.L

    @property
    def n_circuits(self) -> int:
        return 2 * self.n_tasks

    def theta0(self, seed: int | None = None) -> np.ndarray:
        return seeds.theta0(self.n, self.layers, self.seed if seed is None else seed)

    def arrays(self):
        return lcu.to_arrays(self.terms)


@lru_cache(maxsize=None)
def _tridiag_terms(n: int, eps: float, a: float = 2.0):
    A, _ = problems.tridiag_toeplitz(n, a, -1.0, -1.0)
    return tuple(lcu.decompose_pruned(A, eps))


def tridiag(n: int, layers: int, eps: float = 0.01, seed: int = 0, a: float = 2.0) -> Workload:
    A, rhs = problems.tridiag_toeplitz(n, a, -1.0, -1.0) if n <= 10 else (None, None)
    return Workload(f"tridiag_n{n}_eps{eps}", n, layers, list(_tridiag_terms(n, eps, a)),
                    B_UNIFORM, None, seed, A=A, rhs=rhs)


def cfg1(seed: int = 0) -> Workload:
    """4-qubit tridiagonal Toeplitz (16x16), L=16, d=4, single cost eval."""
    w = tridiag(4, 4, 0.01, seed)
    w.name = "cfg1_tridiag_n4_L16_d4"
    return w


def cfg2_velocity(seed: int = 0, layers: int = 4) -> Workload:
    A, rhs = problems.hele_shaw_velocity(4)
    terms = lcu.decompose_pruned(A, 0.01)
    return Workload("cfg2_heleshaw_u_n4", 4, layers, terms, B_UNIFORM, None, seed, A=A, rhs=rhs)


def cfg2_pressure(seed: int = 0, layers: int = 4) -> Workload:
    A, rhs = problems.hele_shaw_pressure(4)
    terms = lcu.decompose_pruned(A, 0.01)
    return Workload("cfg2_heleshaw_p_n4", 4, layers, terms, B_AMPLITUDES,
                    problems.normalise(rhs), seed, A=A, rhs=rhs)


def cfg3(seed: int = 0) -> Workload:
    """10-qubit, L=64 (eps=0.01), d=10: 45,056 tasks = 90,112 circuits."""
    w = tridiag(10, 10, 0.01, seed)
    w.name = "cfg3_tridiag_n10_L64_d10"
    return w


def cfg4(seed: int = 0) -> Workload:
    """10-qubit, L=128 (eps=0.005), d=10: 180,224 tasks = 360,448 circuits."""
    w = tridiag(10, 10, 0.005, seed)
    w.name = "cfg4_tridiag_n10_L128_d10"
    return w


def cfg5(n: int, seed: int = 0) -> Workload:
    """n in 12..24: LCU = I^{(n-7)} (x) pruned-tridiag(7) (L=64), d=3."""
    base = list(_tridiag_terms(7, 0.01))
    terms = lcu.identity_padded(base, n - 7)
    return Workload(f"cfg5_n{n}_L64_d3", n, 3, terms, B_UNIFORM, None, seed)


def cfg5_amplitudes(n: int, seed: int = 0) -> Workload:
    """Config 5's LCU and depth with a general b ("general b"): a seeded random normalised
    complex b, U_b its Householder completion (SURVEY §8(c) reading 5)."""
    w = cfg5(n, seed)
    w.name = f"cfg5_amp_n{n}_L64_d3"
    w.bkind = B_AMPLITUDES
    w.b = seeds.random_b(n, seed + 1)
    return w


def random_workload(n: int, L: int, layers: int, seed: int = 0, amplitudes: bool = False,
                    entangler: int = 0) -> Workload:
    terms = seeds.random_lcu(n, L, seed)
    b = seeds.random_b(n, seed + 1) if amplitudes else None
    return Workload(f"random_n{n}_L{L}_d{layers}_{'amp' if amplitudes else 'uni'}", n, layers,
                    terms, B_AMPLITUDES if amplitudes else B_UNIFORM, b, seed, entangler)
