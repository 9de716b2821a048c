"""ORACLE - TEST INFRASTRUCTURE ONLY.

Dense-matrix references (numpy) used to pin the gate-by-gate simulator and the
LCU inputs.  Each function is the textbook definition written out; none of
them shares code with oracle/sim.cpp or with the CUDA path.

* Pauli matrices, Kronecker strings, products
* brute-force trace decomposition c_P = tr(P A)/2^n
* dense ansatz V(theta) as a product of full 2^n x 2^n gate matrices
                                                          
* U_b: H^{(x)n} by Kronecker products; Householder completion
                                                          (SURVEY §8(c) reading 5)
* dense quadratic forms <x|B|x>, B = A_l U_b Z_j U_b^+ A_k (Eq. 4)
* local cost, Alg. 1 form 1/2 - (1/2n) sum_j ... and Eq. 2 form
* global cost Eq. 1, C_G = 1 - |<b|A|x>|^2 / <x|A^+A|x>
* closed-form Pauli expectation <x|P|x> in O(2^n)        (SURVEY §8(c) pin (ii))
"""

from __future__ import annotations

import itertools
from functools import reduce

import numpy as np

I2 = np.eye(2, dtype=np.complex128)
X2 = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y2 = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z2 = np.array([[1, 0], [0, -1]], dtype=np.complex128)
H2 = np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2.0)
PAULI = {"I": I2, "X": X2, "Y": Y2, "Z": Z2}

# single-qubit Pauli products a*b = phase * r   (XY = iZ, YZ = iX, ZX = iY, ...)
_PROD = {
    ("X", "Y"): (1j, "Z"), ("Y", "X"): (-1j, "Z"),
    ("Y", "Z"): (1j, "X"), ("Z", "Y"): (-1j, "X"),
    ("Z", "X"): (1j, "Y"), ("X", "Z"): (-1j, "Y"),
}


def kron_all(mats):
    return reduce(np.kron, mats)


def pauli_matrix(s: str) -> np.ndarray:
    """Kronecker product in string order: char 0 = qubit 0 = most significant."""
    return kron_all([PAULI[ch] for ch in s])


def pauli_product(p: str, q: str):
    """matrix(p) @ matrix(q) = phase * matrix(r)."""
    if len(p) != len(q):
        raise ValueError("pauli_product: length mismatch")
    phase = 1 + 0j
    r = []
    for a, b in zip(p, q):
        if a == "I":
            r.append(b)
        elif b == "I":
            r.append(a)
        elif a == b:
            r.append("I")
        else:
            ph, c = _PROD[(a, b)]
            phase *= ph
            r.append(c)
    return phase, "".join(r)


def decompose_bruteforce(A: np.ndarray) -> dict:
    """All 4^n coefficients c_P = tr(P A) / 2^n (definition; n <= 4)."""
    N = A.shape[0]
    n = N.bit_length() - 1
    out = {}
    for tup in itertools.product("IXYZ", repeat=n):
        s = "".join(tup)
        out[s] = complex(np.trace(pauli_matrix(s) @ A) / N)
    return out


def reconstruct(terms, n: int) -> np.ndarray:
    A = np.zeros((1 << n, 1 << n), dtype=np.complex128)
    for c, s in terms:
        A += c * pauli_matrix(s)
    return A


def embed_1q(U: np.ndarray, q: int, n: int) -> np.ndarray:
    return kron_all([U if i == q else I2 for i in range(n)])


def controlled_matrix(U2: np.ndarray, c: int, t: int, n: int) -> np.ndarray:
    """|0><0|_c (x) I + |1><1|_c (x) U_t, as a full 2^n x 2^n matrix."""
    P0 = np.array([[1, 0], [0, 0]], dtype=np.complex128)
    P1 = np.array([[0, 0], [0, 1]], dtype=np.complex128)
    a = kron_all([P0 if i == c else I2 for i in range(n)])
    b = kron_all([P1 if i == c else (U2 if i == t else I2) for i in range(n)])
    return a + b


def ry(t):
    return np.array([[np.cos(t / 2), -np.sin(t / 2)], [np.sin(t / 2), np.cos(t / 2)]],
                    dtype=np.complex128)


def rz(t):
    return np.array([[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]], dtype=np.complex128)


def ansatz_matrix(n: int, layers: int, theta, entangler: int = 0) -> np.ndarray:
    """V(theta) = product of full gate matrices (applied right to left)."""
    theta = np.asarray(theta, dtype=np.float64)
    V = np.eye(1 << n, dtype=np.complex128)
    for layer in range(layers):
        for q in range(n):
            a, b, c = theta[(layer * n + q) * 3:(layer * n + q) * 3 + 3]
            for G in (ry(a), rz(b), ry(c)):
                V = embed_1q(G, q, n) @ V
        if n >= 2:
            for q in range(n):
                G = X2 if entangler == 0 else Z2
                V = controlled_matrix(G, q, (q + 1) % n, n) @ V
    return V


def ansatz_state(n, layers, theta, entangler=0) -> np.ndarray:
    return ansatz_matrix(n, layers, theta, entangler)[:, 0]


def ub_dense(n: int, bkind: int, b=None) -> np.ndarray:
    if bkind == 0:
        return kron_all([H2] * n)
    b = np.asarray(b, dtype=np.complex128)
    w = b[0] / abs(b[0]) if abs(b[0]) > 0 else 1.0 + 0j
    e0 = np.zeros_like(b)
    e0[0] = 1
    v = e0 - np.conj(w) * b
    vv = np.vdot(v, v).real
    Hh = np.eye(b.size, dtype=np.complex128)
    if vv > 0:
        Hh -= 2.0 * np.outer(v, np.conj(v)) / vv
    return w * Hh


def z_on(j: int, n: int) -> np.ndarray:
    return embed_1q(Z2, j, n)


def term_operator(sl: str, sk: str, s: int, Ub: np.ndarray) -> np.ndarray:
    """B = A_l U_b Z_j U_b^+ A_k (s = 1+j) or A_l A_k (s = 0)   (Eq. 4)."""
    n = len(sl)
    Al, Ak = pauli_matrix(sl), pauli_matrix(sk)
    if s == 0:
        return Al @ Ak
    return Al @ Ub @ z_on(s - 1, n) @ Ub.conj().T @ Ak


def quad(B: np.ndarray, x: np.ndarray) -> complex:
    return complex(np.vdot(x, B @ x))


def all_terms_dense(w, x: np.ndarray) -> np.ndarray:
    """Canonical 2(n+1)L^2 array [Re, Im of <x|B|x> per task] via dense matrices."""
    n, L = w.n, w.L
    Ub = ub_dense(n, w.bkind, w.b)
    out = np.empty(2 * (n + 1) * L * L)
    t = 0
    for l in range(L):
        for k in range(L):
            for s in range(n + 1):
                v = quad(term_operator(w.terms[l][1], w.terms[k][1], s, Ub), x)
                out[2 * t], out[2 * t + 1] = v.real, v.imag
                t += 1
    return out


def local_cost(A: np.ndarray, Ub: np.ndarray, x: np.ndarray, n: int) -> float:
    """Alg. 1 form: 1/2 - (1/2n) sum_j (Ax)^+ U_b Z_j U_b^+ (Ax) / ||Ax||^2."""
    Ax = A @ x
    den = np.vdot(Ax, Ax).real
    num = sum(np.vdot(Ax, Ub @ z_on(j, n) @ Ub.conj().T @ Ax).real for j in range(n))
    return 0.5 - 0.5 * num / (n * den)


def local_cost_eq2(A: np.ndarray, Ub: np.ndarray, x: np.ndarray, n: int) -> float:
    """Eq. 2 read with P_j = Z_j: 1 - (1/n) sum_j <x|A^+ U_b Z_j U_b^+ A|x>/<x|A^+A|x>."""
    Ax = A @ x
    den = np.vdot(Ax, Ax).real
    num = sum(np.vdot(Ax, Ub @ z_on(j, n) @ Ub.conj().T @ Ax).real for j in range(n))
    return 1.0 - num / (n * den)


def global_cost(A: np.ndarray, b: np.ndarray, x: np.ndarray) -> float:
    """Eq. 1: C_G = 1 - |<b|A|x>|^2 / <x|A^+A|x>."""
    Ax = A @ x
    return 1.0 - abs(np.vdot(b, Ax)) ** 2 / np.vdot(Ax, Ax).real


def masks(s: str):
    """(x_mask, z_mask, n_Y) of a big-endian Pauli string (char q <-> bit n-1-q)."""
    n = len(s)
    xm = zm = ny = 0
    for q, ch in enumerate(s):
        bit = 1 << (n - 1 - q)
        if ch in "XY":
            xm |= bit
        if ch in "YZ":
            zm |= bit
        if ch == "Y":
            ny += 1
    return xm, zm, ny


def pauli_expectation(x: np.ndarray, s: str) -> complex:
    """<x|P|x> = sum_i conj(x_i) i^{nY} (-1)^{popcount((i^m)&z)} x_{i^m}, O(2^n).

    Uses P|j> = i^{nY} (-1)^{popcount(j & z)} |j ^ m> (Y = i X Z per factor).
    """
    xm, zm, ny = masks(s)
    idx = np.arange(x.size)
    src = idx ^ xm
    sign = 1.0 - 2.0 * _parity(src & zm)
    return complex((1j ** ny) * np.sum(np.conj(x) * sign * x[src]))


def _parity(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.int64).copy()
    p = np.zeros_like(v)
    while np.any(v):
        p ^= v & 1
        v >>= 1
    return p


def term_closed_form_uniform(x: np.ndarray, sl: str, sk: str, s: int) -> complex:
    """<x|A_l X_j A_k|x> for U_b = H^{(x)n} (H Z H = X) or <x|A_l A_k|x> (s = 0)."""
    n = len(sl)
    if s == 0:
        ph, r = pauli_product(sl, sk)
    else:
        xj = "".join("X" if q == s - 1 else "I" for q in range(n))
        ph1, r1 = pauli_product(xj, sk)
        ph2, r = pauli_product(sl, r1)
        ph = ph1 * ph2
    return ph * pauli_expectation(x, r)
