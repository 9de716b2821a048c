"""ORACLE - TEST INFRASTRUCTURE ONLY (NEXT-4: Pauli decomposition + pruning of a dense A).

Alg. 1 Steps 1-2: decompose A = sum_P c_P P over all 4^n Pauli strings,
then keep the terms above 1 % of the l2 norm, as definitions written out:

  c_P = tr(P^+ A) / 2^n = tr(P A) / 2^n                       (P Hermitian)

With P = P(m, z) acting as P|k> = i^{popcount(m & z)} (-1)^{popcount(k & z)} |k ^ m>
(x-mask m, z-mask z, big-endian bits; n_Y = popcount(m & z)), the only nonzero entries of P
are P[k ^ m, k], so the trace is the plain sum

  tr(P A) = sum_k P[k ^ m, k] A[k, k ^ m] = i^{popcount(m & z)} sum_k (-1)^{popcount(k & z)} A[k, k ^ m].

For each m this is the Walsh matrix W[z, k] = (-1)^{popcount(z & k)} (the definition of the
+-1 matrix, built entry by entry) times the vector B[:, m] = A[k, k ^ m]: one library matmul
W @ B over all m.  No fast transform, no blocking.

Pruning (SURVEY.md §8(c) reading 15): drop |c| < 1e-14, keep |c| >= eps * ||c||_2 (inclusive,
||c||_2 = sqrt(sum_P |c_P|^2)), order by descending |c| then lexicographic with I<X<Y<Z.
Magnitudes within 1e-12 * ||c||_2 of each other are ties (reading 15b): the key is
round(|c| / (1e-12 * ||c||_2)), an integer, so both sides order ties identically.
"""

from __future__ import annotations

import numpy as np

CHARS = "IXYZ"


def walsh_matrix(n: int) -> np.ndarray:
    N = 1 << n
    k = np.arange(N)
    pc = np.zeros((N, N), dtype=np.int64)
    zk = k[:, None] & k[None, :]
    for b in range(n):
        pc += (zk >> b) & 1
    return np.where(pc & 1, -1.0, 1.0)


def coefficients(A: np.ndarray) -> np.ndarray:
    """C[m, z] = c_{P(m, z)} for all x-masks m and z-masks z (4^n values)."""
    A = np.asarray(A, dtype=np.complex128)
    N = A.shape[0]
    n = N.bit_length() - 1
    k = np.arange(N)
    B = np.empty((N, N), dtype=np.complex128)  # B[k, m] = A[k, k ^ m]
    for m in range(N):
        B[:, m] = A[k, k ^ m]
    S = walsh_matrix(n) @ B  # S[z, m] = sum_k (-1)^{popcount(z & k)} A[k, k ^ m]
    m = np.arange(N)[None, :]
    z = np.arange(N)[:, None]
    ny = np.zeros((N, N), dtype=np.int64)
    mz = m & z
    for b in range(n):
        ny += (mz >> b) & 1
    phase = (1j) ** (ny % 4)
    return (phase * S / N).T  # [m, z]


def pauli_string(m: int, z: int, n: int) -> str:
    """Big-endian: character q <-> index bit n-1-q; (x, z) bits -> I, X, Y, Z."""
    out = []
    for q in range(n):
        b = n - 1 - q
        xb, zb = (m >> b) & 1, (z >> b) & 1
        out.append("I" if not xb and not zb else "X" if xb and not zb else "Y" if xb else "Z")
    return "".join(out)


def lex_code(m: int, z: int, n: int) -> int:
    """Integer whose order equals the lexicographic order of the string (I<X<Y<Z)."""
    code = 0
    for q in range(n):
        b = n - 1 - q
        xb, zb = (m >> b) & 1, (z >> b) & 1
        d = 0 if not xb and not zb else 1 if xb and not zb else 2 if xb else 3
        code = code * 4 + d
    return code


def decompose_pruned(A: np.ndarray, eps: float):
    """[(c, string)] after pruning and canonical ordering, plus ||c||_2."""
    C = coefficients(A)
    N = C.shape[0]
    n = N.bit_length() - 1
    norm = float(np.sqrt(np.sum(np.abs(C) ** 2)))
    out = []
    for m in range(N):
        for z in range(N):
            a = abs(C[m, z])
            if a >= 1e-14 and a >= eps * norm:
                out.append((C[m, z], m, z))
    q = 1e-12 * norm
    out.sort(key=lambda t: (-int(round(abs(t[0]) / q)), lex_code(t[1], t[2], n)))
    return [(complex(c), pauli_string(m, z, n)) for c, m, z in out], norm


def coefficient(A: np.ndarray, m: int, z: int) -> complex:
    """One coefficient by the same definition, O(2^n): i^{popcount(m & z)} / 2^n *
    sum_k (-1)^{popcount(k & z)} A[k, k ^ m] (for sampled checks at sizes where the full
    4^n transform by matmul is too slow)."""
    A = np.asarray(A)
    N = A.shape[0]
    k = np.arange(N)
    kz = k & z
    par = np.zeros(N, dtype=np.int64)
    for b in range(N.bit_length() - 1):
        par ^= (kz >> b) & 1
    s = np.sum(np.where(par == 1, -1.0, 1.0) * A[k, k ^ m])
    return complex((1j) ** (bin(m & z).count("1") % 4) * s / N)
