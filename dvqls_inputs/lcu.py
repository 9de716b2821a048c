"""LCU inputs: A = sum_l c_l A_l with Pauli-string A_l.

Alg. 1 Step 1 decomposes A "via FWHT-based Pauli decomposition"
(P:379); Step 2 prunes terms below 1 % of the l2 norm.  This
is one-off pre-processing of the hot path's input, done here in numpy:

* ``decompose`` - the recursive 2x2 block transform of SPEC.md S:100: with
  A = [[A00, A01], [A10, A11]] split on the leading (most significant) qubit,
  I <- (A00+A11)/2, X <- (A01+A10)/2, Y <- i(A01-A10)/2, Z <- (A00-A11)/2,
  recursing on every block.  O(4^n n) work (the paper's "O(n^2 log n)" cannot
  hold, SURVEY.md §8(c) reading 24).
* ``prune`` - keep |c| >= eps * ||c_full||_2 (inclusive), after dropping
  |c| < 1e-14 dust; order by descending |c| then lexicographic I<X<Y<Z
  (SURVEY.md §8(c) reading 15).

Pauli strings are big-endian: character q acts on qubit q = the most
significant index bit first (SURVEY.md §8(c) reading 9).  Pins live in
tests/test_inputs_lcu.py (brute-force trace formula from ``oracle.dense``,
Table II term counts).
"""

from __future__ import annotations

import numpy as np

PAULI_CHARS = "IXYZ"


def decompose(A: np.ndarray):
    """Return (coeffs[4^n] complex128, source_norm) indexed by base-4 string code.

    Code digit order: qubit 0 is the most significant base-4 digit, digit
    values I=0, X=1, Y=2, Z=3.
    """
    A = np.asarray(A, dtype=np.complex128)
    N = A.shape[0]
    if A.ndim != 2 or A.shape[1] != N or N & (N - 1) or N < 2:
        raise ValueError("decompose: A must be square with power-of-two dimension >= 2")
    n = N.bit_length() - 1
    blocks = A[None, :, :]
    for _ in range(n):
        h = blocks.shape[1] // 2
        a00 = blocks[:, :h, :h]
        a01 = blocks[:, :h, h:]
        a10 = blocks[:, h:, :h]
        a11 = blocks[:, h:, h:]
        nxt = np.stack(
            [(a00 + a11) / 2, (a01 + a10) / 2, 1j * (a01 - a10) / 2, (a00 - a11) / 2], axis=1
        )
        blocks = nxt.reshape(-1, h, h)
    coeffs = blocks.reshape(-1)
    return coeffs, float(np.linalg.norm(coeffs))


def code_to_string(code: int, n: int) -> str:
    s = []
    for q in range(n):
        s.append(PAULI_CHARS[(code >> (2 * (n - 1 - q))) & 3])
    return "".join(s)


def prune(coeffs: np.ndarray, source_norm: float, n: int, eps: float):
    """Pruned, canonically ordered LCU as a list of (coefficient, pauli_string)."""
    if not 0.0 <= eps < 1.0:
        raise ValueError("prune: eps out of range")
    mags = np.abs(coeffs)
    keep = np.nonzero((mags >= 1e-14) & (mags >= eps * source_norm))[0]
    terms = [(complex(coeffs[c]), code_to_string(int(c), n)) for c in keep]
    # descending |c| (rounded to 12 significant digits so fp dust cannot reorder
    # equal-magnitude groups), then lexicographic with I<X<Y<Z (ASCII order works)
    terms.sort(key=lambda t: (-float(f"{abs(t[0]):.12e}"), t[1]))
    return terms


def decompose_pruned(A: np.ndarray, eps: float):
    coeffs, norm = decompose(A)
    n = A.shape[0].bit_length() - 1
    return prune(coeffs, norm, n, eps)


def identity_padded(terms, n_pad: int):
    """I^{(x) n_pad} (x) A: prepend n_pad identity factors (SURVEY.md §8(d) cfg 5)."""
    return [(c, "I" * n_pad + s) for c, s in terms]


def to_arrays(terms):
    """(pauli_chars bytes [L*n], coeffs float64 [2L] interleaved re,im) for the C ABIs."""
    n = len(terms[0][1])
    chars = "".join(s for _, s in terms).encode("ascii")
    assert len(chars) == n * len(terms)
    co = np.empty(2 * len(terms), dtype=np.float64)
    co[0::2] = [c.real for c, _ in terms]
    co[1::2] = [c.imag for c, _ in terms]
    return chars, co
