"""ORACLE - TEST INFRASTRUCTURE ONLY.

Alg. 1 Steps 4b-4c, written out as plain loops over the
canonical task order (SURVEY.md §8 notation; reading 17):

    E   = sum_{l,k} sum_{j} c_l^* c_k (Re + i Im)_{num(l,k,j)}     (Step 4b)
    Psi = sum_{l,k}         c_l^* c_k (Re + i Im)_{den(l,k)}       (Step 4b)
    C   = 1/2 - 1/2 * Re E / (n * Re Psi)                          (Step 4c)

The real parts are used in C (reading 12); Re Psi <= 1e-12 is an error
(reading 13).
"""

from __future__ import annotations

import numpy as np


class DegenerateDenominator(ValueError):
    pass


def aggregate(terms: np.ndarray, coeffs, n: int, L: int, circuits=None):
    """(E, Psi) from term expectations.

    ``terms[i]`` is the value of circuit ``circuits[i]`` (default: all circuits in
    canonical order c = 2t + part).
    """
    c = np.asarray(coeffs, dtype=np.complex128)
    E = 0j
    Psi = 0j
    idx = range(len(terms)) if circuits is None else None
    items = zip(idx, terms) if circuits is None else zip(circuits, terms)
    for circ, val in items:
        t, part = divmod(int(circ), 2)
        s = t % (n + 1)
        k = (t // (n + 1)) % L
        l = t // ((n + 1) * L)
        w = np.conj(c[l]) * c[k]
        contrib = w * (val if part == 0 else 1j * val)
        if s == 0:
            Psi += contrib
        else:
            E += contrib
    return complex(E), complex(Psi)


def cost_from(E: complex, Psi: complex, n: int) -> float:
    if Psi.real <= 1e-12:
        raise DegenerateDenominator(f"Re Psi = {Psi.real} <= 1e-12")
    return 0.5 - 0.5 * E.real / (n * Psi.real)


def cost(terms: np.ndarray, coeffs, n: int, L: int):
    E, Psi = aggregate(terms, coeffs, n, L)
    return cost_from(E, Psi, n), E, Psi


def coeffs_of(w) -> np.ndarray:
    return np.array([c for c, _ in w.terms], dtype=np.complex128)


def global_cost(overlaps: np.ndarray, coeffs, Psi: complex) -> float:
    """NEXT-3, Eq. 1: C_G = 1 - |<b|A|x>|^2 / <x|A^+A|x>, with
    <b|A|x> = sum_l c_l beta_l (beta_l = Re + i Im of the overlap Hadamard tests) and
    <x|A^+A|x> = Re Psi, the local cost's denominator sum (Alg. 1 Step 4b)."""
    c = np.asarray(coeffs, dtype=np.complex128)
    beta = np.asarray(overlaps[0::2]) + 1j * np.asarray(overlaps[1::2])
    s = 0j
    for l in range(len(c)):
        s += c[l] * beta[l]
    if Psi.real <= 1e-12:
        raise DegenerateDenominator(f"Re Psi = {Psi.real} <= 1e-12")
    return 1.0 - abs(s) ** 2 / Psi.real


def shift_gradient(E_plus, Psi_plus, E_minus, Psi_minus, E0: complex, Psi0: complex, n: int) -> np.ndarray:
    """Parameter-shift gradient of C (SURVEY §8(c) reading 23; "parameter-shift
    gradients"), written out step by step.  Every parameter enters V(theta) through one
    exp(-i theta sigma/2), so each term f obeys df/dtheta_p = [f(theta + pi/2 e_p) - f(theta -
    pi/2 e_p)] / 2; Re E and Re Psi are fixed linear combinations of terms (Step 4b), hence
        dReE_p   = (Re E(theta + pi/2 e_p)   - Re E(theta - pi/2 e_p))   / 2
        dRePsi_p = (Re Psi(theta + pi/2 e_p) - Re Psi(theta - pi/2 e_p)) / 2
    and C = 1/2 - Re E / (2 n Re Psi) (Step 4c) by the quotient rule:
        dC/dtheta_p = -(dReE_p Re Psi - Re E dRePsi_p) / (2 n Re Psi^2).
    E_plus[p], Psi_plus[p] (E_minus, Psi_minus) are the sums at theta +(-) pi/2 e_p."""
    if Psi0.real <= 1e-12:
        raise DegenerateDenominator(f"Re Psi = {Psi0.real} <= 1e-12")
    P = len(E_plus)
    g = np.empty(P)
    for p in range(P):
        dE = (E_plus[p].real - E_minus[p].real) / 2
        dPsi = (Psi_plus[p].real - Psi_minus[p].real) / 2
        g[p] = -(dE * Psi0.real - E0.real * dPsi) / (2 * n * Psi0.real ** 2)
    return g


def workload_gradient(w, theta, terms_fn):
    """(C, dC/dtheta) of a workload at theta: the 2P shifted term arrays from ``terms_fn(w,
    theta)`` (the gate-by-gate simulator), aggregated and combined by shift_gradient."""
    co = coeffs_of(w)
    C0, E0, Psi0 = cost(terms_fn(w, theta), co, w.n, w.L)
    Ep, Pp, Em, Pm = [], [], [], []
    for p in range(len(theta)):
        e = np.zeros(len(theta))
        e[p] = np.pi / 2
        a = aggregate(terms_fn(w, theta + e), co, w.n, w.L)
        b = aggregate(terms_fn(w, theta - e), co, w.n, w.L)
        Ep.append(a[0]); Pp.append(a[1]); Em.append(b[0]); Pm.append(b[1])
    return C0, shift_gradient(Ep, Pp, Em, Pm, E0, Psi0, w.n)
