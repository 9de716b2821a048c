"""ORACLE - TEST INFRASTRUCTURE ONLY.  ctypes front-end of oracle/sim.cpp.

The C++ library is compiled here on first use (plain ``g++ -O2``; no -ffast-math,
no -march flags, so no FMA contraction or vectorised reassociation).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sim.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-fcx-limited-range", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            L.oracle_terms.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                       ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_int,
                                       ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.c_int64, dp]
            L.oracle_terms.restype = ctypes.c_int
            L.oracle_ansatz_state.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp]
            L.oracle_ansatz_state.restype = ctypes.c_int
            L.oracle_ub_matrix.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp]
            L.oracle_ub_matrix.restype = ctypes.c_int
            L.oracle_hardware_threads.restype = ctypes.c_int
            L.oracle_set_householder_form.argtypes = [ctypes.c_int]
            L.oracle_set_householder_form.restype = ctypes.c_int
            L.oracle_overlap_terms.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                               ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_int, dp]
            L.oracle_overlap_terms.restype = ctypes.c_int
            _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def _interleave(z):
    z = np.ascontiguousarray(z, dtype=np.complex128)
    return z.view(np.float64).copy()


def set_householder_form(form: int) -> int:
    """Test hook: how the oracle applies an amplitude-b U_b (0 = dense matrix for n <= 12, else
    from the definition w(I - 2vv^+/v^+v); 1 = definition form at every n; 2 = dense).  Returns
    the previous setting."""
    return int(lib().oracle_set_householder_form(int(form)))


def hardware_threads() -> int:
    return int(lib().oracle_hardware_threads())


def terms(n, layers, paulis: bytes, theta, bkind=0, b=None, entangler=0, mode=1,
          nthreads=0, idx=None) -> np.ndarray:
    """<Z_anc> of circuits (all 2(n+1)L^2 in canonical order, or those in idx).

    mode 0 = faithful (ansatz per circuit), 1 = prefix-shared (bitwise identical).
    """
    L = len(paulis) // n
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    assert theta.size == 3 * n * layers, "theta must have P = 3 n d entries"
    bamps = _interleave(b) if (bkind == 1) else None
    if idx is None:
        count = 2 * (n + 1) * L * L
        ip = None
    else:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        count = idx.size
        ip = idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    out = np.empty(count, dtype=np.float64)
    rc = lib().oracle_terms(n, layers, L, paulis, entangler, bkind, _dp(bamps), _dp(theta),
                            mode, nthreads, ip, count, _dp(out))
    if rc != 0:
        raise ValueError(f"oracle_terms failed rc={rc}")
    return out


def ansatz_state(n, layers, theta, entangler=0) -> np.ndarray:
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    assert theta.size == 3 * n * layers
    out = np.empty(2 << n, dtype=np.float64)
    if lib().oracle_ansatz_state(n, layers, entangler, _dp(theta), _dp(out)) != 0:
        raise ValueError("oracle_ansatz_state failed")
    return out.view(np.complex128)


def ub_matrix(n, bkind, b=None) -> np.ndarray:
    N = 1 << n
    out = np.empty(2 * N * N, dtype=np.float64)
    bamps = _interleave(b) if bkind == 1 else None
    if lib().oracle_ub_matrix(n, bkind, _dp(bamps), _dp(out)) != 0:
        raise ValueError("oracle_ub_matrix failed")
    return out.view(np.complex128).reshape(N, N)


def workload_terms(w, theta=None, mode=1, nthreads=0, idx=None) -> np.ndarray:
    """Convenience: terms of a dvqls_inputs.configs.Workload."""
    chars, _ = w.arrays()
    th = w.theta0() if theta is None else theta
    return terms(w.n, w.layers, chars, th, w.bkind, w.b, w.entangler, mode, nthreads, idx)


def overlap_terms(n, layers, paulis: bytes, theta, bkind=0, b=None, entangler=0, nthreads=0) -> np.ndarray:
    """NEXT-3: 2L values, [2l + part] = Re / Im <b|A_l|x> from the gate-by-gate overlap
    Hadamard test (controlled V, controlled A_l, controlled U_b^+)."""
    L = len(paulis) // n
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    assert theta.size == 3 * n * layers
    bamps = _interleave(b) if (bkind == 1) else None
    out = np.empty(2 * L, dtype=np.float64)
    rc = lib().oracle_overlap_terms(n, layers, L, paulis, entangler, bkind, _dp(bamps), _dp(theta), nthreads,
                                    _dp(out))
    if rc != 0:
        raise ValueError(f"oracle_overlap_terms failed rc={rc}")
    return out


def workload_overlaps(w, theta=None, nthreads=0) -> np.ndarray:
    chars, _ = w.arrays()
    th = w.theta0() if theta is None else theta
    return overlap_terms(w.n, w.layers, chars, th, w.bkind, w.b, w.entangler, nthreads)
