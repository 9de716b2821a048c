"""Benchmark linear systems of the paper, as dense numpy inputs.

* Tridiagonal Toeplitz (§II-D1 matrix display P:479-487):
  A[i,i] = a, A[i,i+1] = b, A[i+1,i] = c.  The paper never states (a, b, c);
  SURVEY.md §8(c) reading 4 takes (2, -1, -1) (the 1-D Laplacian stencil) and
  the uniform rhs (reading 3), so U_b = H^{(x)n}.
* Hele-Shaw flow on a 4x4 interior grid ("second-order finite
  differences", "Dirichlet and Neumann boundary conditions", SPD).  The
  discretisation is unstated; SURVEY.md §8(c) reading 21 fixes it:
  - pressure: 5-point -Laplacian, Dirichlet p_in = 1 (left) / p_out = 0 (right)
    folded into the rhs, face-centred mirror Neumann (ghost = self) top/bottom;
  - velocity: same stencil, Dirichlet 0 top/bottom (no-slip), mirror Neumann
    left/right, rhs = -dp/dx from the central difference of the solved pressure.
  Unknown (row y, column x) has index y*G + x (row-major; big-endian qubits).
"""

from __future__ import annotations

import numpy as np


def tridiag_toeplitz(n: int, a: float = 2.0, b: float = -1.0, c: float = -1.0):
    """Dense 2^n x 2^n tridiagonal Toeplitz matrix and its normalised uniform rhs."""
    N = 1 << n
    A = np.zeros((N, N), dtype=np.float64)
    idx = np.arange(N)
    A[idx, idx] = a
    A[idx[:-1], idx[:-1] + 1] = b
    A[idx[:-1] + 1, idx[:-1]] = c
    rhs = np.full(N, 1.0 / np.sqrt(N))
    return A, rhs


def _laplacian_2d(G: int, dirichlet_lr: bool, dirichlet_tb: bool) -> np.ndarray:
    """5-point -Laplacian (unit spacing) on a G x G interior grid.

    A Dirichlet face keeps the diagonal 4 (the ghost value goes to the rhs);
    a mirror-Neumann face (ghost = self) removes 1 from the diagonal.
    """
    N = G * G
    A = np.zeros((N, N), dtype=np.float64)
    for y in range(G):
        for x in range(G):
            i = y * G + x
            diag = 4.0
            for dy, dx in ((0, -1), (0, 1), (-1, 0), (1, 0)):
                yy, xx = y + dy, x + dx
                if 0 <= yy < G and 0 <= xx < G:
                    A[i, yy * G + xx] = -1.0
                else:
                    lr_face = dx != 0
                    dirichlet = dirichlet_lr if lr_face else dirichlet_tb
                    if not dirichlet:
                        diag -= 1.0
            A[i, i] = diag
    return A


def hele_shaw_pressure(G: int = 4, p_in: float = 1.0, p_out: float = 0.0):
    """Pressure system (nabla^2 p = 0): returns (A, rhs_unnormalised)."""
    A = _laplacian_2d(G, dirichlet_lr=True, dirichlet_tb=False)
    rhs = np.zeros(G * G)
    for y in range(G):
        rhs[y * G + 0] += p_in
        rhs[y * G + (G - 1)] += p_out
    return A, rhs


def hele_shaw_velocity(G: int = 4, p_in: float = 1.0, p_out: float = 0.0):
    """Velocity system (nabla^2 u = grad p): returns (A, rhs_unnormalised)."""
    Ap, rp = hele_shaw_pressure(G, p_in, p_out)
    p = np.linalg.solve(Ap, rp).reshape(G, G)
    A = _laplacian_2d(G, dirichlet_lr=False, dirichlet_tb=True)
    rhs = np.zeros(G * G)
    for y in range(G):
        for x in range(G):
            left = p[y, x - 1] if x > 0 else p_in
            right = p[y, x + 1] if x < G - 1 else p_out
            rhs[y * G + x] = -(right - left) / 2.0  # -dp/dx, central difference
    return A, rhs


def normalise(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.complex128)
    return v / np.linalg.norm(v)
