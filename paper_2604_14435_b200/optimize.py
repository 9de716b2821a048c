"""Host optimiser loop of D-VQLS (Alg. 1 while-loop).

SciPy L-BFGS-B over theta in [-2pi, 2pi]^P with the finite-difference
gradient SciPy would use by default (forward differences, step 1e-8, P+1 cost
evaluations per gradient, SURVEY §8(c) reading 20) -- but the P+1 points of each
gradient are evaluated in ONE batched call (dvqls_cost_batch), so every cost
evaluation of the loop runs on the GPU path and the launch/allreduce latency is
amortised over the batch.  Evaluation counts are reported
in cost evaluations (P+1 per gradient), the unit the paper's budgets use.

gradient="shift" instead takes the exact parameter-shift gradient of the library
(dvqls_cost_grad: 2P + 1 cost evaluations per gradient, every circuit simulated; P:13,
SURVEY §8(c) reading 23) as L-BFGS-B's jac.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
from scipy.optimize import minimize

from .dvqls import Context


@dataclass
class SolveResult:
    theta: np.ndarray
    cost: float
    n_evals: int
    n_iter: int
    seconds: float
    message: str


def solve(ctx: Context, theta0, max_evals: int = 20000, fd_step: float = 1e-8, target_cost: float = 0.0,
          gtol: float = 1e-12, ftol: float = 1e-16, gradient: str = "fd") -> SolveResult:
    P = ctx.P
    if gradient not in ("fd", "shift"):
        raise ValueError("gradient must be 'fd' or 'shift'")
    if gradient == "fd" and ctx.max_batch < P + 1:
        raise ValueError(f"context max_batch={ctx.max_batch} < P+1={P + 1} (needed for batched FD)")
    per_grad = P + 1 if gradient == "fd" else 2 * P + 1
    evals = [0]
    best = [np.inf, np.asarray(theta0, dtype=np.float64).copy()]

    class _Stop(Exception):
        pass

    def fun_grad(th):
        if gradient == "shift":
            f, g = ctx.cost_grad(th)
            evals[0] += 2 * P + 1
            if f < best[0]:
                best[0], best[1] = f, th.copy()
            return f, g
        pts = np.repeat(th[None, :], P + 1, axis=0)
        pts[1:] += fd_step * np.eye(P)
        c, _ = ctx.cost_batch(pts)
        evals[0] += P + 1
        f = float(c[0])
        g = (c[1:] - f) / fd_step
        if f < best[0]:
            best[0], best[1] = f, th.copy()
        return f, g

    def cb(xk):
        if best[0] <= target_cost or evals[0] >= max_evals:
            raise _Stop

    t0 = time.perf_counter()
    bounds = [(-2 * np.pi, 2 * np.pi)] * P
    try:
        res = minimize(fun_grad, np.asarray(theta0, dtype=np.float64), jac=True, method="L-BFGS-B",
                       bounds=bounds, callback=cb,
                       options={"maxfun": max(1, max_evals // per_grad), "maxiter": 10 ** 6,
                                "gtol": gtol, "ftol": ftol, "maxcor": 20})
        msg, nit = str(res.message), int(res.nit)
    except _Stop:
        msg, nit = "stopped: target cost or evaluation budget reached", -1
    return SolveResult(best[1], best[0], evals[0], nit, time.perf_counter() - t0, msg)


def fidelity(psi: np.ndarray, phi: np.ndarray) -> float:
    """F = |<psi|phi>|^2 of normalised states."""
    psi = psi / np.linalg.norm(psi)
    phi = phi / np.linalg.norm(phi)
    return float(abs(np.vdot(psi, phi)) ** 2)
