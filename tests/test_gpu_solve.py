"""GPU: the full D-VQLS loop (BASELINE config 2) - L-BFGS-B on dvqls_cost_batch.

Pin: fidelity F = |<x(theta*)|x*>|^2 > 0.9999 against the classical solution
x* = A^{-1} b of the same 4x4 Hele-Shaw systems (PAPER.md P:29-31, P:40-52:
"fidelity results exceeding 0.9999").  Budget 20,000 cost evaluations (SURVEY
§8(c) reading 22; the paper's 3-4K / 9-10K counts are context).
"""

import numpy as np
import pytest

from dvqls_inputs import configs
from oracle import sim

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_14435_b200 import build, dvqls, optimize
    build.build()
    return dvqls, optimize


def test_state_matches_oracle_ansatz(dv):
    dvqls, _ = dv
    for w in (configs.cfg1(), configs.cfg3(), configs.random_workload(7, 3, 2, seed=4, entangler=1)):
        ctx = dvqls.from_workload(w)
        try:
            th = w.theta0(2)
            x = ctx.state(th)
            assert np.max(np.abs(x - sim.ansatz_state(w.n, w.layers, th, w.entangler))) < 1e-12
        finally:
            ctx.destroy()


@pytest.mark.parametrize("which", ["velocity", "pressure"])
def test_hele_shaw_converges_to_classical_solution(dv, which):
    dvqls, optimize = dv
    mk = configs.cfg2_velocity if which == "velocity" else configs.cfg2_pressure
    hits = []
    for seed in range(5):
        w = mk(seed)
        ctx = dvqls.from_workload(w, max_batch=w.n_params + 1)
        try:
            res = optimize.solve(ctx, w.theta0(), max_evals=20000, target_cost=1e-10)
            x = ctx.state(res.theta)
        finally:
            ctx.destroy()
        xstar = np.linalg.solve(w.A, w.rhs)
        F = optimize.fidelity(x, xstar.astype(complex))
        hits.append(F > 0.9999)
        print(f"{w.name} seed {seed}: C={res.cost:.3e} F={F:.6f} evals={res.n_evals} {res.seconds:.2f}s")
    assert sum(hits) >= 4, hits
