"""GPU: the parameter-shift gradient (dvqls_cost_grad; NEXT-1 with 2P shift points; SURVEY
§8(c) reading 23) against the oracle's gradient (oracle.cost.workload_gradient: the gate-by-gate
terms at theta +- pi/2 e_p, aggregated, combined by the quotient rule), 1e-10 per component."""

import numpy as np
import pytest

from dvqls_inputs import configs
from oracle import cost as ocost
from oracle import sim

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def dv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_14435_b200 import build, dvqls
    build.build()
    return dvqls


def _terms(w, th):
    return sim.workload_terms(w, th)


@pytest.mark.parametrize("name,mk,max_batch", [
    ("cfg1", configs.cfg1, 16),                                               # chunked: 97 rows / 16
    ("cfg2p", configs.cfg2_pressure, 97),                                     # Householder, one launch
    ("n10", lambda: configs.random_workload(10, 3, 1, seed=31), 8),           # plane kernel
    ("n12", lambda: configs.random_workload(12, 2, 1, seed=32, entangler=1), 16),  # on-chip kernel
    ("n13", lambda: configs.random_workload(13, 2, 1, seed=33), 16),          # streaming kernel
])
def test_shift_gradient_matches_oracle(dv, name, mk, max_batch):
    w = mk()
    th = w.theta0()
    ctx = dv.from_workload(w, max_batch=max_batch)
    try:
        C, g, E, Psi = ctx.cost_grad(th, with_E_Psi=True)
        C2, g2 = ctx.cost_grad(th)  # graph replay: bitwise the same
    finally:
        ctx.destroy()
    Cr, gr = ocost.workload_gradient(w, th, _terms)
    assert abs(C - Cr) <= TOL
    assert np.max(np.abs(g - gr)) <= TOL, np.max(np.abs(g - gr))
    assert C2 == C and np.array_equal(g, g2)


def test_shift_gradient_device_entry_and_fd_agreement(dv):
    """dvqls_cost_grad_dev writes (C, grad, E, Psi) to device memory; the gradient also agrees with a
    central difference of the GPU cost (O(h^2), a check independent of the shift rule)."""
    import torch
    w = configs.cfg1(3)
    th = w.theta0()
    ctx = dv.from_workload(w, max_batch=32)
    try:
        out = torch.zeros(1 + w.n_params + 4, dtype=torch.float64, device="cuda")
        ctx.cost_grad_dev(torch.tensor(th, dtype=torch.float64, device="cuda"), out)
        ctx.check()
        o = out.cpu().numpy()
        C, g = ctx.cost_grad(th)
        h = 1e-5
        fd = np.empty(w.n_params)
        for p in range(w.n_params):
            e = np.zeros(w.n_params)
            e[p] = h
            cb, _ = ctx.cost_batch(np.stack([th + e, th - e]))
            fd[p] = (cb[0] - cb[1]) / (2 * h)
    finally:
        ctx.destroy()
    assert o[0] == C and np.array_equal(o[1:1 + w.n_params], g)
    assert np.max(np.abs(g - fd)) <= 1e-8
