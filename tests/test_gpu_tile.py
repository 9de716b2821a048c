"""GPU parity of the n >= 11 tile path (SMEM tile n <= 12, global streaming n >= 13).

Same bar as the register path: 1e-10 absolute per term and on the cost.  Large n
use dvqls_terms_subset on evenly strided circuits (config 5 samples).
"""

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


@pytest.mark.parametrize("n,L,amp,ent", [(11, 3, False, 0), (11, 2, True, 0), (12, 3, False, 1),
                                         (12, 2, True, 0), (13, 2, False, 0), (14, 2, False, 1)])
def test_full_parity_small_L(dv, n, L, amp, ent):
    w = configs.random_workload(n, L, 2, seed=50 + n, amplitudes=amp, entangler=ent)
    th = w.theta0()
    ctx = dv.from_workload(w)
    try:
        g = ctx.terms(th)
        ref = sim.workload_terms(w, th)
        assert np.max(np.abs(g - ref)) <= TOL
        C, E, Psi = ctx.cost(th, with_E_Psi=True)
        Cr, Er, Pr = ocost.cost(ref, ocost.coeffs_of(w), w.n, w.L)
        assert abs(C - Cr) <= TOL
        x = ctx.state(th)
        assert np.max(np.abs(x - sim.ansatz_state(n, 2, th, ent))) < 1e-12
    finally:
        ctx.destroy()


@pytest.mark.parametrize("n,nsample", [(12, 96), (14, 48), (16, 24), (18, 12), (20, 6)])
def test_cfg5_sampled(dv, n, nsample):
    """Config 5 workload (I^(n-7) (x) pruned tridiag(7), L=64, d=3): strided circuit sample."""
    w = configs.cfg5(n)
    th = w.theta0()
    idx = np.linspace(0, w.n_circuits - 1, nsample).astype(np.int64)
    idx[1::2] |= 1  # mix Re and Im circuits
    ctx = dv.from_workload(w)
    try:
        g = ctx.terms_subset(th, idx)
    finally:
        ctx.destroy()
    ref = sim.workload_terms(w, th, idx=idx)
    assert np.max(np.abs(g - ref)) <= TOL


def test_parameter_shift_pair_cost(dv):
    """Config 5 parameter-shift pair theta +- (pi/2) e_0 at n=12, full cost vs oracle."""
    w = configs.cfg5(12)
    th = w.theta0()
    ctx = dv.from_workload(w)
    try:
        pair = np.stack([th, th])
        pair[0, 0] += np.pi / 2
        pair[1, 0] -= np.pi / 2
        cb, _ = ctx.cost_batch(pair)
    finally:
        ctx.destroy()
    idx = None
    for k in range(2):
        ref = sim.workload_terms(w, pair[k], idx=idx)
        Cr = ocost.cost(ref, ocost.coeffs_of(w), w.n, w.L)[0]
        assert abs(cb[k] - Cr) <= TOL


@pytest.mark.parametrize("n,ent", [(15, 0), (16, 1), (17, 0)])
def test_team_mode_full(dv, n, ent, monkeypatch):
    """n >= 15 with DVQLS_TEAM=1 runs the team kernel (T CTAs per circuit, cooperative launch): full
    terms, cost and a batch of 3 thetas against the oracle."""
    monkeypatch.setenv("DVQLS_TEAM", "1")
    w = configs.random_workload(n, 2, 2, seed=70 + n, entangler=ent)
    ctx = dv.from_workload(w, max_batch=4)
    try:
        th = w.theta0()
        g = ctx.terms(th)
        C = ctx.cost(th)
        ths = np.stack([w.theta0(s) for s in range(3)])
        cb, _ = ctx.cost_batch(ths)
    finally:
        ctx.destroy()
    ref = sim.workload_terms(w, th)
    assert np.max(np.abs(g - ref)) <= TOL
    assert abs(C - ocost.cost(ref, ocost.coeffs_of(w), w.n, w.L)[0]) <= TOL
    for k in range(3):
        rk = sim.workload_terms(w, ths[k])
        assert abs(cb[k] - ocost.cost(rk, ocost.coeffs_of(w), w.n, w.L)[0]) <= TOL


@pytest.mark.parametrize("team", ["0", "1"])
def test_cfg5_n16_full_sampled(dv, team, monkeypatch):
    """Config 5 at n = 16, all 139,264 circuits (per-CTA kernel, and the team kernel with
    DVQLS_TEAM=1), strided sample vs oracle."""
    monkeypatch.setenv("DVQLS_TEAM", team)
    w = configs.cfg5(16)
    th = w.theta0()
    ctx = dv.from_workload(w)
    try:
        g = ctx.terms(th)
    finally:
        ctx.destroy()
    idx = np.linspace(0, w.n_circuits - 1, 24).astype(np.int64)
    idx[1::2] |= 1
    assert np.max(np.abs(g[idx] - sim.workload_terms(w, th, idx=idx))) <= TOL


@pytest.mark.parametrize("n,L,ent", [(11, 3, 0), (12, 2, 1), (13, 2, 0), (14, 2, 0)])
def test_complex_stream_kernel(dv, n, L, ent, monkeypatch):
    """DVQLS_PLANE=0 keeps the complex-layout streaming kernel (uniform b) selectable: full terms
    and a batch of two thetas against the oracle (the default above is the real-plane kernel)."""
    monkeypatch.setenv("DVQLS_PLANE", "0")
    w = configs.random_workload(n, L, 2, seed=90 + n, entangler=ent)
    ctx = dv.from_workload(w, max_batch=2)
    try:
        th = w.theta0()
        g = ctx.terms(th)
        ths = np.stack([w.theta0(s) for s in range(2)])
        cb, _ = ctx.cost_batch(ths)
    finally:
        ctx.destroy()
    assert np.max(np.abs(g - sim.workload_terms(w, th))) <= TOL
    for k in range(2):
        rk = sim.workload_terms(w, ths[k])
        assert abs(cb[k] - ocost.cost(rk, ocost.coeffs_of(w), w.n, w.L)[0]) <= TOL
