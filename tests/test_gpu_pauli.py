"""GPU parity of the NEXT-2 algebraic fast path (opts.mode = DVQLS_MODE_PAULI, pauli.cuh):
the same term array and cost as the gate-by-gate oracle, 1e-10 absolute (the circuit path's
bar), on uniform-b workloads (the only ones the identity U_b Z_j U_b^+ = X_j covers)."""

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


def _check(dv, w, idx=None):
    th = w.theta0()
    ctx = dv.from_workload(w, mode=dv.DVQLS_MODE_PAULI)
    try:
        assert 0 < ctx.num_observables() <= w.n_tasks
        g = ctx.terms(th) if idx is None else ctx.terms_subset(th, idx)
        C, E, Psi = ctx.cost(th, with_E_Psi=True)
        thetas = np.stack([w.theta0(s) for s in range(3)])
        cb, _ = ctx.cost_batch(thetas)
    finally:
        ctx.destroy()
    ref = sim.workload_terms(w, th, idx=idx)
    assert np.max(np.abs(g - ref)) <= TOL
    if idx is None:
        Cr, Er, Pr = ocost.cost(ref, ocost.coeffs_of(w), w.n, w.L)
        assert abs(C - Cr) <= TOL
        assert abs(E - Er) <= TOL * max(1.0, abs(Er)) and abs(Psi - Pr) <= TOL * max(1.0, abs(Pr))
        for s in range(3):
            rs = sim.workload_terms(w, thetas[s])
            assert abs(cb[s] - ocost.cost(rs, ocost.coeffs_of(w), w.n, w.L)[0]) <= TOL


def test_cfg1(dv):
    _check(dv, configs.cfg1())


def test_hele_shaw_velocity(dv):
    _check(dv, configs.cfg2_velocity())


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 10])
def test_random_lcu(dv, n):
    _check(dv, configs.random_workload(n, min(5, 4 ** n), 2, seed=300 + n))


def test_cz_ring(dv):
    _check(dv, configs.random_workload(6, 4, 3, seed=9, entangler=1))


def test_cfg3_full(dv):
    _check(dv, configs.cfg3())


def test_cfg5_n14_sampled(dv):
    w = configs.cfg5(14)
    idx = np.linspace(0, w.n_circuits - 1, 64).astype(np.int64)
    idx[1::2] |= 1
    _check(dv, w, idx=idx)


def test_amplitude_b_rejected(dv):
    w = configs.cfg2_pressure()
    with pytest.raises(dv.DvqlsError) as e:
        dv.from_workload(w, mode=dv.DVQLS_MODE_PAULI)
    assert e.value.code == dv.DVQLS_E_UNSUPPORTED
