"""GPU parity of the n = 10 real-plane Hadamard-test kernel (csrc/plane.cuh) and of the
complex-layout kernel it replaced as the default (DVQLS_PLANE=0), both vs the CPU oracle.

The plane kernel splits each circuit's branch into Re/Im planes on a warp pair and combines
the two readout halves every 8 circuits, so the cases below cover: the Im readout path
(non-Hermitian random LCUs), circuit ranges that end mid-batch (L values whose circuit
counts are not multiples of 8 per pair), a batch of thetas flattened over one grid, and
the bitwise determinism of repeated calls.  Tolerance 1e-10 (BASELINE.json north_star).
"""

import os

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
    dvqls.load()
    return dvqls


def _ctx(dv, w, plane):
    old = os.environ.get("DVQLS_PLANE")
    os.environ["DVQLS_PLANE"] = "1" if plane else "0"
    try:
        return dv.from_workload(w)
    finally:
        if old is None:
            del os.environ["DVQLS_PLANE"]
        else:
            os.environ["DVQLS_PLANE"] = old


@pytest.mark.parametrize("plane", [True, False])
@pytest.mark.parametrize("L,seed", [(3, 1), (5, 2), (7, 3)])
def test_random_lcu_n10(dv, plane, L, seed):
    w = configs.random_workload(10, L, 2, seed=200 + seed)
    ctx = _ctx(dv, w, plane)
    try:
        th = w.theta0()
        g = ctx.terms(th)
        ref = sim.workload_terms(w, th)
        assert np.max(np.abs(g - ref)) <= TOL
        C, E, Psi = ctx.cost(th, with_E_Psi=True)
        Cr, Er, Pr = ocost.cost(ref, ocost.coeffs_of(w), w.n, w.L)
        assert abs(C - Cr) <= TOL and abs(E - Er) <= TOL * max(1, abs(Er))
    finally:
        ctx.destroy()


@pytest.mark.parametrize("plane", [True, False])
def test_theta_batch_n10(dv, plane):
    """K thetas in one flattened grid: every cost equals the oracle's for its theta."""
    w = configs.random_workload(10, 4, 2, seed=211)
    ctx = _ctx(dv, w, plane)
    try:
        ths = np.stack([w.theta0(s) for s in range(6)])
        cb, _ = ctx.cost_batch(ths)
        for k in range(len(ths)):
            ref = ocost.cost(sim.workload_terms(w, ths[k]), ocost.coeffs_of(w), w.n, w.L)[0]
            assert abs(cb[k] - ref) <= TOL
            assert abs(cb[k] - ctx.cost(ths[k])) <= 1e-14
    finally:
        ctx.destroy()


def test_plane_matches_complex_cfg3(dv):
    """Full cfg3 term array: plane and complex kernels agree to rounding; plane is deterministic."""
    w = configs.cfg3()
    th = w.theta0(5)
    a = _ctx(dv, w, True)
    b = _ctx(dv, w, False)
    try:
        ta, tb = a.terms(th), b.terms(th)
        assert np.max(np.abs(ta - tb)) <= 1e-12
        assert np.array_equal(ta, a.terms(th))
        assert abs(a.cost(th) - b.cost(th)) <= 1e-12
    finally:
        a.destroy()
        b.destroy()
