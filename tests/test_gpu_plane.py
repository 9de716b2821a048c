"""GPU parity of the n = 10 real-plane Hadamard-test kernel (csrc/plane.cuh, the headline kernel)
vs the CPU oracle, and of its launch variants (CUDA-graph replay, programmatic dependent launch).

The plane kernel splits each circuit's branch into Re/Im planes on a warp pair and combines
the two readout halves every 8 circuits, so the cases below cover: the Im readout path
(non-Hermitian random LCUs), circuit ranges that end mid-batch (L values whose circuit
counts are not multiples of 8 per pair), a batch of thetas flattened over one grid, and
the bitwise determinism of repeated calls.  Tolerance 1e-10 (BASELINE.json north_star).
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
    dvqls.load()
    return dvqls


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("L,seed", [(3, 1), (5, 2), (7, 3)])
def test_random_lcu_n10(dv, L, seed, variant):
    w = configs.random_workload(10, L, 2, seed=200 + seed)
    ctx = dv.from_workload(w, variant=variant)
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


@pytest.mark.parametrize("variant", [1, 2])
def test_theta_batch_n10(dv, variant):
    """K thetas in one flattened grid: every cost equals the oracle's for its theta."""
    w = configs.random_workload(10, 4, 2, seed=211)
    ctx = dv.from_workload(w, variant=variant)
    try:
        ths = np.stack([w.theta0(s) for s in range(6)])
        cb, _ = ctx.cost_batch(ths)
        for k in range(len(ths)):
            ref = ocost.cost(sim.workload_terms(w, ths[k]), ocost.coeffs_of(w), w.n, w.L)[0]
            assert abs(cb[k] - ref) <= TOL
            assert abs(cb[k] - ctx.cost(ths[k])) <= 1e-14
    finally:
        ctx.destroy()


def test_cfg3_launch_variants_bitwise(dv):
    """Full cfg3: the plain launch sequence, the CUDA-graph replay (default) and the graph without
    programmatic dependent launch give bitwise identical terms and costs (K = 1 and K = 16)."""
    import torch
    w = configs.cfg3()
    ths = np.stack([w.theta0(s) for s in range(16)])
    ctxs = [dv.from_workload(w, graphs=False, pdl=False), dv.from_workload(w), dv.from_workload(w, pdl=False)]
    try:
        th_dev = torch.tensor(ths, dtype=torch.float64, device="cuda")
        res = []
        for ctx in ctxs:
            out = torch.zeros(5 * 16, dtype=torch.float64, device="cuda")
            for K in (1, 16, 16):
                ctx.cost_dev(K, th_dev, out)
            ctx.check()
            res.append((ctx.terms(ths[3]), out.cpu().numpy(), ctx.cost_batch(ths)[0]))
        assert ctxs[0].num_graphs() == 0 and ctxs[1].num_graphs() >= 2
        for r in res[1:]:
            assert np.array_equal(r[0], res[0][0])
            assert np.array_equal(r[1], res[0][1])
            assert np.array_equal(r[2], res[0][2])
        ref = sim.workload_terms(w, ths[3])
        assert np.max(np.abs(res[0][0] - ref)) <= TOL
    finally:
        for ctx in ctxs:
            ctx.destroy()


def test_cfg3_two_circuits_per_warp_matches_one(dv):
    """plane2_kernel (two circuits in flight per warp, skewed phases) computes every circuit with
    the same operations in the same order as plane_kernel: bitwise identical terms at cfg3; the
    weighted sums differ only in summation grouping (6 vs 10 warp pairs per CTA)."""
    w = configs.cfg3()
    th = w.theta0(7)
    a = dv.from_workload(w, variant=1)
    b = dv.from_workload(w, variant=2)
    try:
        ta, tb = a.terms(th), b.terms(th)
        ca, cb = a.cost(th), b.cost(th)
        ths = np.stack([w.theta0(s) for s in range(16)])
        ba, bb = a.cost_batch(ths)[0], b.cost_batch(ths)[0]
    finally:
        a.destroy()
        b.destroy()
    assert np.array_equal(ta, tb)
    assert abs(ca - cb) <= 1e-13 and np.max(np.abs(ba - bb)) <= 1e-13
    assert np.max(np.abs(ta - sim.workload_terms(w, th))) <= TOL
