"""GPU parity of NEXT-3 (global cost C_G, Eq. 1; global.cuh): the 2L overlap
Hadamard-test values beta_l = <b|A_l|x> and C_G against the gate-by-gate oracle (1e-10
absolute, the circuit path's bar), and the GPU-side check C_L <= C_G <= n C_L."""

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


def _check(dv, w, mode=0, seeds=(0, 1)):
    ctx = dv.from_workload(w, mode=mode)
    try:
        for seed in seeds:
            th = w.theta0(seed)
            CL, CG, E, Psi, beta = ctx.global_cost(th, with_beta=True)
            ov = sim.workload_overlaps(w, th)
            ref_beta = ov[0::2] + 1j * ov[1::2]
            assert np.max(np.abs(beta - ref_beta)) <= TOL
            T = sim.workload_terms(w, th)
            CLr, Er, Pr = ocost.cost(T, ocost.coeffs_of(w), w.n, w.L)
            CGr = ocost.global_cost(ov, ocost.coeffs_of(w), Pr)
            assert abs(CL - CLr) <= TOL and abs(CG - CGr) <= TOL
            assert CL <= CG + 1e-12 and CG <= w.n * CL + 1e-12
    finally:
        ctx.destroy()


@pytest.mark.parametrize("mk", [configs.cfg1, configs.cfg2_velocity, configs.cfg2_pressure])
def test_small_configs(dv, mk):
    _check(dv, mk())


@pytest.mark.parametrize("n,amp", [(1, False), (3, True), (6, False), (9, True), (10, False), (11, True),
                                   (12, False)])
def test_random_non_hermitian(dv, n, amp):
    _check(dv, configs.random_workload(n, 3, 2, seed=500 + n, amplitudes=amp), seeds=(0,))


def test_cfg3(dv):
    _check(dv, configs.cfg3(), seeds=(0,))


def test_pauli_mode(dv):
    _check(dv, configs.cfg1(), mode=dv.DVQLS_MODE_PAULI)


def test_batched_device_entry(dv):
    import torch
    w = configs.cfg1()
    K = 4
    thetas = np.stack([w.theta0(s) for s in range(K)])
    ctx = dv.from_workload(w, max_batch=K)
    try:
        th = torch.tensor(thetas, dtype=torch.float64, device="cuda")
        out6 = torch.empty(6 * K, dtype=torch.float64, device="cuda")
        beta = torch.empty(2 * w.L * K, dtype=torch.float64, device="cuda")
        ctx.costs_dev(K, th, out6, beta)
        torch.cuda.synchronize()
        o = out6.view(K, 6).cpu().numpy()
        b = beta.view(K, w.L, 2).cpu().numpy()
    finally:
        ctx.destroy()
    for k in range(K):
        ov = sim.workload_overlaps(w, thetas[k])
        assert np.max(np.abs(b[k].reshape(-1) - ov)) <= TOL
        T = sim.workload_terms(w, thetas[k])
        CLr, Er, Pr = ocost.cost(T, ocost.coeffs_of(w), w.n, w.L)
        assert abs(o[k, 0] - CLr) <= TOL and abs(o[k, 5] - ocost.global_cost(ov, ocost.coeffs_of(w), Pr)) <= TOL
