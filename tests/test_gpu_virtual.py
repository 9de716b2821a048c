"""GPU: the multi-rank sharding and the global reduction on ONE GPU (virtual ranks).

dvqls_opts.virtual_rank / virtual_world evaluate the contiguous circuit block [rC/W, (r+1)C/W)
that rank r of a W-way split owns ("strided workload allocation": contiguous
blocks) and return that block's partial (E, Psi) (Alg. 1 Step 4b).  Summing the W
partials in rank order is Step 4c's Allreduce; the result must equal the oracle's
cost.  This runs the rank-offset code paths (c0 != 0 decode, cost-weighted ranges starting mid
period, the per-block grid) on the driver's 1-GPU box.
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


WORKLOADS = {
    "cfg1": configs.cfg1,
    "cfg2p": configs.cfg2_pressure,                                     # Householder U_b, n = 4
    "cfg3": configs.cfg3,                                               # headline plane kernel
    "n12": lambda: configs.random_workload(12, 2, 1, seed=81),          # on-chip kernel
    "n14": lambda: configs.random_workload(14, 2, 1, seed=82, entangler=1),  # streaming kernel
    "n13hh": lambda: configs.random_workload(13, 2, 1, seed=83, amplitudes=True),
}


@pytest.mark.parametrize("name,W", [("cfg1", 2), ("cfg1", 3), ("cfg2p", 3), ("cfg3", 2), ("cfg3", 3),
                                    ("cfg3", 8), ("n12", 3), ("n14", 2), ("n13hh", 3)])
def test_virtual_ranks_sum_to_the_oracle_cost(dv, name, W):
    w = WORKLOADS[name]()
    ths = np.stack([w.theta0(s) for s in (0, 1)])
    co = ocost.coeffs_of(w)
    refs = [sim.workload_terms(w, th) for th in ths]
    acc = np.zeros((2, 4))
    terms = np.full(w.n_circuits, np.nan)
    prev = 0
    for r in range(W):
        ctx = dv.from_workload(w, virtual_rank=r, virtual_world=W, max_batch=2)
        try:
            c0, c1 = ctx.local_range()
            assert (c0, c1) == dv.dvqls_shard_range(w.n_circuits, r, W) and c0 == prev
            prev = c1
            cb, ep = ctx.cost_batch(ths)
            t = ctx.terms(ths[0])
        finally:
            ctx.destroy()
        assert np.all(np.isnan(cb))  # a block has no cost of its own
        assert np.all(np.isnan(t[:c0])) and np.all(np.isnan(t[c1:]))
        terms[c0:c1] = t[c0:c1]
        for k in range(2):  # this block's (E, Psi) = the oracle's Step 4b over the block
            E, Psi = ocost.aggregate(refs[k][c0:c1], co, w.n, w.L, circuits=range(c0, c1))
            assert np.max(np.abs(ep[k] - [E.real, E.imag, Psi.real, Psi.imag])) <= TOL
        acc += ep  # Step 4c, fixed rank order
    assert prev == w.n_circuits
    assert np.max(np.abs(terms - refs[0])) <= TOL
    for k in range(2):
        C = ocost.cost_from(complex(acc[k, 0], acc[k, 1]), complex(acc[k, 2], acc[k, 3]), w.n)
        assert abs(C - ocost.cost(refs[k], co, w.n, w.L)[0]) <= TOL


def test_virtual_rank_rejects_foreign_subset_and_global_calls(dv):
    w = configs.random_workload(14, 2, 1, seed=84)
    ctx = dv.from_workload(w, virtual_rank=1, virtual_world=2)
    try:
        c0, c1 = ctx.local_range()
        th = w.theta0()
        idx = np.array([c0, c0 + 1, c1 - 1])
        g = ctx.terms_subset(th, idx)
        assert np.max(np.abs(g - sim.workload_terms(w, th, idx=idx))) <= TOL
        with pytest.raises(dv.DvqlsError):
            ctx.terms_subset(th, np.array([0]))
        with pytest.raises(dv.DvqlsError):
            ctx.global_cost(th)
        with pytest.raises(dv.DvqlsError):
            ctx.cost_grad(th)
    finally:
        ctx.destroy()
