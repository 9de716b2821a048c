"""cfg5 at n = 22 and 24 (the largest sizes of the sweep): a few strided circuits through
dvqls_terms_subset against the gate-by-gate oracle (prefix-shared mode), |diff| <= 1e-10."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dvqls_inputs import configs  # noqa: E402
from oracle import sim  # noqa: E402
from paper_2604_14435_b200 import build, dvqls  # noqa: E402

build.build()
for n in (22, 24):
    w = configs.cfg5(n)
    th = w.theta0()
    idx = np.linspace(0, w.n_circuits - 1, 4).astype(np.int64)
    idx[1::2] |= 1
    t0 = time.time()
    ctx = dvqls.from_workload(w, device=0)
    g = ctx.terms_subset(th, idx)
    ctx.destroy()
    t1 = time.time()
    ref = sim.workload_terms(w, th, idx=idx)
    err = float(np.max(np.abs(g - ref)))
    print(f"n={n} circuits={list(idx)} gpu={list(g)} max|err|={err:.3e} gpu {t1 - t0:.1f}s oracle {time.time() - t1:.1f}s",
          flush=True)
    assert err <= 1e-10
