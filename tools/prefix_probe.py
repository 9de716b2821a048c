"""Prefix kernels of cfg3 (n = 10, d = 10) for profiling / timing: the one-CTA prefix (default) and
the cluster prefix (opts.prefix = 1), K thetas per call, timing events on (per-kernel times).

    python tools/prefix_probe.py [K]
"""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from dvqls_inputs import configs  # noqa: E402
from paper_2604_14435_b200 import dvqls  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = configs.cfg3()
th = torch.tensor(np.stack([w.theta0(s) for s in range(K)]), dtype=torch.float64, device="cuda")
out = torch.empty(5 * K, dtype=torch.float64, device="cuda")
res = {}
for name, pf in (("cluster", 1), ("one_cta", 0)):
    ctx = dvqls.from_workload(w, max_batch=K, timing=True, prefix=pf)
    ms = []
    for i in range(30):
        ctx.cost_dev(K, th, out)
        if i >= 5:
            ms.append(ctx.last_timings()["prefix_ms"])
    torch.cuda.synchronize()
    res[f"{name}_prefix_us_median"] = 1e3 * statistics.median(ms)
    res[f"{name}_prefix_us_min"] = 1e3 * min(ms)
    ctx.destroy()
print(json.dumps(res, indent=1))
