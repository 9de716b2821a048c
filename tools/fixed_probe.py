"""Fixed cost of one Hadamard-kernel launch: n = 10, d = 10 with L = 1 (22 circuits) and L = 2
(88 circuits), K = 1 and 16, kernel time from the library's CUDA events (median of 50 calls)."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dvqls_inputs import configs  # noqa: E402
from paper_2604_14435_b200 import build, dvqls  # noqa: E402

build.build()
res = {}
for L in (1, 2):
    w = configs.random_workload(10, L, 10, seed=11)
    ctx = dvqls.from_workload(w, device=0, timing=True, max_batch=16)
    ths = torch.tensor(np.stack([w.theta0(s) for s in range(16)]), dtype=torch.float64, device="cuda")
    out = torch.empty(80, dtype=torch.float64, device="cuda")
    for K in (1, 16):
        had, pre, call = [], [], []
        for i in range(55):
            ctx.cost_dev(K, ths, out)
            torch.cuda.synchronize()
            t = ctx.last_timings()
            if i >= 5:
                had.append(t["hadamard_ms"]); pre.append(t["prefix_ms"]); call.append(t["call_ms"])
        res[f"L{L}_K{K}"] = {"circuits": w.n_circuits * K, "hadamard_ms": statistics.median(had),
                             "prefix_ms": statistics.median(pre), "call_ms": statistics.median(call)}
    ctx.destroy()
print(json.dumps(res))
