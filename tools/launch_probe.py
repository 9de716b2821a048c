"""A/B of the launch variants of the cost path: plain launches, programmatic dependent launch of
the Hadamard kernel behind the prefix (opts.pdl), one CUDA graph per call (opts.graphs), both.

Per-call device time of back-to-back dvqls_cost_dev calls (timing events off), torch CUDA events
on the library's stream, median of 7 runs of 50 calls.
Workloads: cfg3 (n = 10, 90,112 circuits) at K = 1 and 16, and n = 10, L = 1 (22 circuits) where
the per-call fixed cost dominates.  The costs of all arms must agree bit for bit.
"""
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
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
res = {}
for name, w in (("cfg3", configs.cfg3()), ("n10_L1", configs.random_workload(10, 1, 10, seed=11))):
    ths = torch.tensor(np.stack([w.theta0(s) for s in range(16)]), dtype=torch.float64, device="cuda")
    outs = {}
    arms = {"plain": dict(graphs=False, pdl=False), "pdl": dict(graphs=False, pdl=True),
            "graph": dict(graphs=True, pdl=False), "graph_pdl": dict(graphs=True, pdl=True)}
    for arm, kw in arms.items():
        ctx = dvqls.from_workload(w, device=0, timing=False, max_batch=16, stream=stream, **kw)
        out = torch.empty(80, dtype=torch.float64, device="cuda")
        for K in (1, 16):
            reps = 50 if name != "cfg3" or K == 1 else 10
            with torch.cuda.stream(stream):
                for _ in range(5):
                    ctx.cost_dev(K, ths, out)
                ms = []
                for _ in range(7):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    for _ in range(reps):
                        ctx.cost_dev(K, ths, out)
                    b.record(stream)
                    b.synchronize()
                    ms.append(a.elapsed_time(b) / reps)
            torch.cuda.synchronize()
            res[f"{name}_K{K}_{arm}_us"] = 1e3 * statistics.median(ms)
            outs[(arm, K)] = out[:5 * K].cpu().numpy().copy()
        ctx.destroy()
    for K in (1, 16):
        res[f"{name}_K{K}_same_cost"] = all(np.array_equal(outs[("plain", K)], outs[(a, K)]) for a in arms)
print(json.dumps(res, indent=1))
