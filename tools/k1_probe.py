"""Per-call fixed cost at K = 1 (n = 10, d = 10, uniform b): L = 1 (22 circuits), L = 8 and cfg3
(L = 64, 90,112 circuits).  Timing context: the library's CUDA events around the prefix and the
Hadamard kernel; graph context (the default): CUDA events around one dvqls_cost_dev call.
Median of 50 calls.  `--ncu`: only cfg3 K = 1 calls (for an ncu capture of the Hadamard kernel)."""
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
if "--ncu" in sys.argv:
    w = configs.cfg3()
    ctx = dvqls.from_workload(w, device=0)
    th = torch.tensor(w.theta0(1)[None], dtype=torch.float64, device="cuda")
    out = torch.empty(5, dtype=torch.float64, device="cuda")
    for _ in range(8):
        ctx.cost_dev(1, th, out)
    torch.cuda.synchronize()
    ctx.destroy()
    sys.exit(0)
res = {}
for name, w in (("L1", configs.random_workload(10, 1, 10, seed=11)),
                ("L8", configs.random_workload(10, 8, 10, seed=12)), ("cfg3", configs.cfg3())):
    th = torch.tensor(w.theta0(1)[None], dtype=torch.float64, device="cuda")
    out = torch.empty(5, dtype=torch.float64, device="cuda")
    r = {"circuits": w.n_circuits}
    ctx = dvqls.from_workload(w, device=0, timing=True)
    had, pre = [], []
    for i in range(55):
        ctx.cost_dev(1, th, out)
        torch.cuda.synchronize()
        t = ctx.last_timings()
        if i >= 5:
            had.append(t["hadamard_ms"]); pre.append(t["prefix_ms"])
    ctx.destroy()
    r["hadamard_ms"], r["prefix_ms"] = statistics.median(had), statistics.median(pre)
    st = torch.cuda.Stream()
    ctx = dvqls.from_workload(w, device=0, stream=st)
    calls = []
    for i in range(55):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.cost_dev(1, th, out)
        e1.record(st)
        torch.cuda.synchronize()
        if i >= 5:
            calls.append(e0.elapsed_time(e1))
    ctx.destroy()
    r["graph_call_ms"] = statistics.median(calls)
    res[name] = r
print(json.dumps(res, indent=1))
