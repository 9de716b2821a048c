"""Per-call fixed cost of the Hadamard-test kernel: cfg3 cost calls at K = 1, 2, 4, 8, 16 thetas,
kernel time from the library's own CUDA events (dvqls_last_timings), median of 20 calls each.
A linear fit t(K) = F + K w separates the per-theta work w from the per-call fixed cost F.

    python tools/k_probe.py            (GPU)
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


def main():
    build.build()
    w = configs.cfg3()
    ctx = dvqls.from_workload(w, device=0, timing=True, max_batch=16)
    ths = torch.tensor(np.stack([w.theta0(s) for s in range(16)]), dtype=torch.float64, device="cuda")
    out = torch.empty(16 * 5, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    res = {}
    for K in (1, 2, 4, 8, 16):
        had, pre = [], []
        for i in range(23):
            flush.zero_()
            torch.cuda.synchronize()  # the flush runs on torch's stream, the call on the library's
            ctx.cost_dev(K, ths, out)
            torch.cuda.synchronize()
            t = ctx.last_timings()
            if i >= 3:
                had.append(t["hadamard_ms"])
                pre.append(t["prefix_ms"])
        res[K] = {"hadamard_ms": statistics.median(had), "prefix_ms": statistics.median(pre)}
    Ks = np.array(sorted(res))
    T = np.array([res[k]["hadamard_ms"] for k in Ks])
    wfit, F = np.polyfit(Ks, T, 1)
    print(json.dumps({"per_K": res, "fit": {"per_theta_ms": wfit, "fixed_ms": F}}))
    ctx.destroy()


if __name__ == "__main__":
    main()
