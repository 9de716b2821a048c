"""cfg5 at n = 24 (the largest size; 5 streaming passes, x from DRAM): one warm-up and one timed
parameter-shift pair (K = 2) through dvqls_cost_dev, Hadamard-kernel time from the library's CUDA
events; DRAM model 160N per numerator circuit + 32N per denominator (bench.hbm_bytes_per_eval)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from dvqls_inputs import configs  # noqa: E402
from paper_2604_14435_b200 import build, dvqls  # noqa: E402

build.build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
w = configs.cfg5(n)
ctx = dvqls.from_workload(w, device=0, timing=True, max_batch=2)
th = w.theta0()
pair = np.stack([th, th])
pair[0, 0] += np.pi / 2
pair[1, 0] -= np.pi / 2
ths = torch.tensor(pair, dtype=torch.float64, device="cuda")
out = torch.empty(10, dtype=torch.float64, device="cuda")
ctx.cost_dev(2, ths, out)
torch.cuda.synchronize()
ctx.cost_dev(2, ths, out)
torch.cuda.synchronize()
t = ctx.last_timings()
ctx.destroy()
had_s = t["hadamard_ms"] * 1e-3
byts = bench.hbm_bytes_per_eval(w) * 2
peak = float(bench.load_peaks()[0]["hbm_gbs"])
print(json.dumps({"n": n, "circuits_per_s": 2 * w.n_circuits / (t["call_ms"] * 1e-3), "timings_ms": t,
                  "dram_model_bytes": byts, "GBps": byts / had_s / 1e9, "hbm_frac": byts / had_s / 1e9 / peak,
                  "costs": out.view(2, 5)[:, 0].tolist()}))
