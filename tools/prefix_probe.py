"""Run the cfg3 hot path with K thetas at once (one prefix CTA per theta) for profiling."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from dvqls_inputs import configs
from paper_2604_14435_b200 import dvqls
K = int(sys.argv[1]) if len(sys.argv) > 1 else 148
w = configs.cfg3()
ctx = dvqls.from_workload(w, max_batch=K)
th = torch.tensor(np.stack([w.theta0(s) for s in range(K)]), dtype=torch.float64, device="cuda")
out = torch.empty(5 * K, dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.cost_dev(K, th, out)
torch.cuda.synchronize()
print("ok", out[:5].tolist())
