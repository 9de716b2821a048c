"""Multi-rank D-VQLS protocol (Alg. 1 Steps 4a-4c).

* CPU (gloo, world_size 2): each rank takes the contiguous circuit block the
  library assigns (dvqls_shard_range, pure host code), evaluates it with the
  oracle, aggregates (E_loc, Psi_loc), allreduces over gloo; the result must
  equal the single-process cost.  This exercises the sharding + reduction
  logic of the multi-GPU path without a GPU.
* GPU (NCCL): torchrun over the visible GPUs runs tools/multirank_check.py
  through the C ABI (skipped with fewer than 2 GPUs).
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from dvqls_inputs import configs
    from oracle import cost as ocost
    from oracle import sim
    from paper_2604_14435_b200 import dvqls

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w = configs.random_workload(3, 5, 2, seed=11, amplitudes=True)
    th = w.theta0()
    c0, c1 = dvqls.dvqls_shard_range(w.n_circuits, rank, world)
    idx = np.arange(c0, c1)
    vals = sim.workload_terms(w, th, idx=idx, nthreads=1)
    E, Psi = ocost.aggregate(vals, ocost.coeffs_of(w), w.n, w.L, circuits=idx)  # Step 4b
    t = torch.tensor([E.real, E.imag, Psi.real, Psi.imag], dtype=torch.float64)
    dist.all_reduce(t)                                                           # Step 4c
    C = ocost.cost_from(complex(t[0], t[1]), complex(t[2], t[3]), w.n)
    out[rank] = (C, c0, c1)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_reduction_equals_single_process(world):
    from dvqls_inputs import configs
    from oracle import cost as ocost
    from oracle import sim

    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    w = configs.random_workload(3, 5, 2, seed=11, amplitudes=True)
    C1 = ocost.cost(sim.workload_terms(w, w.theta0()), ocost.coeffs_of(w), w.n, w.L)[0]
    blocks = sorted((out[r][1], out[r][2]) for r in range(world))
    assert blocks[0][0] == 0 and blocks[-1][1] == w.n_circuits
    assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
    for r in range(world):
        assert abs(out[r][0] - C1) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("config,mode", [("cfg1", 0), ("cfg2p", 0), ("cfg3", 0), ("n12", 0), ("cfg1", 1), ("cfg3", 1)])
def test_nccl_multigpu(config, mode):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), "--nproc-per-node", str(min(n, 8)),
           os.path.join(ROOT, "tools", "multirank_check.py"), "--config", config, "--mode", str(mode)]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
