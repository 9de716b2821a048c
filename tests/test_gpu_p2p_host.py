"""GPU: the fused NVLink/peer-memory reduction (a10; "Global Reduction", Alg. 1 Step 4c
P:461-463) with 2, 3 and 8 processes on ONE GPU, bootstrapped through the caller's host allgather
(dvqls_opts.host_allgather over torch.distributed gloo) instead of NCCL, so the kernel-tail
reduction runs on the driver's single-GPU box:

* parity: every rank's terms, cost, batch and device-entry results equal the oracle's (1e-10)
  and each other's bitwise;
* error path: if a peer never publishes, the waiting rank's call returns DVQLS_E_NCCL after
  p2p_timeout_ms (never NaN with DVQLS_OK) and the context refuses further evaluations.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from dvqls_inputs import configs
    from paper_2604_14435_b200 import dvqls

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cb = dvqls.make_host_allgather()
    w = {"n6": lambda: configs.random_workload(6, 3, 2, seed=5),
         "cfg3": configs.cfg3,
         "n13": lambda: configs.random_workload(13, 2, 1, seed=6)}[case if case != "timeout" else "n6"]()
    timeout_ms = 3000 if case == "timeout" else 0
    ctx = dvqls.from_workload(w, device=0, rank=rank, world=world, host_allgather=cb, max_batch=4,
                              p2p_timeout_ms=timeout_ms)
    th = w.theta0()
    try:
        if case == "timeout":
            res = {}
            if rank == 0:
                try:
                    ctx.cost(th)
                    res["first"] = "no error"
                except dvqls.DvqlsError as e:
                    res["first"] = e.code
                try:
                    ctx.cost(th)
                    res["second"] = "no error"
                except dvqls.DvqlsError as e:
                    res["second"] = e.code
            dist.barrier()  # rank 1 never evaluates
            out[rank] = res
        else:
            terms = ctx.terms(th)
            C, E, Psi = ctx.cost(th, with_E_Psi=True)
            ths = np.stack([w.theta0(s) for s in range(3)])
            cbat, _ = ctx.cost_batch(ths)
            o = torch.zeros(15, dtype=torch.float64, device="cuda")
            tdev = torch.tensor(ths, dtype=torch.float64, device="cuda")
            for _ in range(3):  # capture + replays of the graph
                ctx.cost_dev(3, tdev, o)
            ctx.check()
            out[rank] = {"terms": terms, "C": C, "E": E, "Psi": Psi, "batch": cbat, "dev": o.cpu().numpy(),
                         "range": ctx.local_range(), "graphs": ctx.num_graphs()}
    finally:
        ctx.destroy()
        dist.destroy_process_group()


def _run(case, world=2):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_14435_b200 import build
    build.build()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    return {r: out[r] for r in range(world)}


@pytest.mark.parametrize("case,world", [("n6", 2), ("cfg3", 2), ("n13", 2), ("n6", 3), ("n6", 8)])
def test_processes_one_gpu_fused_reduction(case, world):
    """world 2 (each case), 3 (uneven task blocks) and 8 (the box's full rank count: 7 peers mapped
    per rank, 8 epoch slots per theta)"""
    from dvqls_inputs import configs
    from oracle import cost as ocost
    from oracle import sim

    res = _run(case, world)
    w = {"n6": lambda: configs.random_workload(6, 3, 2, seed=5), "cfg3": configs.cfg3,
         "n13": lambda: configs.random_workload(13, 2, 1, seed=6)}[case]()
    th = w.theta0()
    ref = sim.workload_terms(w, th)
    co = ocost.coeffs_of(w)
    Cr, Er, Pr = ocost.cost(ref, co, w.n, w.L)
    assert res[0]["range"][0] == 0 and res[world - 1]["range"][1] == w.n_circuits
    for r in range(world - 1):
        assert res[r]["range"][1] == res[r + 1]["range"][0]
    for r in range(world):
        assert np.max(np.abs(res[r]["terms"] - ref)) <= 1e-10
        assert abs(res[r]["C"] - Cr) <= 1e-10 and abs(res[r]["E"] - Er) <= 1e-10 * max(1, abs(Er))
        for k in range(3):
            Ck = ocost.cost(sim.workload_terms(w, w.theta0(k)), co, w.n, w.L)[0]
            assert abs(res[r]["batch"][k] - Ck) <= 1e-10
            assert res[r]["dev"][5 * k] == res[r]["batch"][k]
        assert res[r]["graphs"] >= 1
    for r in range(1, world):
        assert res[0]["C"] == res[r]["C"] and np.array_equal(res[0]["dev"], res[r]["dev"])


def test_peer_timeout_is_an_error_not_nan():
    res = _run("timeout")
    from paper_2604_14435_b200 import dvqls
    assert res[0]["first"] == dvqls.DVQLS_E_NCCL, res
    assert res[0]["second"] == dvqls.DVQLS_E_NCCL, res
