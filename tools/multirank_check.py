"""Multi-rank check of the NCCL path (run under torchrun, one process per GPU).

    torchrun --standalone --nproc-per-node N tools/multirank_check.py [--config cfg1|cfg3]

Every rank builds a context with its (rank, world) and a shared ncclUniqueId,
evaluates dvqls_terms (allgathered) and dvqls_cost / dvqls_cost_batch (one
NCCL allreduce of (E, Psi) per theta).  Rank 0 compares against the oracle
(test infrastructure) with the 1e-10 tolerance and exits non-zero on mismatch.
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--mode", type=int, default=0, help="0 = circuits, 1 = NEXT-2 Pauli fast path")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from dvqls_inputs import configs
    from paper_2604_14435_b200 import dvqls

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [dvqls.dvqls_nccl_unique_id() if rank == 0 else None, dvqls.dvqls_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    w = {"cfg1": configs.cfg1, "cfg3": configs.cfg3, "cfg2p": configs.cfg2_pressure,
         "n12": lambda: configs.random_workload(12, 2, 2, seed=77)}[args.config]()
    ctx = dvqls.from_workload(w, device=local, rank=rank, world=world, nccl_id=obj[0], mode=args.mode)
    th = w.theta0()
    terms = ctx.terms(th)
    C, E, Psi = ctx.cost(th, with_E_Psi=True)
    ths = np.stack([w.theta0(s) for s in range(3)])
    cb, _ = ctx.cost_batch(ths)
    CLg, CG, _, _ = ctx.global_cost(th)
    c0, c1 = ctx.local_range()
    # a second context of the same ranks (its own communicator, NCCL reduction path) alongside
    ctx2 = dvqls.from_workload(w, device=local, rank=rank, world=world, nccl_id=obj[1], mode=args.mode,
                               allreduce=dvqls.DVQLS_ALLREDUCE_NCCL)
    C2 = ctx2.cost(th)
    ctx2.destroy()
    ok = True
    # every rank must hold identical global results
    t = torch.tensor([C, cb[0], cb[1], cb[2], float(terms.sum()), CG, C2], dtype=torch.float64, device="cuda")
    lst = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(lst, t)
    if rank == 0:
        from oracle import cost as ocost
        from oracle import sim
        ref = sim.workload_terms(w, th)
        err = float(np.max(np.abs(terms - ref)))
        Cr, Er, Pr = ocost.cost(ref, ocost.coeffs_of(w), w.n, w.L)
        refb = [ocost.cost(sim.workload_terms(w, ths[k]), ocost.coeffs_of(w), w.n, w.L)[0] for k in range(3)]
        same = all(torch.equal(lst[0], x) for x in lst)
        CGr = ocost.global_cost(sim.workload_overlaps(w, th), ocost.coeffs_of(w), Pr)
        ok = (err <= 1e-10 and abs(C - Cr) <= 1e-10 and abs(C2 - Cr) <= 1e-10 and max(abs(cb[k] - refb[k]) for k in range(3)) <= 1e-10
              and same and abs(CG - CGr) <= 1e-10 and abs(CLg - Cr) <= 1e-10)
        print(f"world={world} mode={args.mode} {w.name}: max|term err|={err:.2e} C={C:.12f} oracle={Cr:.12f} "
              f"C_G={CG:.12f} oracle={CGr:.12f} "
              f"batch_err={max(abs(cb[k] - refb[k]) for k in range(3)):.2e} ranks_agree={same} "
              f"rank0 block=[{c0},{c1}) -> {'OK' if ok else 'FAIL'}", flush=True)
    flag = torch.tensor([1.0 if ok else 0.0], device="cuda")
    dist.broadcast(flag, src=0)
    ctx.destroy()
    dist.destroy_process_group()
    return 0 if flag.item() == 1.0 else 1


if __name__ == "__main__":
    sys.exit(main())
