#!/usr/bin/env python3
"""Benchmark of the D-VQLS hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3|cfg4|cfg1]
                    [--batch KT] [--impl dvqls|reference] [--no-cpu-baseline]

One *step* = one pass of the whole hot path (prefix
V(theta)|0>, all 2(n+1)L^2 Hadamard-test circuits, weighted reduction,
cross-rank allreduce, cost) for KT thetas.  Default workload: BASELINE config 3
(n=10, L=64, d=10; 90,112 circuits per cost evaluation).  With N ranks each GPU
evaluates a contiguous 1/N block of the circuits and one NCCL allreduce of
4 doubles per theta combines them (strong scaling over a fixed workload).

`value` = whole-job circuits/s with theta resident in HBM (device entry point
dvqls_cost_dev), timed with CUDA events on the library's stream, L2 flushed
(256 MiB write) before every step, max over ranks.  `e2e` = the same metric
through the host-buffer C-ABI call dvqls_cost (theta H2D + result D2H inside).
The oracle (oracle/, test infrastructure) is only executed for `cpu_baseline`
(rank 0, N = 1) and for `--impl reference`.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from dvqls_inputs import configs  # noqa: E402

CONFIGS = {"cfg1": configs.cfg1, "cfg3": configs.cfg3, "cfg4": configs.cfg4, "cfg5": configs.cfg5}
METRIC = "Hadamard-test circuits/sec & cost evals/sec, 10q 90,112 circuits, 1/2/4/8 B200"
L2_FLUSH_BYTES = 256 << 20


def fp64_ops_per_eval(w, circuits=None):
    """Algorithmic FP64-pipe ops (DADD and DFMA count 1 each), SURVEY §8(d):
    numerator circuit (4n+2)N (two n-stage FWHTs at 2N DADD/stage + 2N DFMA
    readout), denominator 2N; uniform b."""
    N = 1 << w.n
    n1 = w.n + 1
    c = np.arange(w.n_circuits) if circuits is None else circuits
    s = (c // 2) % n1
    num = int(np.count_nonzero(s))
    den = c.size - num
    return num * (4 * w.n + 2) * N + den * 2 * N


def hbm_bytes_per_eval(w, circuits=None):
    """Streaming-path algorithmic DRAM bytes (n > 12): the branch of a numerator circuit makes 3
    passes through its per-CTA scratch (P0 writes 16N, P1 reads + writes 32N, P2 reads 16N: 64N)
    while x (K x <= 32 MB for n <= 21) stays L2-resident; from n = 22 x (K x 64-256 MB) is read from
    DRAM twice (32N, also by the denominators), and n >= 23 takes 5 passes (128N).
    SURVEY §8(d) counts x as HBM traffic at every n (96N); that figure is reported beside it."""
    N = 1 << w.n
    c = np.arange(w.n_circuits) if circuits is None else circuits
    s = (c // 2) % (w.n + 1)
    num = int(np.count_nonzero(s))
    den = c.size - num
    if w.n <= 21:
        return num * 64 * N
    passes = 64 if w.n <= 22 else 128
    return num * (passes + 32) * N + den * 32 * N


def smem_bytes_per_eval(w, circuits=None):
    """On-chip model bytes: numerator 96N, denominator 32N."""
    N = 1 << w.n
    c = np.arange(w.n_circuits) if circuits is None else circuits
    s = (c // 2) % (w.n + 1)
    num = int(np.count_nonzero(s))
    return num * 96 * N + (c.size - num) * 32 * N


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.lines = []

    def __enter__(self):
        self.recording = False
        self.raw = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", ",".join(map(str, self.gpus)), "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.raw and time.time() - t0 < 10:  # wait until sampling is live
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        return self

    def start(self):
        self.recording = True

    def stop(self):
        self.recording = False

    def _read(self):
        for line in self.proc.stdout:
            self.raw.append(line.strip())
            if self.recording:
                self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0,
                    "raw": self.raw[:3]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "hadamard_dram_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


def streaming_roofline(w, local_c, KT, had_ms, peaks, peak_src, grid=None):
    b = hbm_bytes_per_eval(w, local_c) * KT
    b96 = smem_bytes_per_eval(w, local_c) * KT
    ach = b / (had_ms * 1e-3)
    peak = float(peaks["hbm_gbs"]) * 1e9
    plane = w.bkind == 0 and os.environ.get("DVQLS_PLANE", "1") != "0" and os.environ.get("DVQLS_TEAM", "0") != "1"
    staged = os.environ.get("DVQLS_STAGE", "") != "0" and (w.n >= 16 or os.environ.get("DVQLS_STAGE") == "1")
    kern = (f"stream_plane_kernel<12, {'TMA-staged' if staged else 'direct'}>" if plane
            else "stream_hadamard_kernel<12>")
    out = {"bound": "hbm", "kernel": kern, "achieved": ach / 1e9, "peak": peak / 1e9,
           "unit": "GB/s", "frac": ach / peak, "traffic": None,
           "model96_GBps": b96 / (had_ms * 1e-3) / 1e9,
           "note": (f"algorithmic DRAM bytes per launch = {b:.4g} (64N per numerator circuit: 3 passes "
                    f"through the per-CTA scratch, x L2-resident; n >= 23: 160N + 32N per denominator) / mean "
                    f"CUDA-event kernel time; peak = hbm_gbs of {peak_src} MEASURED_PEAKS.json. model96_GBps "
                    f"= the SURVEY §8(d) 96N model (x reads counted as HBM)")}
    if grid is not None:
        scratch = grid * (1 << w.n) * (8 if plane else 16)
        out["scratch_bytes"] = scratch
        if scratch <= 100 << 20:
            out["note"] += "; the per-CTA scratch fits in L2 at this n, so L2 bandwidth, not HBM, bounds it"
    return out


def onchip_roofline(w, local_c, KT, had_ms, sms, fmax, peak_src):
    """n = 11, 12 (one tile on chip): FP64-pipe ops vs 64 lanes/clk/SM; on-chip bytes = the SURVEY
    §8(d) model of the register path (96N per numerator circuit: x read twice + one exchange per
    FWHT; 32N per denominator), which the default 2-exchange kernel (onchip_plane.cuh) implements
    (its x reads come from L2 through the L1 pipe).  With DVQLS_ONCHIP=0 the 4-exchange tile
    kernel runs against the same model."""
    ops = fp64_ops_per_eval(w, local_c) * KT
    sbytes = smem_bytes_per_eval(w, local_c) * KT
    fp64_peak = 64 * sms * fmax
    smem_peak = 128 * sms * fmax
    t = had_ms * 1e-3
    onchip = w.bkind == 0 and os.environ.get("DVQLS_ONCHIP", "1") != "0" and os.environ.get("DVQLS_PLANE", "1") != "0"
    kern = (f"onchip_plane_kernel<{w.n}>" if onchip else
            f"stream_{'plane' if w.bkind == 0 and os.environ.get('DVQLS_PLANE', '1') != '0' else 'hadamard'}_kernel<{11 if w.n == 11 else 12}>")
    return {"bound": "alu", "kernel": kern,
            "achieved": ops / t / 1e12, "peak": fp64_peak / 1e12, "unit": "Top/s", "frac": ops / t / fp64_peak,
            "traffic": None,
            "smem": {"achieved": sbytes / t / 1e9, "peak": smem_peak / 1e9, "unit": "GB/s",
                     "frac": sbytes / t / smem_peak,
                     "note": "on-chip model bytes: 96N per numerator circuit, 32N per denominator"},
            "model_frac": max(ops / fp64_peak, sbytes / smem_peak) / t,
            "note": (f"FP64-pipe lane-ops per launch = {ops:.4g} / mean CUDA-event kernel time; peak = 64 "
                     f"lanes/clk/SM x {sms} SMs x sm_max_mhz ({peak_src} MEASURED_PEAKS.json)")}


# ----------------------------------------------------------------------------------------------
def cpu_baseline(w, theta, budget_s=12.0):
    """Oracle (as it stands) on all host cores, bounded strided samples of the workload."""
    from oracle import sim
    cores = sim.hardware_threads()
    out = {"kind": "oracle", "cores": cores, "unit": "circuits/s"}
    res = {}
    for mode, name in ((0, "faithful"), (1, "prefix_shared")):
        n_probe = max(cores, 8)
        idx = np.linspace(0, w.n_circuits - 1, n_probe).astype(np.int64)
        t0 = time.perf_counter()
        sim.workload_terms(w, theta, mode=mode, idx=idx, nthreads=cores)
        dt = time.perf_counter() - t0
        per = dt / n_probe
        m = int(min(w.n_circuits, max(n_probe, budget_s / 2 / max(per, 1e-9))))
        idx = np.linspace(0, w.n_circuits - 1, m).astype(np.int64)
        t0 = time.perf_counter()
        sim.workload_terms(w, theta, mode=mode, idx=idx, nthreads=cores)
        dt = time.perf_counter() - t0
        res[name] = (m / dt, m, dt)
    out["value"] = res["faithful"][0]
    out["prefix_shared_value"] = res["prefix_shared"][0]
    out["sample"] = (f"{res['faithful'][1]} (faithful, {res['faithful'][2]:.1f} s) and {res['prefix_shared'][1]} "
                     f"(prefix-shared, {res['prefix_shared'][2]:.1f} s) evenly strided circuits of {w.name}, "
                     f"gate-by-gate C++ oracle, std::thread over {cores} host threads")
    return out


def run_reference(args, w):
    """--impl reference: the oracle as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import sim
    cores = sim.hardware_threads()
    theta = w.theta0()
    # size one step to ~3 s of faithful-mode work on all cores, less when many steps are asked for,
    # so the whole --steps K run stays within ~2 minutes
    step_s = min(3.0, 120.0 / max(args.steps, 1))
    n_probe = max(cores, 8)
    idx = np.linspace(0, w.n_circuits - 1, n_probe).astype(np.int64)
    t0 = time.perf_counter()
    sim.workload_terms(w, theta, mode=0, idx=idx, nthreads=cores)
    per = (time.perf_counter() - t0) / n_probe
    m = int(min(w.n_circuits, max(n_probe, step_s / max(per, 1e-9))))
    idx = np.linspace(0, w.n_circuits - 1, m).astype(np.int64)
    for _ in range(args.warmup):
        sim.workload_terms(w, theta, mode=0, idx=idx[: max(1, m // 10)], nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sim.workload_terms(w, theta, mode=0, idx=idx, nthreads=cores)
    dt = time.perf_counter() - t0
    value = m * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "circuits/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n_qubits": w.n, "L": w.L, "layers": w.layers,
                   "circuits_per_eval": w.n_circuits, "sample_circuits_per_step": m},
        "cpu_baseline": {"value": value, "unit": "circuits/s", "cores": cores, "kind": "oracle",
                         "sample": f"{m} evenly strided circuits of {w.name} per step, faithful mode "
                                   f"(V(theta) re-simulated per circuit, the paper's per-circuit model)"},
        "e2e": {"value": value, "unit": "circuits/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=16,
                    help="thetas per step (dvqls_cost_dev K): one batch of FD-gradient points, the way the "
                         "config-2 L-BFGS-B loop calls the path; K=1 is measured and reported beside it")
    ap.add_argument("--n", type=int, default=16, help="qubits for --config cfg5 (12..24)")
    ap.add_argument("--impl", default="dvqls", choices=["dvqls", "reference"])
    ap.add_argument("--slice", type=int, default=0,
                    help="weak-scaling reference (1 GPU only): evaluate rank 0's block of a SLICE-way split")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next2", action="store_true", help="skip the NEXT-2 fast-path side measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = CONFIGS[args.config](args.n) if args.config == "cfg5" else CONFIGS[args.config]()

    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as dist
    from paper_2604_14435_b200 import build as pbuild
    from paper_2604_14435_b200 import dvqls

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0 and not os.path.exists(dvqls.LIB_PATH):
        pbuild.build()
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [dvqls.dvqls_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    else:
        nccl_id = None

    stream = torch.cuda.Stream(device=dev)
    KT = args.batch
    chars, co = w.arrays()
    # device memory comes from torch: the library carves its tables from this workspace
    if args.slice > 1:
        if world > 1:
            raise SystemExit("--slice is the 1-GPU weak-scaling reference")
        os.environ["DVQLS_SLICE"] = f"0/{args.slice}"
    ws_bytes = dvqls.workspace_size(w.n, w.layers, w.L, device=local, rank=rank, world=world,
                                    max_batch=max(KT, 1))
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ctx = dvqls.Context(w.n, w.layers, chars, co, w.bkind, w.b, device=local, rank=rank, world=world,
                        nccl_id=nccl_id, entangler=w.entangler, stream=stream, timing=True,
                        max_batch=max(KT, 1), workspace=workspace)
    c0, c1 = ctx.local_range()
    thetas = np.stack([w.theta0(s) for s in range(KT)])
    th_dev = torch.tensor(thetas, dtype=torch.float64, device=dev)
    out_dev = torch.empty(5 * KT, dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region ----------------------------------------------------
    sampler = ClockSampler(list(range(world))) if rank == 0 else None
    if sampler:
        sampler.__enter__()
    with torch.cuda.stream(stream):
        # W warm-up steps, continued (in chunks of 8, the same number on every rank: every
        # call contains a cross-rank reduction) until >= 0.5 s of load so the SM clock has ramped
        t_w = time.time()
        i = 0
        while True:
            for _ in range(8):
                flush.zero_()
                ctx.cost_dev(KT, th_dev, out_dev)
                i += 1
            torch.cuda.synchronize()
            more = 1.0 if (i < args.warmup or time.time() - t_w < 0.5) else 0.0
            if world > 1:
                t = torch.tensor([more], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                more = float(t.item())
            if more == 0.0:
                break
        barrier()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        kt = []
        barrier()
        if sampler:
            sampler.start()
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            ctx.cost_dev(KT, th_dev, out_dev)
            ends[i].record(stream)
            kt.append(ctx.last_timings())  # events of the library on the same stream
        barrier()
        if sampler:
            sampler.stop()
    if sampler:
        sampler.__exit__()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    dev_ms = max_over_ranks(dev_ms)

    # ---- the same timed loop with a single theta per step (K = 1) -------------------------------
    k1_steps = max(3, args.steps // 2)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            ctx.cost_dev(1, th_dev, out_dev)
        barrier()
        s1 = [torch.cuda.Event(enable_timing=True) for _ in range(k1_steps)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(k1_steps)]
        k1t = []
        for i in range(k1_steps):
            flush.zero_()
            s1[i].record(stream)
            ctx.cost_dev(1, th_dev, out_dev)
            e1[i].record(stream)
            k1t.append(ctx.last_timings())
        barrier()
    k1_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(s1, e1)))
    res1 = out_dev[:5].cpu().numpy()
    res = out_dev.view(KT, 5).cpu().numpy()
    if not np.all(np.isfinite(res[:, 0])):
        print("error: non-finite cost", res, file=sys.stderr)
        return 1

    # ---- end-to-end through the host-buffer C ABI ---------------------------------------------
    e2e_s = 0.0
    for _ in range(2):
        ctx.cost_batch(thetas) if KT > 1 else ctx.cost(thetas[0])
    barrier()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if KT > 1:
            ctx.cost_batch(thetas)
        else:
            ctx.cost(thetas[0])
        e2e_s += time.perf_counter() - t0
    barrier()
    e2e_s = max_over_ranks(e2e_s)

    # ---- NEXT-3 global cost: C_L and C_G of the same call (dvqls_costs_dev) ----------------------
    next3 = None
    if not args.no_next2:
        out6 = torch.empty(6 * KT, dtype=torch.float64, device=dev)
        g_steps = max(3, args.steps // 4)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                flush.zero_()
                ctx.costs_dev(KT, th_dev, out6)
            barrier()
            gs = [torch.cuda.Event(enable_timing=True) for _ in range(g_steps)]
            ge = [torch.cuda.Event(enable_timing=True) for _ in range(g_steps)]
            for i in range(g_steps):
                flush.zero_()
                gs[i].record(stream)
                ctx.costs_dev(KT, th_dev, out6)
                ge[i].record(stream)
            barrier()
        g_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(gs, ge)))
        o6 = out6.view(KT, 6).cpu().numpy()
        next3 = {"evals_per_s": KT * g_steps / (g_ms * 1e-3), "ms_per_step": g_ms / g_steps,
                 "overhead_vs_local_only": (g_ms / g_steps) / (dev_ms / args.steps) - 1.0,
                 "C_G_theta0": float(o6[0, 5]), "C_L_theta0": float(o6[0, 0]),
                 "sandwich_ok": bool(np.all((o6[:, 0] <= o6[:, 5] + 1e-12) & (o6[:, 5] <= w.n * o6[:, 0] + 1e-12))),
                 "note": "NEXT-3: local cost path + 2L overlap Hadamard tests -> C_G (Eq. 1) in the same call"}

    # ---- NEXT-4 GPU Pauli decomposition + pruning of a dense A (rank 0, side measurement) -------
    next4 = None
    if rank == 0 and not args.no_next2:
        from dvqls_inputs import problems
        nd = 12
        A, _ = problems.tridiag_toeplitz(nd, 2.0, -1.0, -1.0)
        best = None
        for _ in range(3):
            terms, nrm, ms = dvqls.decompose(A, 0.01, device=local, timing=True)
            best = ms if best is None else min(best, ms)
        byts = 16 * 4 ** nd      # algorithmic: A read once (any decomposition must)
        moved = 48 * 4 ** nd     # this design: A read, XOR-diagonal rows B written and read once
        pk = float(load_peaks()[0]["hbm_gbs"])
        next4 = {"n": nd, "terms": len(terms), "ms": best, "GBps": byts / (best * 1e-3) / 1e9,
                 "hbm_frac": byts / (best * 1e-3) / 1e9 / pk,
                 "moved_GBps": moved / (best * 1e-3) / 1e9, "moved_frac": moved / (best * 1e-3) / 1e9 / pk,
                 "note": ("NEXT-4: 4^n coefficients by per-x-mask FWHT in one candidate pass (Parseval bound; exact "
                          "norm filter in the sort) + sort on the GPU; GBps = algorithmic bytes 16*4^n (A read once) "
                          "over the device time (best of 3); moved_GBps = the 48*4^n bytes this design moves")}
        del A

    # ---- NEXT-2 algebraic fast path (flagged; reported separately, never the headline) ----------
    next2 = None
    if w.bkind == 0 and not args.no_next2:
        pctx = dvqls.Context(w.n, w.layers, chars, co, w.bkind, w.b, device=local, rank=rank, world=world,
                             nccl_id=nccl_id, entangler=w.entangler, stream=stream, timing=False,
                             max_batch=max(KT, 1), mode=dvqls.DVQLS_MODE_PAULI)
        p_steps = max(3, args.steps // 4)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                flush.zero_()
                pctx.cost_dev(KT, th_dev, out_dev)
            barrier()
            ps = [torch.cuda.Event(enable_timing=True) for _ in range(p_steps)]
            pe = [torch.cuda.Event(enable_timing=True) for _ in range(p_steps)]
            for i in range(p_steps):
                flush.zero_()
                ps[i].record(stream)
                pctx.cost_dev(KT, th_dev, out_dev)
                pe[i].record(stream)
            barrier()
        p_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(ps, pe)))
        pres = out_dev.view(KT, 5).cpu().numpy()
        next2 = {"evals_per_s": KT * p_steps / (p_ms * 1e-3), "ms_per_step": p_ms / p_steps,
                 "observables": pctx.num_observables(), "tasks": w.n_tasks,
                 "max_abs_cost_diff_vs_circuits": float(np.max(np.abs(pres[:, 0] - res[:, 0]))),
                 "note": ("NEXT-2 algebraic fast path (DVQLS_MODE_PAULI): U_b Z_j U_b^+ = X_j, each distinct "
                          "Pauli observable evaluated once per theta, Re/Im shared. Flagged: not circuits/s, "
                          "not the headline (SURVEY §8(d) headline rules)")}
        pctx.destroy()

    # ---- derived numbers -------------------------------------------------------------------------
    n_eval = (c1 - c0) if args.slice > 1 else w.n_circuits  # circuits this job evaluates per theta
    circuits_step = n_eval * KT
    value = circuits_step * args.steps / (dev_ms * 1e-3)
    e2e_value = circuits_step * args.steps / e2e_s
    had_ms = statistics.mean(t["hadamard_ms"] for t in kt)
    pre_ms = statistics.mean(t["prefix_ms"] for t in kt)
    red_ms = statistics.mean(t["reduce_ms"] for t in kt)
    local_c = np.arange(c0, c1)
    ops = fp64_ops_per_eval(w, local_c) * KT
    sbytes = smem_bytes_per_eval(w, local_c) * KT
    peaks, peak_src = load_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fmax = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    fp64_peak = 64 * sms * fmax  # FP64 pipe lane-ops/s at max clock
    smem_peak = 128 * sms * fmax  # B/s at max clock
    achieved_ops = ops / (had_ms * 1e-3)
    achieved_smem = sbytes / (had_ms * 1e-3)
    clocks = sampler.summary() if sampler else None

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "circuits/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": {
                "workload": w.name, "n_qubits": w.n, "L": w.L, "layers": w.layers,
                "circuits_per_eval": w.n_circuits, "thetas_per_step": KT,
                "l2": "flushed before every step (256 MiB write, outside the timed events)",
                "parallelism": (f"dp{world} (contiguous circuit blocks; 4 fp64 per theta summed across ranks by the "
                                "Hadamard kernel's tail over NVLink peer memory, NCCL allreduce as the fallback)"),
                **({"slice": f"rank 0's block of a {args.slice}-way split ({n_eval} circuits per theta): the "
                             "1-GPU weak-scaling reference"} if args.slice > 1 else {}),
            },
            "evals_per_s": KT * args.steps / (dev_ms * 1e-3),
            "k1": {"value": n_eval * k1_steps / (k1_ms * 1e-3), "unit": "circuits/s",
                   "ms_per_step": k1_ms / k1_steps, "evals_per_s": k1_steps / (k1_ms * 1e-3),
                   "kernel_ms": {"prefix": statistics.mean(t["prefix_ms"] for t in k1t),
                                 "hadamard": statistics.mean(t["hadamard_ms"] for t in k1t),
                                 "reduce": statistics.mean(t["reduce_ms"] for t in k1t)},
                   "note": "one cost evaluation per step (same loop, same L2 flush)"},
            "kernel_ms": {"prefix": pre_ms, "hadamard": had_ms, "reduce": red_ms},
            "roofline": streaming_roofline(w, local_c, KT, had_ms, peaks, peak_src, ctx.grid()) if w.n > 12 else
            onchip_roofline(w, local_c, KT, had_ms, sms, fmax, peak_src) if w.n > 10 else {
                "bound": "alu",
                "kernel": ("plane_kernel<20>" if w.n == 10 and w.bkind == 0 and os.environ.get("DVQLS_PLANE", "1") != "0"
                           else "hadamard_kernel"),
                "achieved": achieved_ops / 1e12,
                "peak": fp64_peak / 1e12,
                "unit": "Top/s",
                "frac": achieved_ops / fp64_peak,
                "traffic": traffic_from_profiles(),
                "note": ("FP64-pipe lane-ops (DADD and DFMA = 1 op each; the kernel is >95% DADD) per launch "
                         f"= {ops:.4g} (SURVEY §8(d)) / mean CUDA-event time of the kernel on the launching "
                         f"stream; peak = 64 lanes/clk/SM x {sms} SMs x sm_max_mhz ({peak_src} "
                         "MEASURED_PEAKS.json)"),
                "smem": {"achieved": achieved_smem / 1e9, "peak": smem_peak / 1e9, "unit": "GB/s",
                         "frac": achieved_smem / smem_peak,
                         "note": "on-chip model bytes: 96N per numerator circuit, 32N per denominator"},
                "model_frac": max(ops / fp64_peak, sbytes / smem_peak) / (had_ms * 1e-3),
            },
            "e2e": {"value": e2e_value, "unit": "circuits/s", "h2d_bytes_per_step": 8 * w.n_params * KT,
                    "d2h_bytes_per_step": 40 * KT},
            "gpu_launches": args.steps * ctx.launches_per_call(),
            "clocks": clocks,
            "cost": float(res[0, 0]),
            "cost_k1": float(res1[0]),
            "next2_pauli": next2,
            "next3_global": next3,
            "next4_decompose": next4,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w, thetas[0])
        print(json.dumps(line), flush=True)
    ctx.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
