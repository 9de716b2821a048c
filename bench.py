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
dvqls_cost_dev, replayed as one CUDA graph per call with the Hadamard kernel launched as a
programmatic dependent of the prefix), timed with CUDA events on the library's stream, L2
flushed (256 MiB write) before every step, max over ranks.  `e2e` = the same metric through
the host-buffer C-ABI call dvqls_cost_batch / dvqls_cost (theta H2D + result D2H inside).
The per-kernel times behind `roofline` come from a second, identically configured context
with the library's CUDA events between the kernels (a probe loop in the same run).
The oracle (oracle/, test infrastructure) is only executed for `cpu_baseline`
(rank 0, N = 1) and for `--impl reference`.
"""

from __future__ import annotations

import argparse
import csv
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

CONFIGS = {"cfg1": configs.cfg1, "cfg3": configs.cfg3, "cfg4": configs.cfg4, "cfg5": configs.cfg5,
           "cfg5amp": configs.cfg5_amplitudes}
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


def hh_stream_bytes_per_eval(w, circuits=None):
    """Householder streaming kernel (stream_hh_kernel, n >= 13): per numerator circuit three read-only
    sweeps of the x gather (16N each) and of h (16N each) plus the readout's x (16N) = 112N; per
    denominator 32N.  x and h stay L2-resident up to n ~ 21, so these are L2 bytes there."""
    N = 1 << w.n
    c = np.arange(w.n_circuits) if circuits is None else circuits
    s = (c // 2) % (w.n + 1)
    num = int(np.count_nonzero(s))
    return num * 112 * N + (c.size - num) * 32 * N


def streaming_roofline(w, local_c, KT, had_ms, peaks, peak_src, grid=None):
    if w.bkind != 0:
        b = hh_stream_bytes_per_eval(w, local_c) * KT
        ach = b / (had_ms * 1e-3)
        peak = float(peaks["hbm_gbs"]) * 1e9
        in_l2 = KT * 16 * (1 << w.n) + 16 * (1 << w.n) <= 100 << 20  # x of every theta + h
        return {"bound": "l2" if in_l2 else "hbm", "kernel": "stream_hh_kernel<12>", "achieved": ach / 1e9,
                "peak": None if in_l2 else peak / 1e9, "unit": "GB/s", "frac": None if in_l2 else ach / peak,
                "traffic": None,
                "note": (f"algorithmic bytes per launch = {b:.4g} (112N per numerator circuit: three read-only "
                         "sweeps of x and h + the readout; 32N per denominator) / mean CUDA-event kernel time; "
                         + ("x and h are L2-resident here and MEASURED_PEAKS.json has no L2 figure, so no fraction"
                            if in_l2 else f"peak = hbm_gbs of {peak_src} MEASURED_PEAKS.json"))}
    b = hbm_bytes_per_eval(w, local_c) * KT
    b96 = smem_bytes_per_eval(w, local_c) * KT
    ach = b / (had_ms * 1e-3)
    peak = float(peaks["hbm_gbs"]) * 1e9
    plane = w.bkind == 0
    kern = (f"stream_plane_kernel<12, {'TMA-staged' if w.n >= 16 else 'direct'}>" if plane
            else "stream_hh_kernel<12>")
    out = {"bound": "hbm", "kernel": kern, "achieved": ach / 1e9, "peak": peak / 1e9,
           "unit": "GB/s", "frac": ach / peak, "traffic": None,
           "model96_GBps": b96 / (had_ms * 1e-3) / 1e9,
           "note": (f"algorithmic DRAM bytes per launch = {b:.4g} (64N per numerator circuit: 3 passes "
                    f"through the per-CTA scratch, x L2-resident; n >= 23: 160N + 32N per denominator) / mean "
                    f"CUDA-event kernel time; peak = hbm_gbs of {peak_src} MEASURED_PEAKS.json. model96_GBps "
                    f"= the SURVEY §8(d) 96N model (x reads counted as HBM); traffic: traffic_note")}
    if grid is not None:
        scratch = grid * (1 << w.n) * 8
        out["scratch_bytes"] = scratch
        if scratch <= 100 << 20:
            out["note"] += "; the per-CTA scratch fits in L2 at this n, so L2 bandwidth, not HBM, bounds it"
    return out


def onchip_roofline(w, local_c, KT, had_ms, sms, fmax, peak_src, kernel):
    """SMEM-resident paths (n <= 12): the SURVEY §8(d) on-chip model.  FP64-pipe ops ((4n+2)N per
    numerator circuit, 2N per denominator) against 64 lanes/clk/SM, on-chip bytes (96N per
    numerator circuit: x read twice + one whole-branch exchange per FWHT; 32N per denominator)
    against 128 B/clk/SM.  `bound` names the binding one (t_model = max of the two times) and
    `frac` = t_model / t_kernel, the §8(d) useful-work fraction; the other figure sits beside it."""
    ops = fp64_ops_per_eval(w, local_c) * KT
    sbytes = smem_bytes_per_eval(w, local_c) * KT
    fp64_peak = 64 * sms * fmax
    smem_peak = 128 * sms * fmax
    t = had_ms * 1e-3
    fp64 = {"achieved": ops / t / 1e12, "peak": fp64_peak / 1e12, "unit": "Top/s", "frac": ops / t / fp64_peak,
            "note": f"FP64-pipe lane-ops per launch = {ops:.4g} (DADD, DFMA = 1 op each)"}
    smem = {"achieved": sbytes / t / 1e9, "peak": smem_peak / 1e9, "unit": "GB/s", "frac": sbytes / t / smem_peak,
            "note": f"on-chip model bytes per launch = {sbytes:.4g} (96N per numerator circuit, 32N per denominator)"}
    smem_binds = sbytes / smem_peak >= ops / fp64_peak
    main, other, oname = (smem, fp64, "fp64") if smem_binds else (fp64, smem, "smem")
    return {"bound": "smem" if smem_binds else "alu", "kernel": kernel,
            "achieved": main["achieved"], "peak": main["peak"], "unit": main["unit"], "frac": main["frac"],
            "traffic": None, oname: other,
            "model_frac": max(ops / fp64_peak, sbytes / smem_peak) / t,
            "note": (f"{main['note']} / mean CUDA-event time of the kernel on the launching stream (probe "
                     f"context, same run); peak = {'128 B' if smem_binds else '64 lanes'}/clk/SM x {sms} SMs x "
                     f"sm_max_mhz ({peak_src} MEASURED_PEAKS.json; per-SM rates confirmed by "
                     f"tools/microbench.cu, profiles/r1_microbench.json). traffic: traffic_note (the kernel "
                     f"reads x, 16 KB per theta, and writes its terms)")}


# ----------------------------------------------------------------------------------------------
def parse_ncu_dram(rows):
    """{metric: value} of dram__bytes_read.sum / dram__bytes_write.sum from the rows of an
    `ncu --csv --print-units base` log (columns ... "Metric Name", "Metric Unit", "Metric Value";
    the ==PROF== lines and other metrics are skipped; the first captured launch wins)."""
    vals, hdr = {}, None
    for row in rows:
        if hdr is None:
            if "Metric Name" in row and "Metric Value" in row:
                hdr = (row.index("Metric Name"), row.index("Metric Value"))
            continue
        if len(row) > max(hdr) and row[hdr[0]] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            try:
                vals.setdefault(row[hdr[0]], float(row[hdr[1]].replace(",", "")))
            except ValueError:
                pass
    return vals


def measure_traffic(args, kernel):
    """roofline.traffic of THIS run's code and configuration: DRAM bytes (read + write) of the
    dominant kernel per launch, from ncu (dram__bytes_read.sum + dram__bytes_write.sum) on a child
    `bench.py --traffic-probe` with the same configuration (two calls of the measured launch
    sequence; the second launch is captured).  Never timed: the throughput numbers come from the
    uninstrumented run.  Returns (bytes or None, note)."""
    import shutil
    import subprocess
    import tempfile
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if ncu is None:
        return None, "ncu not found on this box"
    name = kernel.split("<")[0]
    fwd = ["--config", args.config, "--batch", str(args.batch), "--n", str(args.n), "--variant", str(args.variant),
           "--allreduce", args.allreduce, "--stream-grid", str(args.stream_grid)] + (["--no-graphs"] if args.no_graphs else [])
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "ncu.csv")
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--print-units", "base", "--csv",
               "-k", f"regex:{name}", "-s", "1", "-c", "1", "--log-file", log,
               sys.executable, os.path.abspath(__file__), *fwd, "--traffic-probe"]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=180)
            rows = list(csv.reader(open(log))) if os.path.exists(log) else []
        except (OSError, subprocess.SubprocessError) as e:
            return None, f"ncu capture failed: {type(e).__name__}"
    vals = parse_ncu_dram(rows)
    if len(vals) != 2:
        return None, f"ncu capture failed (rc {r.returncode}): {(r.stderr or r.stdout)[-200:].strip()}"
    return (vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
            f"DRAM bytes (read {vals['dram__bytes_read.sum']:.4g} + write {vals['dram__bytes_write.sum']:.4g}) "
            f"of one {name} launch of this configuration, ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
            "on a --traffic-probe child of this run (not timed)")


def _sized_sample(w, theta, mode, cores, target_s):
    """Evenly strided circuit sample whose oracle run takes ~target_s on `cores` threads: the sample
    doubles until one run takes >= 1 s, then it is scaled to the target (capped at the workload)."""
    from oracle import sim
    m = max(cores, 8)
    while True:
        idx = np.linspace(0, w.n_circuits - 1, m).astype(np.int64)
        t0 = time.perf_counter()
        sim.workload_terms(w, theta, mode=mode, idx=idx, nthreads=cores)
        dt = time.perf_counter() - t0
        if dt >= 1.0 or m >= w.n_circuits:
            break
        m = min(w.n_circuits, 2 * m)
    return int(min(w.n_circuits, max(m, m * target_s / max(dt, 1e-9))))


def cpu_baseline(w, theta, target_s=12.0):
    """Oracle (as it stands) on all host cores, bounded strided samples of the workload (~target_s of
    CPU work per mode)."""
    from oracle import sim
    cores = sim.hardware_threads()
    out = {"kind": "oracle", "cores": cores, "unit": "circuits/s"}
    res = {}
    for mode, name in ((0, "faithful"), (1, "prefix_shared")):
        m = _sized_sample(w, theta, mode, cores, target_s)
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
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
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
    ap.add_argument("--allreduce", default="p2p", choices=["p2p", "nccl"],
                    help="cross-rank reduction: fused into the kernel tail over NVLink peer memory, or NCCL")
    ap.add_argument("--no-graphs", action="store_true", help="plain launches instead of one CUDA graph per call")
    ap.add_argument("--variant", type=int, default=0, help="n = 10 kernel variant (dvqls_opts.variant)")
    ap.add_argument("--stream-grid", type=int, default=0, help="cap on the streaming kernels' CTAs (dvqls_opts.stream_grid)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next2", action="store_true", help="skip the NEXT-2 fast-path side measurement")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic capture of the kernel")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)  # run under ncu by measure_traffic
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = CONFIGS[args.config](args.n) if args.config.startswith("cfg5") else CONFIGS[args.config]()

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
        # one ncclUniqueId per communicator (the measured context, the probe context, NEXT-2's)
        obj = [[dvqls.dvqls_nccl_unique_id() for _ in range(3)] if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_ids = obj[0]
    else:
        nccl_ids = [None, None, None]

    stream = torch.cuda.Stream(device=dev)
    KT = args.batch
    chars, co = w.arrays()
    vopts = {"allreduce": dvqls.DVQLS_ALLREDUCE_NCCL if args.allreduce == "nccl" else dvqls.DVQLS_ALLREDUCE_P2P,
             "graphs": not args.no_graphs, "variant": args.variant, "stream_grid": args.stream_grid}
    if args.slice > 1:  # 1-GPU weak-scaling reference: rank 0's block of a SLICE-way split (virtual rank)
        if world > 1:
            raise SystemExit("--slice is the 1-GPU weak-scaling reference")
        vopts.update(virtual_rank=0, virtual_world=args.slice)

    def make_ctx(timing, nccl_id):
        # device memory comes from torch: the library carves its tables from this workspace
        ws_bytes = dvqls.workspace_size(w.n, w.layers, w.L, device=local, rank=rank, world=world,
                                        max_batch=max(KT, 1), **vopts)
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        return dvqls.Context(w.n, w.layers, chars, co, w.bkind, w.b, device=local, rank=rank, world=world,
                             nccl_id=nccl_id, entangler=w.entangler, stream=stream, timing=timing,
                             max_batch=max(KT, 1), workspace=workspace, **vopts)

    ctx = make_ctx(False, nccl_ids[0])   # the measured path: CUDA graph per call, PDL between prefix and kernel
    if args.traffic_probe:  # two calls of the measured launch sequence for ncu (measure_traffic), nothing else
        th = torch.tensor(np.stack([w.theta0(s) for s in range(KT)]), dtype=torch.float64, device=dev)
        out = torch.empty(5 * KT, dtype=torch.float64, device=dev)
        with torch.cuda.stream(stream):
            for _ in range(2):
                ctx.cost_dev(KT, th, out)
        torch.cuda.synchronize()
        ctx.destroy()
        return 0
    pctx = make_ctx(True, nccl_ids[1])   # probe: CUDA events between the kernels (per-kernel times, roofline)
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

    def warm(c, K, min_s=0.5):
        # W warm-up steps, continued (in chunks of 8, the same number on every rank: every call
        # contains a cross-rank reduction) until >= min_s of load so the SM clock has ramped
        t_w = time.time()
        i = 0
        chunk = 8
        while True:
            t_c = time.time()
            for _ in range(chunk):
                flush.zero_()
                c.cost_dev(K, th_dev, out_dev)
                i += 1
            torch.cuda.synchronize()
            if time.time() - t_c > 1.0:
                chunk = 1  # long steps (cfg5 at large n): warm up one call at a time
            more = 1.0 if (i < args.warmup or time.time() - t_w < min_s) else 0.0
            if world > 1:
                t = torch.tensor([more], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                more = float(t.item())
            if more == 0.0:
                return

    def timed(c, K, steps, probe=False):
        """device ms over `steps` calls (events on the library stream around each call), max over
        ranks; probe: also the library's per-kernel event times of every call"""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        kt = []
        barrier()
        for i in range(steps):
            flush.zero_()
            starts[i].record(stream)
            c.cost_dev(K, th_dev, out_dev)
            ends[i].record(stream)
            if probe:
                kt.append(c.last_timings())  # events of the library on the same stream
        barrier()
        return max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(starts, ends))), kt

    # ---- device-resident timed region (the headline) -----------------------------------------
    sampler = ClockSampler(list(range(world))) if rank == 0 else None
    if sampler:
        sampler.__enter__()
    with torch.cuda.stream(stream):
        warm(ctx, KT)
        if sampler:
            sampler.start()
        dev_ms, _ = timed(ctx, KT, args.steps)
        if sampler:
            sampler.stop()
        # ---- the same loop with a single theta per step (K = 1) --------------------------------
        k1_steps = max(3, args.steps // 2)
        warm(ctx, 1, 0.1)
        k1_ms, _ = timed(ctx, 1, k1_steps)
        res1 = out_dev[:5].cpu().numpy()
        warm(ctx, KT, 0.1)
        ctx.check()
        res = out_dev.view(KT, 5).cpu().numpy()
        # ---- probe context: per-kernel CUDA-event times (roofline), K and K = 1 -----------------
        probe_steps = max(3, args.steps // 4)
        warm(pctx, KT, 0.2)
        probe_ms, kt = timed(pctx, KT, probe_steps, probe=True)
        warm(pctx, 1, 0.05)
        _, k1t = timed(pctx, 1, probe_steps, probe=True)
    if sampler:
        sampler.__exit__()
    if not np.all(np.isfinite(res[:, 0])) and args.slice <= 1:
        print("error: non-finite cost", res, file=sys.stderr)
        return 1

    # ---- end-to-end through the host-buffer C ABI (theta H2D + result D2H every step) ----------
    def e2e_time(K, steps):
        tot = 0.0
        for _ in range(2):
            ctx.cost_batch(thetas[:K]) if K > 1 else ctx.cost(thetas[0])
        barrier()
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if K > 1:
                ctx.cost_batch(thetas[:K])
            else:
                ctx.cost(thetas[0])
            tot += time.perf_counter() - t0
        barrier()
        return max_over_ranks(tot)

    e2e_s = e2e_time(KT, args.steps)
    e2e1_s = e2e_time(1, k1_steps)

    # ---- NEXT-3 global cost: C_L and C_G of the same call (dvqls_costs_dev) ----------------------
    next3 = None
    if not args.no_next2 and args.slice <= 1:
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
        moved = 16 * 4 ** nd     # this design: the XOR diagonals gathered straight from A (round 1: 48 * 4^n)
        pk = float(load_peaks()[0]["hbm_gbs"])
        next4 = {"n": nd, "terms": len(terms), "ms": best, "GBps": byts / (best * 1e-3) / 1e9,
                 "hbm_frac": byts / (best * 1e-3) / 1e9 / pk,
                 "moved_GBps": moved / (best * 1e-3) / 1e9, "moved_frac": moved / (best * 1e-3) / 1e9 / pk,
                 "note": ("NEXT-4: 4^n coefficients by one FWHT per x-mask of the XOR diagonal gathered from A, one "
                          "candidate pass (Parseval bound from ||A||_F^2 summed during the upload; exact norm filter "
                          "in the sort) + sort on the GPU; GBps = algorithmic bytes 16*4^n (A read once) over the "
                          "device time after the upload (best of 3)")}
        del A

    # ---- NEXT-2 algebraic fast path (flagged; reported separately, never the headline) ----------
    next2 = None
    if w.bkind == 0 and not args.no_next2 and args.slice <= 1:
        nctx = dvqls.Context(w.n, w.layers, chars, co, w.bkind, w.b, device=local, rank=rank, world=world,
                             nccl_id=nccl_ids[2], entangler=w.entangler, stream=stream, timing=False,
                             max_batch=max(KT, 1), mode=dvqls.DVQLS_MODE_PAULI)
        p_steps = max(3, args.steps // 4)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                flush.zero_()
                nctx.cost_dev(KT, th_dev, out_dev)
            barrier()
            ps = [torch.cuda.Event(enable_timing=True) for _ in range(p_steps)]
            pe = [torch.cuda.Event(enable_timing=True) for _ in range(p_steps)]
            for i in range(p_steps):
                flush.zero_()
                ps[i].record(stream)
                nctx.cost_dev(KT, th_dev, out_dev)
                pe[i].record(stream)
            barrier()
        p_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(ps, pe)))
        pres = out_dev.view(KT, 5).cpu().numpy()
        next2 = {"evals_per_s": KT * p_steps / (p_ms * 1e-3), "ms_per_step": p_ms / p_steps,
                 "observables": nctx.num_observables(), "tasks": w.n_tasks,
                 "max_abs_cost_diff_vs_circuits": float(np.max(np.abs(pres[:, 0] - res[:, 0]))),
                 "note": ("NEXT-2 algebraic fast path (DVQLS_MODE_PAULI): U_b Z_j U_b^+ = X_j, each distinct "
                          "Pauli observable evaluated once per theta, Re/Im shared. Flagged: not circuits/s, "
                          "not the headline (SURVEY §8(d) headline rules)")}
        nctx.destroy()

    # ---- parameter-shift gradient (NEXT-1 with 2P shift points; every circuit simulated) --------
    grad = None
    if not args.no_next2 and args.slice <= 1 and w.n <= 12:
        gout = torch.empty(1 + w.n_params + 4, dtype=torch.float64, device=dev)
        with torch.cuda.stream(stream):
            ctx.cost_grad_dev(th_dev[0], gout)
            barrier()
            g_steps = 3
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(g_steps):
                ctx.cost_grad_dev(th_dev[0], gout)
            e1.record(stream)
            barrier()
        gms = max_over_ranks(e0.elapsed_time(e1)) / g_steps
        rows = 2 * w.n_params + 1
        grad = {"grads_per_s": 1e3 / gms, "ms_per_grad": gms, "cost_evals_per_grad": rows,
                "circuits_per_s": rows * w.n_circuits / (gms * 1e-3),
                "note": (f"dvqls_cost_grad_dev: the 2P = {2 * w.n_params} parameter-shifted thetas + theta, "
                         f"evaluated in batches of {KT} through the circuit path (one CUDA graph), quotient rule "
                         "on the device")}

    # ---- derived numbers -------------------------------------------------------------------------
    n_eval = (c1 - c0) if args.slice > 1 else w.n_circuits  # circuits this job evaluates per theta
    circuits_step = n_eval * KT
    value = circuits_step * args.steps / (dev_ms * 1e-3)
    e2e_value = circuits_step * args.steps / e2e_s
    had_ms = statistics.mean(t["hadamard_ms"] for t in kt)
    pre_ms = statistics.mean(t["prefix_ms"] for t in kt)
    red_ms = statistics.mean(t["reduce_ms"] for t in kt)
    local_c = np.arange(c0, c1)
    peaks, peak_src = load_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fmax = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    clocks = sampler.summary() if sampler else None
    if w.n > 12:
        roof = streaming_roofline(w, local_c, KT, had_ms, peaks, peak_src, ctx.grid())
    else:
        kern = (("plane_kernel<20>" if args.variant == 1 else "plane2_kernel") if w.n == 10 and w.bkind == 0 else
                f"onchip_plane_kernel<{w.n}>" if w.n > 10 and w.bkind == 0 else
                "stream_hadamard_kernel<HH>" if w.n > 10 else "hadamard_kernel")
        roof = onchip_roofline(w, local_c, KT, had_ms, sms, fmax, peak_src, kern)

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
                "launch": "one CUDA graph per call (prefix -> [PDL] Hadamard kernel with fused reduction)",
                "parallelism": (f"dp{world} (contiguous circuit blocks; 4 fp64 per theta summed across ranks by the "
                                "Hadamard kernel's tail over NVLink peer memory, NCCL allreduce as the fallback)"),
                **({"slice": f"rank 0's block of a {args.slice}-way split ({n_eval} circuits per theta, "
                             "virtual rank): the 1-GPU weak-scaling reference"} if args.slice > 1 else {}),
            },
            "evals_per_s": KT * args.steps / (dev_ms * 1e-3),
            "k1": {"value": n_eval * k1_steps / (k1_ms * 1e-3), "unit": "circuits/s",
                   "ms_per_step": k1_ms / k1_steps, "evals_per_s": k1_steps / (k1_ms * 1e-3),
                   "e2e": {"value": n_eval * k1_steps / e2e1_s, "unit": "circuits/s",
                           "h2d_bytes_per_step": 8 * w.n_params, "d2h_bytes_per_step": 8 * 6},
                   "kernel_ms": {"prefix": statistics.mean(t["prefix_ms"] for t in k1t),
                                 "hadamard": statistics.mean(t["hadamard_ms"] for t in k1t),
                                 "reduce": statistics.mean(t["reduce_ms"] for t in k1t)},
                   "note": "one cost evaluation per step (same loop, same L2 flush)"},
            "kernel_ms": {"prefix": pre_ms, "hadamard": had_ms, "reduce": red_ms,
                          "probe_step_ms": probe_ms / probe_steps,
                          "note": "probe context (CUDA events between the kernels, no graph, no PDL)"},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "circuits/s", "h2d_bytes_per_step": 8 * w.n_params * KT,
                    "d2h_bytes_per_step": 8 * (5 * KT + 1)},
            "gpu_launches": args.steps * ctx.launches_per_call(),
            "graphs": ctx.num_graphs(),
            "clocks": clocks,
            "cost": float(res[0, 0]),
            "cost_k1": float(res1[0]),
            "shift_grad": grad,
            "next2_pauli": next2,
            "next3_global": next3,
            "next4_decompose": next4,
        }
        if world == 1 and not args.no_traffic:
            roof["traffic"], roof["traffic_note"] = measure_traffic(args, roof["kernel"])
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w, thetas[0])
        print(json.dumps(line), flush=True)
    pctx.destroy()
    ctx.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
