"""Condense ncu artefacts into the text summaries committed under profiles/.

    python tools/profile_summary.py launches <launches.csv>            # per-kernel share of a step
    python tools/profile_summary.py full <report.ncu-rep> [kernel-regex]  # key counters + mix + stalls

`launches` reads the `--metrics gpu__time_duration.sum --csv` launch list;
`full` reads an `ncu --set full` report through `ncu -i ... --page raw/source --csv`.
"""

import csv
import io
import re
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "elapsed cycles/SM"),
    ("smsp__cycles_active.avg", "active cycles/SMSP"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "SMEM wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "SMEM wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "SMEM ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "SMEM st bank conflicts"),
    ("smsp__sass_data_bytes_mem_shared.sum", "SMEM data bytes"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[vi]:
            v = float(r[vi].replace(",", ""))
            if r[ui] in ("usecond", "us"):
                v *= 1e3
            elif r[ui] in ("msecond", "ms"):
                v *= 1e6
            d[re.sub(r"\(.*", "", r[ki])[:70]].append(v)
    ours = re.compile(r"dvqls|plane::|plane2::|pclus::|onchip::|streamp::|stream::|pauli::|decomp::|glob::|tile::|shift::")
    tot = sum(sum(v) for k, v in d.items() if ours.search(k))
    print(f"{'kernel':70s} {'launches':>8s} {'mean us':>10s} {'share of dvqls time':>20s}")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / tot:.1f}%" if ours.search(k) else "-"
        print(f"{k:70s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {share:>20s}")


def _ncu(rep, page, kernel):
    cmd = ["ncu", "-i", rep, "--page", page, "--csv"]
    if kernel:
        cmd += ["--kernel-name", f"regex:{kernel}"]
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def full(rep, kernel=None):
    raw = list(csv.reader(io.StringIO(_ncu(rep, "raw", kernel))))
    h, u = raw[0], raw[1]
    for row in raw[2:]:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"== {re.sub(r'[(].*', '', name)[:80]}")
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                print(f"  {label:28s} {row[i]} {u[i]}")
    src = list(csv.reader(io.StringIO(_ncu(rep, "source", kernel))))
    if len(src) < 3:
        return
    sh = src[1]
    si, ei = sh.index("Source"), sh.index("Instructions Executed")
    stall = [i for i, x in enumerate(sh) if x.startswith("stall_") and "Not Issued" not in x]
    ops, st, tot = Counter(), Counter(), 0
    for r in src[2:]:
        try:
            n = int(float(r[ei].replace(",", "")))
        except (ValueError, IndexError):
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si])
        ops[m.group(2) if m else "?"] += n
        tot += n
        for i in stall:
            try:
                st[sh[i]] += int(float(r[i] or 0))
            except ValueError:
                pass
    print(f"  dynamic instruction mix ({tot} warp instructions):")
    for op, n in ops.most_common(14):
        print(f"    {op:10s} {100 * n / tot:5.1f}%")
    s = sum(st.values())
    print(f"  warp stall samples ({s}):")
    for k, v in st.most_common(10):
        print(f"    {k:26s} {100 * v / max(s, 1):5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
