"""Top source lines by warp-stall samples from `ncu -i R --page source --csv --print-source sass,cuda`.

usage: python tools/ncu_lines.py <source.csv> [top]
"""
import csv
import sys

top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
fname, hdr, out = "?", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].strip().isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    stalls = {k: int(v or 0) for k, v in zip(hdr, r) if k.startswith("stall_") and "Not Issued" not in k
              and v.strip().isdigit()}
    best = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    out.append((samp, fname, r[0], r[1].strip()[:70], best))
tot = sum(o[0] for o in out) or 1
for samp, f, ln, src, best in sorted(out, key=lambda o: -o[0])[:top]:
    b = " ".join(f"{k[6:]}={100 * v / max(samp, 1):.0f}%" for k, v in best)
    print(f"{100 * samp / tot:5.1f}% {f}:{ln:<4} {src:70s} {b}")
