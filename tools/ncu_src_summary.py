"""Summarise an `ncu --page source --csv` dump: dynamic instruction mix and stall reasons.

usage: python tools/ncu_src_summary.py <source.csv>
"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ei = h.index("Source"), h.index("Instructions Executed")
stall = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
ops, st = Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ei or not r[ei].strip():
        continue
    try:
        n = int(float(r[ei].replace(",", "")))
    except ValueError:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si])
    op = m.group(2) if m else "?"
    ops[op] += n
    tot += n
    for i in stall:
        try:
            st[h[i]] += int(float(r[i] or 0))
        except ValueError:
            pass
print(f"dynamic warp instructions: {tot}")
for op, n in ops.most_common(25):
    print(f"  {op:10s} {n:12d} {100*n/tot:5.1f}%")
s = sum(st.values())
print("stall samples:", s)
for k, v in st.most_common(12):
    print(f"  {k:28s} {v:9d} {100*v/max(s,1):5.1f}%")
