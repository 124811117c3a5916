#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from `ncu -i rep --page source --csv` output.
Usage: ncu -i X.ncu-rep --page source --csv > x.csv; python scripts/ncu_top_sass.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iss] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for s, a, src in sorted(data, reverse=True)[:N]:
    print(f"{100*s/tot:5.1f}% {a} {src}")
