#!/usr/bin/env python
"""Summarize an ncu launch-list CSV (gpu__time_duration.sum) into per-kernel totals and shares.

Usage: python scripts/summarize_ncu.py gpurun_out/launches_c3_r1.csv > profiles/r1_launches_c3.md
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    kn, mn, mv, un = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        v = float(r[mv].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[un], 1e-6)
        name = r[kn].split("(")[0].replace("void ", "").strip()
        tot[name] += v * scale
        cnt[name] += 1
    allms = sum(tot.values())
    print(f"# ncu launch list: {path}\n")
    print("cold-cache, serialised replay (compare shares, not absolute times)\n")
    print("| kernel | launches | total ms | avg ms | share |")
    print("|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| `{k}` | {cnt[k]} | {tot[k]:.3f} | {tot[k] / cnt[k]:.4f} | {100 * tot[k] / allms:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
