#!/usr/bin/env python
"""Key metrics of one or more `ncu --set full` reports (.ncu-rep) as a markdown table.

Usage: python scripts/ncu_metrics.py gpurun_out/prof_k_step3_tc_c3_r1.ncu-rep [...]
"""
import csv
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_issue_stalled_barrier", None),
]


def metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def main(paths):
    print("| metric | " + " | ".join(p.split("/")[-1].replace(".ncu-rep", "") for p in paths) + " |")
    print("|---|" + "---|" * len(paths))
    ms = [metrics(p) for p in paths]
    for key, label in METRICS:
        if label is None:
            continue
        cells = []
        for m in ms:
            v = m.get(key)
            cells.append(f"{v[0]} {v[1]}".strip() if v else "-")
        print(f"| {label} (`{key}`) | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
