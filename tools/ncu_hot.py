#!/usr/bin/env python
"""Hottest SASS instructions of an ncu report with their stall-reason split.
Usage: tools/ncu_hot.py <report.ncu-rep> [top=20]"""
import csv
import io
import subprocess
import sys

REASONS = ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_selected", "stall_math", "stall_mio",
           "stall_branch_resolving", "stall_lg", "stall_no_inst", "stall_dispatch"]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    S = "Warp Stall Sampling (All Samples)"
    f = lambda r, k: float(r[idx[k]] or 0) if k in idx else 0.0
    tot = sum(f(r, S) for r in data) or 1.0
    order = sorted(range(len(data)), key=lambda i: -f(data[i], S))[:top]
    for i in sorted(order):
        r = data[i]
        split = ", ".join(f"{k[6:]} {100 * f(r, k) / max(f(r, S), 1):.0f}%" for k in REASONS if f(r, k) > 0.1 * f(r, S))
        print(f"{r[idx['Address']][-5:]} {100 * f(r, S) / tot:5.1f}%  {r[idx['Source']][:58]:58s} [{split}]")
    agg = {k: sum(f(r, k) for r in data) for k in REASONS}
    print("total:", ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])))


if __name__ == "__main__":
    main()
