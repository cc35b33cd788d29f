#!/usr/bin/env python
"""Summarise an ncu report: key throughput/traffic metrics and top stall reasons.
Usage: tools/ncu_summary.py <report.ncu-rep> [algorithmic_bytes]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__warps_active.avg.per_cycle_active", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        kernels.append({h: (v, u) for h, v, u in zip(hdr, vals, units)})
    return kernels


def main():
    path = sys.argv[1]
    algo = float(sys.argv[2]) if len(sys.argv) > 2 else None
    for d in raw(path):
        print(f"kernel: {d.get('Kernel Name', ('?',))[0][:110]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k][0]:>18s} {d[k][1]}")
        stalls = []
        for k, (v, _) in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("  stall samples: " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))
        if algo:
            rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(d["dram__bytes_read.sum"][1], 1)
            wr *= scale.get(d["dram__bytes_write.sum"][1], 1)
            print(f"  dram traffic / algorithmic = {(rd + wr) / algo:.3f}  ({(rd + wr) / 1e9:.3f} GB vs {algo / 1e9:.3f} GB)")


if __name__ == "__main__":
    main()
