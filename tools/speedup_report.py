#!/usr/bin/env python
"""Speed-up surfaces from tools/gpu_speedup.sh CSVs.
Usage: tools/speedup_report.py [gpurun_out/speedup] [profiles] [tag]"""
import csv
import os
import shutil
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/speedup"
DST = sys.argv[2] if len(sys.argv) > 2 else "profiles"
TAG = sys.argv[3] if len(sys.argv) > 3 else "r2"


def table(rows, col, var):
    ns = sorted({int(r["n"]) for r in rows})
    ms = sorted({int(r["m"]) for r in rows})
    out = ["| N \\ M | " + " | ".join(str(m) for m in ms) + " |", "|---" * (len(ms) + 1) + "|"]
    for n in ns:
        cells = []
        for m in ms:
            v = [r[col] for r in rows if int(r["n"]) == n and int(r["m"]) == m and r["variant"] == var]
            cells.append(f"{float(v[0]):.2f}" if v else "")
        out.append(f"| {n} | " + " | ".join(cells) + " |")
    return out


def main():
    os.makedirs(os.path.join(DST, f"{TAG}_speedup"), exist_ok=True)
    out = [f"# {TAG}: speed-up surfaces on one B200 (the paper's Fig. 2-4 protocol)", "",
           "Crank-Nicolson time stepping (`bandsolve_bench_run`, the reference's `pde.cpp` driver) on the GPU, "
           "through `paper_1909_04539_b200/bandsolve_b200 bench` (the reference CLI's `run_bench`, same CSV "
           "schema); per cell the mean device time per step over the run's steps. Variants: `shared` (this "
           "library's shared-LHS sweep), `uniform` (scalar epsilon), `persystem` (this library's per-system "
           "kernels: band copies rewritten every step, the paper's cuThomasBatch/cuPentBatch protocol), "
           "`cusparse` (the same step with cuSPARSE `gtsvInterleavedBatch` (Thomas) / `gpsvInterleavedBatch` "
           "as the solver). Raw CSVs next to this file. Command: `tools/gpu_speedup.sh`.", ""]
    for prob in ("diffusion", "hyperdiffusion"):
        for mode in ("exact", "fast"):
            base = os.path.join(SRC, f"{prob}_{mode}")
            if not os.path.exists(base + ".csv"):
                continue
            for suf in (".csv", ".speedup.csv", ".speedup_cusparse.csv"):
                if os.path.exists(base + suf):
                    shutil.copy(base + suf, os.path.join(DST, f"{TAG}_speedup", f"{prob}_{mode}{suf}"))
            sp = list(csv.DictReader(open(base + ".speedup.csv")))
            sc = list(csv.DictReader(open(base + ".speedup_cusparse.csv")))
            out += [f"## {prob} ({'tridiagonal' if prob == 'diffusion' else 'pentadiagonal'}), {mode} mode", ""]
            out += ["Shared-LHS speed-up over cuSPARSE (time cusparse / time shared):", ""] + \
                table(sc, "speedup_vs_cusparse", "shared") + [""]
            out += ["Shared-LHS speed-up over the per-system kernels:", ""] + \
                table(sp, "speedup_vs_persystem", "shared") + [""]
            if any(r["variant"] == "uniform" for r in sp):
                out += ["Uniform (scalar epsilon) over per-system:", ""] + table(sp, "speedup_vs_persystem", "uniform") + [""]
            out += ["cuSPARSE over the per-system kernels:", ""] + table(sp, "speedup_vs_persystem", "cusparse") + [""]
    open(os.path.join(DST, f"{TAG}_speedup.md"), "w").write("\n".join(out) + "\n")
    print("written", os.path.join(DST, f"{TAG}_speedup.md"))


if __name__ == "__main__":
    main()
