#!/usr/bin/env python
"""Turn a tools/gpu_round.sh run (gpurun_out/) into the committed profiles/ summaries.

Usage: tools/round_report.py [gpurun_out] [profiles] [round tag, default r1]
Writes <tag>_bench_sweep.md/.jsonl, <tag>_bench_default.json, <tag>_bench_reference.json,
<tag>_launches_c2.md/.csv and <tag>_launches_c4tri_fast.md from the run's files.
"""
import collections
import csv
import json
import os
import shutil
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
DST = sys.argv[2] if len(sys.argv) > 2 else "profiles"
TAG = sys.argv[3] if len(sys.argv) > 3 else "r1"
PEAK = 6545.9


def label(c):
    n, m = c["n"], c["batch_per_gpu"]
    if n == 4096 and m == 4096:
        return "configs[3]"
    return {(256, 4096): "configs[0]", (512, 65536): "configs[1]", (1024, 2097152): "configs[4] shard"}.get(
        (n, m), "north-star target")


def sweep():
    rows = [json.loads(l) for l in open(os.path.join(SRC, "bench_sweep.jsonl")) if l.strip()]
    shutil.copy(os.path.join(SRC, "bench_sweep.jsonl"), os.path.join(DST, f"{TAG}_bench_sweep.jsonl"))
    out = [f"# Round {TAG[1:]} bench sweep (B200, 1 GPU, device-resident, CUDA-event timed)", "",
           "Command: `tools/gpu_round.sh` (`python bench.py --config C [--mode M] [--periodic|--cn] --no-cpu`).",
           "rows/s = systems x N (x2 axes for ADI) / time per step; frac = 16 B per row per axis (8 B fp32) / "
           f"step time / {PEAK} GB/s (MEASURED_PEAKS.json).",
           "`tmem=R`: rows per system kept in Tensor Memory; `head(L2)`: rows spilled to L2; `tail(smem)`: rows "
           "in shared memory; `partition K=..`: the partitioned fast path (DESIGN.md §3.4b).", "",
           "| config | kind | N | systems | dtype | mode | variant | rows/s | GB/s | frac | plan |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in rows:
        c = d["config"]
        var = "ADI" if c["n"] == 4096 and c["batch_per_gpu"] == 4096 else (
            "CN step" if c.get("cn_step") else ("periodic" if c.get("periodic") else "shared"))
        r = d["roofline"]
        out.append(f"| {label(c)} | {c['kind']} | {c['n']} | {c['batch_per_gpu']} | {d['dtype']} | {c['mode']} | "
                   f"{var} | {d['value']:.3e} | {r['achieved']:.0f} | {r['frac']:.3f} | {c['plan'][:80]} |")
    open(os.path.join(DST, f"{TAG}_bench_sweep.md"), "w").write("\n".join(out) + "\n")


def launches(csv_name, md_name, title):
    path = os.path.join(SRC, csv_name)
    if not os.path.exists(path):
        return
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.OrderedDict()
    for v in per.values():
        name = v["k"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0) / 1e3
        a[2] += v.get("dram__bytes_read.sum", 0.0) / 1e6
        a[3] += v.get("dram__bytes_write.sum", 0.0) / 1e6
    total = sum(a[1] for a in agg.values())
    out = [f"# ncu launch list: {title}", "",
           "`ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --clock-control none` "
           "(cold-cache, serialised: the share of the step, not the absolute time, is what matters).", "",
           "| kernel | launches | mean us | total us | share | DRAM read MB/launch | DRAM write MB/launch |",
           "|---|---|---|---|---|---|---|"]
    for name, (cnt, t, rd, wr) in agg.items():
        out.append(f"| {name} | {cnt} | {t / cnt:.1f} | {t:.1f} | {t / total:.1%} | {rd / cnt:.1f} | {wr / cnt:.1f} |")
    open(os.path.join(DST, md_name), "w").write("\n".join(out) + "\n")
    shutil.copy(path, os.path.join(DST, f"{TAG}_{csv_name}"))


def main():
    os.makedirs(DST, exist_ok=True)
    sweep()
    for src, dst in (("bench_default.json", "bench_default.json"), ("bench_ref.json", "bench_reference.json")):
        p = os.path.join(SRC, src)
        if os.path.exists(p) and os.path.getsize(p):
            shutil.copy(p, os.path.join(DST, f"{TAG}_{dst}"))
    launches("launches_c2.csv", f"{TAG}_launches_c2.md",
             "`python bench.py --steps 5 --warmup 3 --no-cpu` (configs[1], pent exact)")
    launches("launches_c4tri_fast.csv", f"{TAG}_launches_c4tri_fast.md",
             "`python bench.py --config c4tri --mode fast --steps 2 --warmup 3` (configs[3] ADI, partitioned path)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
