#!/usr/bin/env python
"""Turn a tools/gpu_round2.sh run (gpurun_out/) into committed profiles/ summaries.

Usage: tools/round_report2.py [gpurun_out] [profiles] [tag, default r2]

Writes <tag>_bench_sweep.md/.jsonl, <tag>_bench_default.json,
<tag>_bench_reference.json, <tag>_launches_default.md/.csv, one
<tag>_ncu_<config>_<mode>.md per `ncu --set full` capture (key counters, stall
reasons, hottest SASS lines) and updates profiles/ncu_traffic.json (DRAM bytes
per launch, read by bench.py's roofline.traffic).
"""
import collections
import csv
import gzip
import io
import json
import os
import shutil
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
DST = sys.argv[2] if len(sys.argv) > 2 else "profiles"
TAG = sys.argv[3] if len(sys.argv) > 3 else "r2"
PEAK = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6545.9) if os.path.exists("MEASURED_PEAKS.json") else 6545.9

CONFIG_LABEL = {(256, 4096): "configs[0]", (512, 65536): "configs[1]", (1024, 2097152): "configs[4] 8-GPU shard",
                (1024, 16777216): "configs[4]", (4096, 4096): "configs[3] (both axes)"}


def label(c):
    return CONFIG_LABEL.get((c["n"], c["batch_per_gpu"]), "north-star target" if c["n"] == 512 else "")


def sweep():
    path = os.path.join(SRC, "bench_sweep.jsonl")
    if not os.path.exists(path):
        return
    rows = [json.loads(l) for l in open(path) if l.strip()]
    shutil.copy(path, os.path.join(DST, f"{TAG}_bench_sweep.jsonl"))
    out = [f"# {TAG}: bench sweep (1 B200, device-resident, CUDA-event timed)", "",
           f"`frac` = 16 B (fp64) / 8 B (fp32) per system-row per axis solve / mean launch time / {PEAK} GB/s "
           "(MEASURED_PEAKS.json). Source: `tools/gpu_round2.sh` -> gpurun_out/bench_sweep.jsonl.", "",
           "| workload | kind | N | systems | dtype | mode | variant | rows/s | frac | plan |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for d in rows:
        c = d["config"]
        var = "CN step" if c.get("cn_step") else ("periodic" if c.get("periodic") else "plain")
        out.append(f"| {label(c)} | {c['kind']} | {c['n']} | {c['batch_per_gpu']} | {d['dtype']} | {c['mode']} | {var} | "
                   f"{d['value']:.3e} | {d['roofline']['frac']:.3f} | {c['plan'][:70]} |")
    open(os.path.join(DST, f"{TAG}_bench_sweep.md"), "w").write("\n".join(out) + "\n")


def launches():
    path = os.path.join(SRC, "launches_default.csv")
    if not os.path.exists(path):
        return
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    shutil.copy(path, os.path.join(DST, f"{TAG}_launches_default.csv"))
    per = collections.OrderedDict()
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        per.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    out = [f"# {TAG}: ncu launch list of the default bench (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
           "dram__bytes_write.sum --clock-control none python bench.py --steps 3 --warmup 3`)", "",
           "Per-launch times are cold-cache and serialised (ncu); the sweep's SHARE of the step is the comparable "
           "number.", "", "| id | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | GB/s |", "|---|---|---|---|---|---|"]
    tot = collections.Counter()
    for (i, k), m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        unit_us = t / 1e3 if t > 1e5 else t  # ns vs us
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        name = k.split("(")[0][:70]
        tot[name] += unit_us
        gbs = (rd + wr) / (unit_us * 1e3) if unit_us else 0.0
        out.append(f"| {i} | `{name}` | {unit_us:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbs:.0f} |")
    allt = sum(tot.values()) or 1.0
    out += ["", "Share of GPU time by kernel: " + ", ".join(f"`{k}` {100 * v / allt:.1f}%" for k, v in tot.most_common())]
    open(os.path.join(DST, f"{TAG}_launches_default.md"), "w").write("\n".join(out) + "\n")
    # DRAM bytes per sweep launch of the default workload (single-pass
    # counters: the --set full replay of a 128 GiB in-place launch is not run)
    sw = [(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0), k) for (i, k), m in per.items()
          if "sweep_" in k]
    if not sw:
        return None
    return {"dram_bytes_per_launch": sum(b for b, _ in sw) / len(sw), "kernel": sw[0][1][:90],
            "source": f"profiles/{TAG}_launches_default.md (dram__bytes_read.sum + dram__bytes_write.sum, mean over "
                      f"{len(sw)} sweep launches of the default bench)"}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]


def ncu_reports(traffic):
    d = os.path.join(SRC, "ncu")
    if not os.path.isdir(d):
        return
    for f in sorted(os.listdir(d)):
        if not f.endswith(".raw.csv"):
            continue
        tag = f[:-len(".raw.csv")]
        rows = list(csv.reader(open(os.path.join(d, f))))
        if len(rows) < 3:
            continue
        hdr, units, vals = rows[0], rows[1], rows[2]
        m = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        kern = m.get("Kernel Name", "?")
        cfg, mode = tag.split("_", 1)
        t = float(m["gpu__time_duration.sum"])
        t_s = t * (1e-3 if u.get("gpu__time_duration.sum") == "ms" else 1e-6 if u.get("gpu__time_duration.sum") == "us"
                   else 1e-9)

        def gb(k):
            v = float(m.get(k, "0") or 0)
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u.get(k, "byte"), 1.0)

        dram = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
        out = [f"# {TAG}: ncu --set full, `{cfg}` {mode} mode", "",
               f"Kernel: `{kern[:150]}`", "",
               "Command: `ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 3 -c 1 "
               f"python bench.py --config {cfg} --mode {mode} --no-cpu --no-e2e --steps 2 --warmup 3` "
               "(tools/gpu_round2.sh). A number taken under ncu is never a bench value.", "",
               "| counter | value | unit |", "|---|---|---|"]
        for k in KEYS:
            if k in m:
                out.append(f"| {k} | {m[k]} | {u.get(k, '')} |")
        out += ["", f"DRAM bytes per launch: {dram / 1e9:.3f} GB; over {t_s * 1e3:.3f} ms = {dram / t_s / 1e9:.0f} GB/s "
                    f"({dram / t_s / 1e9 / PEAK:.3f} of {PEAK} GB/s)."]
        st = [(k, float(v or 0)) for k, v in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("_not_issued")]
        tot = sum(v for _, v in st) or 1.0
        out += ["", "Warp-state samples (all warps, incl. producer):", ""]
        out += [f"- {k[len('smsp__pcsamp_warps_issue_stalled_'):]}: {100 * v / tot:.1f}%"
                for k, v in sorted(st, key=lambda x: -x[1])[:8]]
        sass = os.path.join(d, tag + ".sass.csv.gz")
        if os.path.exists(sass):
            srows = list(csv.reader(io.StringIO(gzip.open(sass, "rt").read())))
            hi = next((i for i, r in enumerate(srows[:6]) if "Address" in r), None)
            if hi is not None:
                h = srows[hi]
                ix = {k: i for i, k in enumerate(h)}
                S = "Warp Stall Sampling (All Samples)"
                data = [r for r in srows[hi + 1:] if len(r) == len(h)]
                fv = lambda r: float(r[ix[S]] or 0) if S in ix else 0.0
                total = sum(fv(r) for r in data) or 1.0
                ops = collections.Counter()
                for r in data:
                    toks = [t for t in r[ix["Source"]].split() if not t.startswith("@")]
                    if toks:
                        ops[toks[0].split(".")[0]] += fv(r)
                out += ["", "Stall samples by SASS opcode: " +
                        ", ".join(f"{k} {100 * v / total:.1f}%" for k, v in ops.most_common(10)),
                        "", "Hottest SASS lines:", "", "```"]
                for r in sorted(data, key=lambda r: -fv(r))[:12]:
                    out.append(f"{100 * fv(r) / total:5.1f}%  {r[ix['Source']][:90]}")
                out.append("```")
                # tensor-core / TMA / TMEM proof
                mn = collections.Counter()
                for r in data:
                    op = r[ix["Source"]].split()
                    for t in op:
                        if t.split(".")[0] in ("UTMALDG", "UTMAPF", "UBLKCP", "UTMASTG", "STTM", "LDTM", "SYNCS"):
                            mn[t.split(".")[0]] += 1
                out += ["", "SASS proof of the Blackwell paths (instruction counts in the kernel): " +
                        ", ".join(f"{k} x{v}" for k, v in sorted(mn.items()))]
        open(os.path.join(DST, f"{TAG}_ncu_{tag}.md"), "w").write("\n".join(out) + "\n")
        traffic[f"{cfg}/{mode}"] = {"dram_bytes_per_launch": dram, "kernel": kern[:90],
                                    "source": f"profiles/{TAG}_ncu_{tag}.md (dram__bytes_read.sum + "
                                              "dram__bytes_write.sum, one ncu --set full capture)"}


def main():
    os.makedirs(DST, exist_ok=True)
    sweep()
    for src, dst in (("bench_default.json", "bench_default.json"), ("bench_ref.json", "bench_reference.json")):
        p = os.path.join(SRC, src)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(DST, f"{TAG}_{dst}"))
    dflt = launches()
    tp = os.path.join(DST, "ncu_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    if dflt:
        sys.path.insert(0, os.getcwd())
        import bench  # noqa: E402  (the default config / mode keys bench.py looks up)
        traffic[f"{bench.DEFAULT_CONFIG}/{bench.DEFAULT_MODE}"] = dflt
    ncu_reports(traffic)
    json.dump(traffic, open(tp, "w"), indent=1)
    print("written:", sorted(f for f in os.listdir(DST) if f.startswith(TAG)))


if __name__ == "__main__":
    main()
