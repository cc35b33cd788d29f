#!/usr/bin/env python
"""Shared-LHS batch solve throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--mode exact|fast]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N     (N > 1)
    python bench.py --impl reference                                            (CPU reference arm)

A step is one in-place solve of one synthetic batch. Default workload is
BASELINE.json configs[4], the configuration the metric is quoted on at
1/2/4/8 B200: pentadiagonal shared-LHS, fp64, N = 1024 rows, a global batch
of 2^24 systems (128 GiB) sharded across the GPUs ("strong" scaling: rank g
of G solves columns [M g/G, M (g+1)/G) of the one global batch, the
reference's split, parallel.cpp:53-54, via partition.shard_range),
hyperdiffusion LHS sigma_x = 1 (pde.cpp:67-71). At one GPU the whole
128 GiB batch is one device-resident in-place buffer (1000x the L2, so every
step streams from HBM). Other configs (--config) are per-GPU ("weak")
workloads. No data-path collective: NCCL carries only the start barrier and
the max-over-ranks of the device time.

Prints one JSON line on rank 0. Fields: value (device-resident, CUDA-event
timed), e2e (through the reference-facing C ABI with a pinned host batch,
H2D + sweep + D2H inside the timed region), roofline of the sweep kernel
against MEASURED_PEAKS.json, cpu_baseline (the reference CPU solver on this
host), clocks sampled during the timed regions.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "batch·N rows solved/s (fp64) and % of HBM roofline at 1/2/4/8 B200 vs CPU ref"

CONFIGS = {
    # name: (kind, n, systems per GPU, description); STRONG configs give the
    # GLOBAL batch instead, sharded across the ranks
    "c1": ("tri", 256, 4096, "configs[0]: tridiagonal shared-LHS, N=256, batch=4096, diffusion LHS sigma_x=1"),
    "c2": ("pent", 512, 65536, "configs[1]: pentadiagonal shared-LHS, N=512, batch=65536, hyperdiffusion LHS sigma_x=1"),
    "tri512": ("tri", 512, 1 << 20, "north-star target: tridiagonal N=512, batch=2^20, diffusion LHS sigma_x=1"),
    "pent512": ("pent", 512, 1 << 20, "north-star target: pentadiagonal N=512, batch=2^20, hyperdiffusion sigma_x=1"),
    "c5": ("pent", 1024, 1 << 24, "configs[4]: pentadiagonal shared-LHS, N=1024, batch=2^24 sharded across the "
                                  "GPUs, hyperdiffusion LHS sigma_x=1"),
    "c5s": ("pent", 1024, 1 << 21, "configs[4] shard: pentadiagonal N=1024, 2^21 systems per GPU (the 8-GPU shard)"),
    "c4tri": ("tri", 4096, 4096, "configs[3]: 2D ADI step (Peaceman-Rachford, periodic diffusion) on a 4096x4096 "
                                 "grid, tridiagonal solves along both axes"),
    "c4pent": ("pent", 4096, 4096, "configs[3]: 2D ADI step (periodic hyperdiffusion) on a 4096x4096 grid, "
                                   "pentadiagonal solves along both axes"),
}
STRONG = {"c5"}
DEFAULT_CONFIG = "c5"
DEFAULT_MODE = "fast"
E2E_MAX_SYSTEMS = 1 << 21  # pinned host batch for e2e, split over the ranks (16 GiB at N=1024): host RAM bound
SEED = 42

NVML_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


def lhs_for(kind: str, n: int):
    from paper_1909_04539_b200 import bandsolve as bs
    return bs.diffusion_bands(1.0, n) if kind == "tri" else bs.hyper_bands(1.0, n)


# ---- clocks -------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while marked windows are open."""

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.samples: list[tuple[float, int, int]] = []
        self.windows: list[tuple[float, float]] = []
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.period = period_s
        self.stop_evt = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                clk = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), clk, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def window(self):
        sampler = self

        class _W:
            def __enter__(self):
                self.t0 = time.perf_counter()

            def __exit__(self, *a):
                sampler.windows.append((self.t0, time.perf_counter()))
        return _W()

    def summary(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_evt.set()
        self.th.join(timeout=1)
        inside = [s for s in self.samples if any(a <= s[0] <= b for a, b in self.windows)]
        use = inside or self.samples
        reasons = set()
        for _, _, rs in use:
            for bit, name in NVML_REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(c for _, c, _ in use) if use else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(use), "samples_in_timed_regions": len(inside)}


# ---- CPU reference ------------------------------------------------------------------------
def reference_library():
    """(Library, kind): the reference compiled from its own sources
    (oracle/_ref, built here and shipped with the repo snapshot), else None."""
    from oracle.oracle import REF_LIB, build_ref
    from paper_1909_04539_b200.bandsolve import Library
    path = REF_LIB if os.path.exists(REF_LIB) else build_ref()
    if path and os.path.exists(path):
        return Library(path), "reference"
    return None, "port"


def cpu_solve_fn(kind: str, n: int, m: int):
    """Return (solve() -> seconds, cores, kind, sample) for the CPU reference
    on an n x m batch. The factor is created outside the timing, as in the
    paper."""
    from oracle.oracle import Oracle
    orc = Oracle()
    rhs = orc.rhs(SEED, n, m)
    bands = lhs_for(kind, n)
    lib, lkind = reference_library()
    if lib is not None:
        from paper_1909_04539_b200.bandsolve import Batch, PentFactor, TriFactor
        cores = os.cpu_count() or 1
        lib.set_threads(cores)
        fac = TriFactor(lib, *bands) if kind == "tri" else PentFactor(lib, *bands)
        batch = Batch.from_array(lib, rhs)

        def solve():
            batch.array[...] = rhs  # restore b (outside the timed call)
            t0 = time.perf_counter()
            fac.solve(batch)
            return time.perf_counter() - t0
        return solve, cores, lkind
    f = orc.tri_prefactor(*bands) if kind == "tri" else orc.pent_prefactor(*bands)

    def solve_port():
        x = rhs.copy()
        t0 = time.perf_counter()
        (orc.tri_solve if kind == "tri" else orc.pent_solve)(f, x)
        return time.perf_counter() - t0
    return solve_port, 1, "port"


def cpu_sample_columns(n: int, m: int, budget_rows: int = 1 << 26) -> int:
    """Bounded CPU sample: whole batch when small, else a column subsample."""
    return max(1, min(m, budget_rows // n))


def cpu_baseline(kind: str, n: int, m: int, seconds: float = 4.0) -> dict:
    ms = cpu_sample_columns(n, m)
    solve, cores, lkind = cpu_solve_fn(kind, n, ms)
    solve()  # warm-up (first-touch, thread team)
    times = []
    t_end = time.perf_counter() + seconds
    while len(times) < 3 or (time.perf_counter() < t_end and len(times) < 200):
        times.append(solve())
    t = statistics.median(times)
    return {"value": n * ms / t, "unit": "rows/s", "cores": cores, "kind": lkind,
            "sample": f"{kind} N={n} x {ms} systems ({'full batch' if ms == m else 'column subsample'}), "
                      f"median of {len(times)} solves, bandsolve_{kind}_solve_shared, "
                      f"{cores} threads, {os.cpu_count()} host cores"}


def run_reference_arm(args, rank: int) -> None:
    if rank != 0:
        return
    kind, n, m, desc = CONFIGS[args.config]
    ms = cpu_sample_columns(n, m)
    solve, cores, lkind = cpu_solve_fn(kind, n, ms)
    for _ in range(args.warmup):
        solve()
    times = [solve() for _ in range(args.steps)]
    total = sum(times)
    value = n * ms * len(times) / total
    sample = (f"{kind} N={n} x {ms} systems ({'full batch' if ms == m else 'column subsample'}) per step, "
              f"{cores} threads on {os.cpu_count()} host cores")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
            "higher_is_better": True, "scaling": "strong" if args.config in STRONG else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": desc, "kind": kind, "n": n, "batch": ms},
            "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": lkind, "sample": sample},
            "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- GPU arm --------------------------------------------------------------------------------
def load_peak() -> tuple[float, str]:
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(config: str, mode: str) -> float | None:
    """Per-launch DRAM bytes of the sweep kernel from the committed ncu capture."""
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return float(json.load(f)[f"{config}/{mode}"]["dram_bytes_per_launch"])
    except Exception:
        return None


def sustained_copy_gbs(torch, ms_timed: float) -> float | None:
    """Device copy rate (read + write bytes) back to back for as long as the
    timed region lasted (0.2-1.5 s), right after it: what the board sustains
    under its power cap for a long step, next to the burst copy figure of
    MEASURED_PEAKS.json that `frac` is quoted against. Context only."""
    if ms_timed < 100.0:
        return None
    try:
        nbytes = 2 << 30
        a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        b = torch.empty_like(a)
        a.fill_(1)
        b.copy_(a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        reps = max(4, int(min(max(ms_timed, 200.0), 1500.0) / max(e0.elapsed_time(e1), 1e-3)))
        e0.record()
        for _ in range(reps):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        gbs = 2.0 * nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
        del a, b
        torch.cuda.empty_cache()
        return gbs
    except Exception:  # no room next to the batch: leave it out
        return None


def kernel_name(plan: str, f32: bool, kind: str, mode: str) -> str:
    """Name of the sweep kernel the plan launches (what ncu lists)."""
    k = plan.split()[0] if plan else "?"
    name = {"stream": "sweep_stream", "regs": "sweep_regs", "persist": "sweep_persist",
            "smem-tma": "sweep_smem", "global-inplace": "sweep_global",
            "partition": "part_fwd_kernel+part_bwd_kernel", "spike": "sweep_spike"}.get(k, k)
    return f"{name}<{'float' if f32 else 'double'},{kind},{mode}>"


def run_gpu_arm(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_1909_04539_b200 import bandsolve as bs

    torch.cuda.set_device(local_rank)
    lib = bs.load()
    lib.set_mode(bs.MODE_FAST if args.mode == "fast" else bs.MODE_EXACT)
    from paper_1909_04539_b200.partition import shard_range, weak_shard

    kind, n, m_cfg, desc = CONFIGS[args.config]
    strong = args.config in STRONG
    # this rank's shard [j0, j1) of the global batch
    j0, j1 = shard_range(m_cfg, rank, world) if strong else weak_shard(m_cfg, rank)
    m = j1 - j0
    m_global = m_cfg if strong else m_cfg * world
    elem = 4 if args.f32 else 8
    dt = torch.float32 if args.f32 else torch.float64
    bands = lhs_for(kind, n)
    adi = args.config.startswith("c4")
    args.periodic = args.periodic or args.cn
    if adi:  # field C[y][x] = n x m; one step = an x-sweep and a y-sweep
        fac = bs.ADI(lib, 0 if kind == "tri" else 1, 1.0, m, n)
    elif args.periodic:  # cyclic constant-band system: shared sweep of A' + wrap correction
        consts = (-1.0, 3.0, -1.0) if kind == "tri" else (1.0, -4.0, 7.0, -4.0, 1.0)
        fac = bs.PeriodicTri(lib, *consts, n) if kind == "tri" else bs.PeriodicPent(lib, *consts, n)
        if args.f32:
            raise SystemExit("--periodic is fp64 only")
    else:
        fac = bs.TriFactor(lib, *bands) if kind == "tri" else bs.PentFactor(lib, *bands)

    # Every timed step must stream from HBM: one in-place buffer when it alone
    # is >= 4x the 126 MB L2 (configs[4]: 128 GiB at one GPU), else rotating
    # in-place buffers whose working set is >= 4x L2. ADI and CN steps
    # ping-pong between two buffers.
    l2 = 132644864
    bytes_per = n * m * elem
    nbuf = 1 if bytes_per >= 4 * l2 else -(-4 * l2 // bytes_per)  # configs[0] (8 MiB): 64 buffers
    if adi or args.cn:
        nbuf = max(2, nbuf)
    ld = m + args.pitch_pad  # row pitch of the device batch (elements)
    bufs = [torch.empty((n, ld), dtype=dt, device="cuda") for _ in range(nbuf)]
    for b in bufs:
        lib.fill_rhs_dev(b.data_ptr(), n, m, ld, SEED, j0, torch.cuda.current_stream().cuda_stream, f32=args.f32)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    clocks = ClockSampler(local_rank)

    cn_sigma = 1.0  # pde.cpp default dt: sigma_x = 1

    def step(k):
        if adi:
            fac.step_dev(bufs[k % nbuf].data_ptr(), bufs[(k + 1) % nbuf].data_ptr(), ld=ld, stream=sptr)
        elif args.cn:  # one Crank-Nicolson step: u_{k+1} = A^-1 B u_k, ping-pong buffers
            fac.cn_step_dev(cn_sigma, bufs[k % nbuf].data_ptr(), bufs[(k + 1) % nbuf].data_ptr(), n, m, ld=ld,
                            stream=sptr)
        else:
            fac.solve_dev(bufs[k % nbuf].data_ptr(), n, m, ld=ld, stream=sptr, f32=args.f32)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks.window():
        e0.record(stream)
        for k in range(args.steps):
            step(k)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    ms_local = e0.elapsed_time(e1)
    t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    axes = 2 if adi else 1  # an ADI step solves every grid point along both axes
    rows_total = float(n) * m_global * args.steps * axes
    value = rows_total / (ms_max / 1e3)
    ms_per_step = ms_max / args.steps

    # roofline of the sweep kernel: algorithmic bytes (read b once, write x
    # once) per launch / average launch duration on the launching stream
    algo_bytes = 2.0 * elem * n * m * axes  # 16 B per point per axis solve
    achieved = algo_bytes / (ms_local / args.steps / 1e3) / 1e9
    peak, peak_src = load_peak()
    traffic = load_traffic(args.config, args.mode)
    sustained = sustained_copy_gbs(torch, ms_local) if not args.no_sustained else None
    plan = lib.describe_plan(0 if kind == "tri" else 1, n, m, ld, args.f32)

    # e2e through the reference-facing host API (pinned host batch; H2D,
    # sweep, D2H inside bandsolve_*_solve_shared, synchronous)
    e2e = None
    if not args.f32 and not args.cn and not adi and not args.no_e2e:
        # pinned host batch of this rank's columns (a leading column sample
        # when the shard exceeds E2E_MAX_SYSTEMS: host RAM, not the device,
        # bounds it), regenerated from the same generator indices
        me = min(m, max(32, E2E_MAX_SYSTEMS // world // 32 * 32))  # 16 GiB of pinned host memory in all
        host = bs.Batch(lib, n, me)
        tmp = torch.empty((n, me), dtype=torch.float64, device="cuda")
        lib.fill_rhs_dev(tmp.data_ptr(), n, me, me, SEED, j0, sptr)
        torch.from_numpy(host.array).copy_(tmp)
        del tmp
        torch.cuda.empty_cache()
        e2e_steps = max(1, min(args.steps, 50, (32 << 30) // (n * me * 8)))
        fac.solve(host)  # warm-up
        if world > 1:
            dist.barrier()
        with clocks.window():
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                fac.solve(host)
            t_e2e = time.perf_counter() - t0
        te = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        me_total = torch.tensor([me], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(me_total, op=dist.ReduceOp.SUM)
        e2e = {"value": float(n) * float(me_total.item()) * e2e_steps / float(te.item()), "unit": "rows/s",
               "h2d_bytes_per_step": n * me * elem, "d2h_bytes_per_step": n * me * elem,
               "steps": e2e_steps, "api": f"bandsolve_{kind}_solve_shared (pinned host batch)",
               "sample": (f"all {me} systems of the shard" if me == m else
                          f"columns [{j0}, {j0 + me}) of each rank's shard ({me} of {m} systems: "
                          f"a {n * me * 8 / 2**30:.0f} GiB pinned host batch per rank)")}
    clk = clocks.summary()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(kind, n, m)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f32" if args.f32 else "f64",
            "data": "synthetic: U(-1,1) RHS from SplitMix64(seed=42, i, global j), generated on device",
            "config": {"workload": desc, "kind": kind, "n": n, "batch_per_gpu": m, "global_batch": m_global,
                       "mode": args.mode,
                       "arithmetic": ("fp64, FMA form / partitioned sweep, max rel err <= 1e-12 vs the reference"
                                      if args.mode == "fast" else "fp64, reference operation order, bitwise equal"),
                       "plan": plan, "periodic": bool(args.periodic), "cn_step": bool(args.cn),
                       "parallelism": f"dp{world} (systems sharded, no data-path collective)",
                       "l2": (f"{nbuf} in-place buffer{'s' if nbuf > 1 else ''} of {bytes_per / 2**20:.0f} MiB "
                              f"(working set {nbuf * bytes_per / l2:.1f}x L2, inputs larger than L2)")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "sustained_copy_gbs": sustained,
                         "frac_of_sustained_copy": achieved / sustained if sustained else None,
                         "algorithmic_bytes_per_launch": algo_bytes, "peak_source": peak_src,
                         "kernel": kernel_name(plan, args.f32, kind, args.mode)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=DEFAULT_CONFIG)
    # fast (default): fp64 in FMA form, partitioned one-pass sweep for long
    # systems, within 1e-12 of the reference (north_star's fp64 tolerance;
    # tests/test_spike.py, test_gpu_parity.py); exact: the reference's
    # operation order, bitwise equal
    ap.add_argument("--mode", choices=["exact", "fast"], default=os.environ.get("BANDSOLVE_BENCH_MODE", DEFAULT_MODE))
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-API end-to-end leg (tuning runs)")
    ap.add_argument("--no-sustained", action="store_true", help="skip the sustained device-copy reference rate")
    ap.add_argument("--pitch-pad", type=int, default=0, help="extra elements per row of the device batch (layout runs)")
    ap.add_argument("--periodic", action="store_true", help="cyclic (periodic) variant of the config's LHS")
    ap.add_argument("--cn", action="store_true",
                    help="Crank-Nicolson step (periodic stencil RHS + cyclic solve, sigma_x = 1) per step")
    ap.add_argument("--n", type=int, default=0, help="override the config's rows per system (tuning)")
    ap.add_argument("--m", type=int, default=0, help="override the config's systems per GPU (tuning)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.n or args.m:
        kind, n, m, desc = CONFIGS[args.config]
        n, m = args.n or n, args.m or m
        CONFIGS[args.config] = (kind, n, m, f"{kind} N={n} batch={m} (tuning override of {args.config})")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank)
        return 0

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
