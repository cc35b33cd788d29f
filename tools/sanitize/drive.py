#!/usr/bin/env python
"""Small-shape driver that launches every kernel family of the library once
per configuration, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck). Each solve is checked against the oracle so a sanitizer run that
passes also computed the right answer. Usage: drive.py [family ...]."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from oracle.oracle import Oracle, per_system_max_rel  # noqa: E402
from paper_1909_04539_b200 import bandsolve as bs  # noqa: E402

lib = bs.load()
orc = Oracle()
stream = 0


def dev_solve(fac, rhs, ld):
    n, m = rhs.shape
    buf = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    buf[:, :m] = torch.from_numpy(rhs).cuda()
    torch.cuda.synchronize()
    fac.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=stream)
    torch.cuda.synchronize()
    return buf[:, :m].cpu().numpy()


def check(got, want, tol, what):
    err = per_system_max_rel(got, want)
    print(f"{what}: max rel err {err:.2e}", flush=True)
    if not err <= tol:
        raise SystemExit(f"{what}: error {err} > {tol}")


def sweep(plan_env, mode, shapes, tol):
    lib.tune_reset()
    for k, v in plan_env.items():
        lib.tune(k, v)
    lib.set_mode(mode)
    rng = np.random.default_rng(1)
    for n, m, ld in shapes:
        rhs = rng.uniform(-1, 1, (n, m))
        tb, pb = bs.diffusion_bands(1.0, n), bs.hyper_bands(1.0, n)
        plan = lib.describe_plan(1, n, m, ld)
        check(dev_solve(bs.TriFactor(lib, *tb), rhs, ld), orc.tri_solve(orc.tri_prefactor(*tb), rhs.copy()), tol,
              f"tri {plan_env} mode={mode} {n}x{m} ld={ld} [{lib.describe_plan(0, n, m, ld)[:40]}]")
        check(dev_solve(bs.PentFactor(lib, *pb), rhs, ld), orc.pent_solve(orc.pent_prefactor(*pb), rhs.copy()), tol,
              f"pent {plan_env} mode={mode} {n}x{m} ld={ld} [{plan[:40]}]")
    lib.tune_reset()
    lib.set_mode(bs.MODE_EXACT)


def fam_stream():  # TMEM tier + L2 spill + smem tail (exact and fast), V=2
    sweep({"PLAN": "stream", "SWG": "128"}, bs.MODE_EXACT, [(512, 300, 300), (640, 256, 258)], 0.0)
    sweep({"PLAN": "stream", "SWG": "96"}, bs.MODE_FAST, [(512, 300, 300)], 1e-12)
    sweep({"PLAN": "stream", "SV": "2"}, bs.MODE_EXACT, [(256, 520, 520)], 0.0)


def fam_other_plans():
    for p in ("persist", "smemW16", "global"):
        sweep({"PLAN": p}, bs.MODE_EXACT, [(300, 100, 100)], 0.0)


def fam_spike():  # single CTA (K = 4, 8) and clusters of 2 / 4 CTAs (K = 16, 32)
    sweep({"SPIKE": "1"}, bs.MODE_FAST, [(512, 300, 302), (1024, 64, 64), (2048, 64, 64), (4096, 32, 32)], 1e-12)


def fam_spike_variants():  # periodic and CN fused, fp32
    rng = np.random.default_rng(5)
    lib.tune_reset()
    lib.tune("SPIKE", "1")
    lib.set_mode(bs.MODE_FAST)
    n, m = 512, 64
    x = rng.uniform(-1, 1, (n, m))
    p = bs.PeriodicPent(lib, 1.0, -4.0, 7.0, -4.0, 1.0, n)
    check(dev_solve(p, x, m), orc.periodic_pent_solve(orc.periodic_pent_prepare(1.0, -4.0, 7.0, -4.0, 1.0, n),
                                                      x.copy()), 1e-12, "spike periodic pent")
    u = torch.from_numpy(x).cuda()
    out = torch.empty_like(u)
    p.cn_step_dev(0.61, u.data_ptr(), out.data_ptr(), n, m, stream=stream)
    torch.cuda.synchronize()
    b32 = torch.from_numpy(x.astype(np.float32)).cuda()
    bs.TriFactor(lib, *bs.diffusion_bands(1.0, 1024)).solve_dev(
        torch.from_numpy(rng.uniform(-1, 1, (1024, 64)).astype(np.float32)).cuda().data_ptr(), 1024, 64, ld=64,
        stream=stream, f32=True)
    torch.cuda.synchronize()
    del b32
    print("spike variants ok", flush=True)
    lib.tune_reset()
    lib.set_mode(bs.MODE_EXACT)


def fam_pipe():  # TMEM only, TMEM + registers + smem, L2 tier, periodic fused (exact)
    sweep({"PIPE": "1"}, bs.MODE_EXACT, [(256, 128, 128), (512, 200, 202)], 0.0)
    sweep({"PIPE": "1", "PIPE_MAX_N": "1024"}, bs.MODE_EXACT, [(1024, 64, 64)], 0.0)
    rng = np.random.default_rng(6)
    lib.tune_reset()
    lib.tune("PIPE", "1")
    n, m = 512, 64
    x = rng.uniform(-1, 1, (n, m))
    p = bs.PeriodicTri(lib, -1.0, 3.0, -1.0, n)
    check(dev_solve(p, x, m), orc.periodic_tri_solve(orc.periodic_tri_prepare(-1.0, 3.0, -1.0, n), x.copy()), 0.0,
          "pipe periodic tri (exact)")
    lib.tune_reset()


def fam_partition():
    sweep({"PARTITION": "1"}, bs.MODE_FAST, [(1024, 64, 64)], 1e-12)


def fam_periodic():
    rng = np.random.default_rng(2)
    for mode, env in ((bs.MODE_EXACT, {}), (bs.MODE_FAST, {}), (bs.MODE_FAST, {"SPIKE": "1"})):
        lib.tune_reset()
        for k, v in env.items():
            lib.tune(k, v)
        lib.set_mode(mode)
        for n, m in ((512, 128),):
            x = rng.uniform(-1, 1, (n, m))
            p = bs.PeriodicPent(lib, 1.0, -4.0, 7.0, -4.0, 1.0, n)
            got = dev_solve(p, x, m)
            want = orc.periodic_pent_solve(orc.periodic_pent_prepare(1.0, -4.0, 7.0, -4.0, 1.0, n), x.copy())
            check(got, want, 0.0 if mode == bs.MODE_EXACT else 1e-12, f"periodic pent mode={mode} {env}")
    lib.tune_reset()
    lib.set_mode(bs.MODE_EXACT)


def fam_cn_adi():
    for mode in (bs.MODE_EXACT, bs.MODE_FAST):
        lib.set_mode(mode)
        n, m = 256, 128
        u = torch.rand((n, m), dtype=torch.float64, device="cuda")
        out = torch.empty_like(u)
        bs.PeriodicPent(lib, 1.0, -4.0, 7.0, -4.0, 1.0, n).cn_step_dev(1.0, u.data_ptr(), out.data_ptr(), n, m,
                                                                         stream=stream)
        a = bs.ADI(lib, 0, 1.0, 256, 256)
        f = torch.rand((256, 256), dtype=torch.float64, device="cuda")
        w = torch.empty_like(f)
        a.step_dev(f.data_ptr(), w.data_ptr(), stream=stream)
        torch.cuda.synchronize()
        print(f"cn/adi mode={mode} ok", flush=True)
    lib.set_mode(bs.MODE_EXACT)


def fam_host():  # pinned host batch through the 4-stream staging pipeline
    rng = np.random.default_rng(3)
    n, m = 512, 3000
    rhs = rng.uniform(-1, 1, (n, m))
    lib.tune("HOST_CHUNK_MIB", "1")
    b = bs.Batch.from_array(lib, rhs)
    pb = bs.hyper_bands(1.0, n)
    bs.PentFactor(lib, *pb).solve(b)
    check(b.array, orc.pent_solve(orc.pent_prefactor(*pb), rhs.copy()), 0.0, "host-API pent (chunked staging)")
    lib.tune_reset()


def fam_per_system():
    rng = np.random.default_rng(4)
    n, m = 128, 64
    a = rng.uniform(-1, 1, (n, m)); a[0] = 0
    c = rng.uniform(-1, 1, (n, m)); c[-1] = 0
    b = np.abs(a) + np.abs(c) + 1.0
    d = rng.uniform(-1, 1, (n, m))
    bb = [bs.Batch.from_array(lib, v) for v in (a, b, c, d)]
    lib.check(lib.lib.bandsolve_tri_solve_per_system(*[x.handle for x in bb]), "per-system")
    print("per-system ok", flush=True)


FAMILIES = {k[4:]: v for k, v in globals().items() if k.startswith("fam_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(FAMILIES)
    for name in names:
        FAMILIES[name]()
    print("DRIVE OK", flush=True)
