"""Crank-Nicolson stepping — SURVEY.md §8(f) rank 2: the reference's
bandsolve_bench_run driver (capi.cpp:369-411, pde.cpp run_benchmark) on the
GPU, and the device-level CN step (periodic explicit stencil + cyclic solve).

Parity anchor: tests/golden/cn_cases.npz, field dumps of the reference's own
driver (tests/golden/make_cn_golden.py); the oracle's restatement reproduces
them bit for bit (CPU test), and so must the B200 driver (GPU test).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle.oracle import bitwise_equal, per_system_max_rel
from paper_1909_04539_b200 import bandsolve as bs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cn_cases.npz")


def cases():
    z = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in z.files})
    out = []
    for nm in names:
        n, m, steps, dt, prob, var = z[nm + "/params"]
        fields = [z[f"{nm}/step{k}"] for k in range(1, int(steps) + 1)]
        out.append((nm, (int(n), int(m), int(steps), float(dt), int(prob), int(var)), fields))
    return out


@pytest.mark.parametrize("name,params,fields", cases())
def test_oracle_reproduces_reference_dumps(oracle, name, params, fields):
    n, m, steps, dt, prob, var = params
    traj = oracle.cn_trajectory(prob, n, m, steps, dt, var)
    for k in range(steps):
        assert bitwise_equal(traj[k], fields[k]), (name, k + 1)


def test_bench_run_checks_match_reference(lib, reflib, tmp_path):
    """Invalid configurations: same status from both libraries (pde.cpp:258-277,
    capi.cpp:374-401); these fail before any device work."""
    bad = [dict(n=2, m=4, steps=1, problem=0), dict(n=5, m=4, steps=1, problem=1),
           dict(n=16, m=4, steps=0, problem=0), dict(n=16, m=4, steps=1, problem=0, variant=2),
           dict(n=16, m=4, steps=1, problem=7), dict(n=16, m=4, steps=1, problem=0, variant=9),
           dict(n=16, m=0, steps=1, problem=0), dict(n=16, m=4, steps=1, problem=0, dump_every=1)]
    for kw in bad:
        sts = []
        for L in (lib, reflib):
            try:
                L.bench_run(**kw)
                sts.append(0)
            except bs.BandsolveError as e:
                sts.append(e.status)
        assert sts[0] == sts[1] == bs.ERR_BAD_ARG, (kw, sts)
    assert lib.lib.bandsolve_bench_run(None, None) == bs.ERR_BAD_ARG


def test_footprint_matches_reference(lib, reflib):
    for v in range(5):
        for n, m in [(2, 1), (512, 65536), (1024, 1 << 24)]:
            assert lib.footprint(v, n, m) == reflib.footprint(v, n, m), (v, n, m)
    with pytest.raises(bs.BandsolveError):
        lib.footprint(0, 1, 1)
    # either out-parameter may be NULL (reference capi.cpp:320-323): the same
    # statuses and the same reduction as the reference
    import ctypes as C
    for L in (lib, reflib):
        red = C.c_double(-1.0)
        assert L.lib.bandsolve_footprint(3, 512, 4096, None, C.byref(red)) == bs.OK
        assert red.value == reflib.footprint(3, 512, 4096)[1]
        assert L.lib.bandsolve_footprint(3, 512, 4096, None, None) == bs.OK
        assert L.lib.bandsolve_footprint(9, 512, 4096, None, None) == bs.ERR_BAD_ARG
        assert L.lib.bandsolve_footprint(3, 1, 4096, None, None) == bs.ERR_BAD_ARG


@pytest.mark.gpu
@pytest.mark.parametrize("name,params,fields", cases())
def test_gpu_bench_run_dumps_bitwise(lib, cuda_device, tmp_path, name, params, fields):
    n, m, steps, dt, prob, var = params
    prefix = str(tmp_path / name)
    r = lib.bench_run(n, m, steps, prob, var, dt, dump_every=1, dump_prefix=prefix)
    assert r.steps == steps and r.per_step_mean_s > 0 and r.wall_s >= r.per_step_mean_s
    assert r.elements == lib.footprint({(0, 0): 1, (0, 1): 0, (1, 0): 3, (1, 1): 2, (1, 2): 4}[(prob, var)], n, m)[0]
    for k in range(steps):
        got = bs.read_ibat(f"{prefix}_step{k + 1}.ibat")
        assert bitwise_equal(got, fields[k]), (name, k + 1)


@pytest.mark.gpu
def test_gpu_cn_step_dev(lib, oracle, cuda_device):
    torch = cuda_device
    rng = np.random.default_rng(8)
    for prob, n, m in [(0, 3, 5), (0, 257, 300), (1, 6, 7), (1, 512, 1000)]:
        s = oracle.cn_sigma(prob, n, 0.0) * 0.37
        u = rng.uniform(-1, 1, (n, m))
        if prob == 0:
            h = bs.PeriodicTri(lib, -s, 1 + 2 * s, -s, n)
            f = oracle.periodic_tri_prepare(-s, 1 + 2 * s, -s, n)
            want = oracle.periodic_tri_solve(f, oracle.cn_rhs(0, s, u))
        else:
            h = bs.PeriodicPent(lib, s, -4 * s, 1 + 6 * s, -4 * s, s, n)
            f = oracle.periodic_pent_prepare(s, -4 * s, 1 + 6 * s, -4 * s, s, n)
            want = oracle.periodic_pent_solve(f, oracle.cn_rhs(1, s, u))
        for ld in (m, m + (m % 2) + 2):
            du = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
            du[:, :m] = torch.from_numpy(u).cuda()
            do = torch.zeros_like(du)
            h.cn_step_dev(s, du.data_ptr(), do.data_ptr(), n, m, ld=ld,
                          stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            assert bitwise_equal(do[:, :m].cpu().numpy(), want), (prob, n, m, ld)
            assert bitwise_equal(du[:, :m].cpu().numpy(), u)  # input untouched
        # fast mode: fused correction, within the fp64 tolerance
        lib.set_mode(bs.MODE_FAST)
        try:
            du = torch.from_numpy(u).cuda()
            do = torch.zeros_like(du)
            h.cn_step_dev(s, du.data_ptr(), do.data_ptr(), n, m, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            assert per_system_max_rel(do.cpu().numpy(), want) <= 1e-12, (prob, n, m)
        finally:
            lib.set_mode(bs.MODE_EXACT)
    # aliasing is rejected
    h = bs.PeriodicTri(lib, -0.5, 2.0, -0.5, 8)
    du = torch.zeros((8, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(bs.BandsolveError):
        h.cn_step_dev(0.5, du.data_ptr(), du.data_ptr(), 8, 4)


def set_stream_plan(lib, plan):
    lib.tune_reset()
    if plan:
        lib.tune("PLAN", "stream")
        for k, v in zip(("SWG", "STAIL", "SKB", "SV", "SKR"), plan):
            lib.tune(k, v)


@pytest.mark.gpu
@pytest.mark.parametrize("plan", [None, ("64", "0"), ("64", "16", "4", "2"), ("96", "40", "3", "1"),
                                  ("32", "100000"), ("128", "33", "2", "2", "0"), ("64", "0", "4", "1", "0")])
def test_gpu_cn_fused_over_plans(lib, oracle, cuda_device, plan):
    """The stencil window crosses ring chunks, the head/tail boundary, partial
    tail chunks and the wrap rows: every split must give the reference's
    bits (exact) / stay within 1e-12 (fast, fused correction)."""
    torch = cuda_device
    set_stream_plan(lib, plan)
    rng = np.random.default_rng(31)
    try:
        for prob, n, m in [(0, 3, 70), (0, 37, 130), (0, 512, 200), (1, 6, 65), (1, 50, 129), (1, 512, 300)]:
            s = 0.61
            u = rng.uniform(-1, 1, (n, m))
            if prob == 0:
                h = bs.PeriodicTri(lib, -s, 1 + 2 * s, -s, n)
                want = oracle.periodic_tri_solve(oracle.periodic_tri_prepare(-s, 1 + 2 * s, -s, n),
                                                 oracle.cn_rhs(0, s, u))
            else:
                h = bs.PeriodicPent(lib, s, -4 * s, 1 + 6 * s, -4 * s, s, n)
                want = oracle.periodic_pent_solve(
                    oracle.periodic_pent_prepare(s, -4 * s, 1 + 6 * s, -4 * s, s, n), oracle.cn_rhs(1, s, u))
            for mode in (bs.MODE_EXACT, bs.MODE_FAST):
                lib.set_mode(mode)
                du = torch.from_numpy(u).cuda()
                do = torch.zeros_like(du)
                h.cn_step_dev(s, du.data_ptr(), do.data_ptr(), n, m, stream=torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                got = do.cpu().numpy()
                if mode == bs.MODE_EXACT:
                    assert bitwise_equal(got, want), (plan, prob, n, m)
                else:
                    assert per_system_max_rel(got, want) <= 1e-12, (plan, prob, n, m)
    finally:
        lib.set_mode(bs.MODE_EXACT)
        set_stream_plan(lib, None)
