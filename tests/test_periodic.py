"""Periodic (cyclic) wrap correction — SURVEY.md §8(f) rank 1, the direct
caller of the shared sweep (reference periodic.cpp, capi.cpp:229-298).

CPU tests pin the oracle restatement against the reference library and its
golden vectors and check the product library's host-side preparation
(statuses, modified bands) — no GPU needed. GPU tests run the B200 solve and
correction through the C ABI against the oracle, bit for bit.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle.oracle import OracleError, bitwise_equal, per_system_max_rel
from paper_1909_04539_b200 import bandsolve as bs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "periodic_cases.npz")


def golden_cases():
    z = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in z.files})
    return [(nm, {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(nm + "/")}) for nm in names]


def oracle_solve(oracle, bands, x, correct_only=False):
    n = x.shape[0]
    if len(bands) == 3:
        f = oracle.periodic_tri_prepare(*bands, n)
        return oracle.periodic_tri_solve(f, x.copy(), correct_only)
    f = oracle.periodic_pent_prepare(*bands, n)
    return oracle.periodic_pent_solve(f, x.copy(), correct_only)


def set_plan(lib, plan):
    """(PLAN, warps/group width, tail rows) override for the sweep under the correction."""
    lib.tune_reset()
    if not plan:
        return
    lib.tune("PLAN", plan[0])
    keys = ("SWG", "STAIL") if plan[0] == "stream" else ("PWARPS", "PTAIL")
    for k, v in zip(keys, plan[1:]):
        lib.tune(k, v)


def make(lib, bands, n):
    return bs.PeriodicTri(lib, *bands, n) if len(bands) == 3 else bs.PeriodicPent(lib, *bands, n)


# ---- oracle pinned to the reference ------------------------------------------------
@pytest.mark.parametrize("name,case", golden_cases())
def test_oracle_matches_golden(oracle, name, case):
    got = oracle_solve(oracle, tuple(case["bands"]), case["rhs"])
    assert bitwise_equal(got, case["x"]), name


def test_oracle_matches_live_reference(oracle, reflib):
    rng = np.random.default_rng(77)
    for n, m in [(3, 1), (6, 2), (17, 9), (128, 33)]:
        x = rng.uniform(-1, 1, (n, m))
        tri = (rng.uniform(-0.5, 0.5), rng.uniform(1.2, 2.0), rng.uniform(-0.5, 0.5))
        b = bs.Batch.from_array(reflib, x)
        bs.PeriodicTri(reflib, *tri, n).solve(b)
        assert bitwise_equal(b.array, oracle_solve(oracle, tri, x)), (n, m)
        if n >= 6:
            pent = (0.1, -0.6, 2.7, -0.4, 0.15)
            b = bs.Batch.from_array(reflib, x)
            bs.PeriodicPent(reflib, *pent, n).solve(b)
            assert bitwise_equal(b.array, oracle_solve(oracle, pent, x)), (n, m)
            # correction alone (bandsolve_periodic_pent_correct)
            b = bs.Batch.from_array(reflib, x)
            bs.PeriodicPent(reflib, *pent, n).correct(b)
            assert bitwise_equal(b.array, oracle_solve(oracle, pent, x, correct_only=True)), (n, m)


def test_oracle_rejects_like_reference(oracle):
    # test_capi.cpp:218-225, test_periodic.cpp:105-119, :220-223
    for args, st in [((1.0, 0.0, 1.0, 8), 4), ((-1.0, 1.0, 0.0, 3), 5), ((1.0, 2.0, 1.0, 2), 1),
                     ((float("nan"), 2.0, 1.0, 8), 1)]:
        with pytest.raises(OracleError) as e:
            oracle.periodic_tri_prepare(*args)
        assert e.value.status == st, args
    with pytest.raises(OracleError) as e:
        oracle.periodic_pent_prepare(0.25, -1.0, 2.5, -1.0, 0.25, 5)
    assert e.value.status == 1


# ---- product library, host side (no GPU) ---------------------------------------------
def test_create_statuses_match_reference(lib, reflib):
    cases = [("tri", (1.0, 0.0, 1.0, 8)), ("tri", (-1.0, 1.0, 0.0, 3)), ("tri", (1.0, 2.0, 1.0, 2)),
             ("tri", (float("inf"), 2.0, 1.0, 8)), ("pent", (0.25, -1.0, 2.5, -1.0, 0.25, 5)),
             ("pent", (0.0, 0.0, 0.0, 0.0, 0.0, 8)), ("tri", (-0.5, 2.0, -0.5, 16)),
             ("pent", (0.25, -1.0, 2.5, -1.0, 0.25, 16))]
    for kind, args in cases:
        sts = []
        for L in (lib, reflib):
            cls = bs.PeriodicTri if kind == "tri" else bs.PeriodicPent
            try:
                cls(L, *args)
                sts.append(0)
            except bs.BandsolveError as e:
                sts.append(e.status)
        assert sts[0] == sts[1], (kind, args, sts)


@pytest.mark.parametrize("name,case", golden_cases())
def test_modified_bands_match_reference(lib, name, case):
    bands = tuple(case["bands"])
    got = make(lib, bands, case["rhs"].shape[0]).modified_bands()
    for i, v in enumerate(got):
        assert bitwise_equal(v, case[f"mod{i}"]), (name, i)


def test_null_arguments(lib):
    assert lib.lib.bandsolve_periodic_tri_create(1.0, 3.0, 1.0, 8, None) == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_periodic_tri_solve(None, None) == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_periodic_pent_correct(None, None) == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_periodic_pent_modified_bands(None, None, None, None, None, None) == bs.ERR_BAD_ARG
    lib.lib.bandsolve_periodic_tri_destroy(None)
    lib.lib.bandsolve_periodic_pent_destroy(None)


# ---- GPU: B200 solve through the C ABI vs the oracle ------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,case", golden_cases())
def test_gpu_periodic_matches_golden(lib, cuda_device, name, case):
    bands = tuple(case["bands"])
    b = bs.Batch.from_array(lib, case["rhs"])
    make(lib, bands, case["rhs"].shape[0]).solve(b)
    assert bitwise_equal(b.array, case["x"]), name


@pytest.mark.gpu
@pytest.mark.parametrize("plan", [None, ("global",), ("stream", "64", "16"), ("persist", "1", "0")])
def test_gpu_periodic_device_bitwise(lib, oracle, cuda_device, plan):
    torch = cuda_device
    set_plan(lib, plan)
    rng = np.random.default_rng(5)
    try:
        for n, m in [(3, 1), (6, 7), (64, 33), (257, 130), (512, 200)]:
            x = rng.uniform(-1, 1, (n, m))
            for bands in [(-0.3, 1.9, -0.5), (0.2, -0.8, 3.1, -0.7, 0.1)]:
                if len(bands) == 5 and n < 6:
                    continue
                p = make(lib, bands, n)
                for ld in (m, m + (m % 2) + 2):
                    for correct_only in (False, True):
                        buf = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
                        buf[:, :m] = torch.from_numpy(x).cuda()
                        fn = p.correct_dev if correct_only else p.solve_dev
                        fn(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
                        torch.cuda.synchronize()
                        got = buf[:, :m].cpu().numpy()
                        want = oracle_solve(oracle, bands, x, correct_only)
                        assert bitwise_equal(got, want), (plan, n, m, ld, bands, correct_only)
    finally:
        set_plan(lib, None)


@pytest.mark.gpu
def test_gpu_periodic_cyclic_residual_and_properties(lib, cuda_device):
    n, m = 512, 4096
    rng = np.random.default_rng(11)
    rhs = rng.uniform(-1, 1, (n, m))
    # tri diffusion sigma = 1 (pde.cpp:62-65) and pent hyperdiffusion (pde.cpp:67-71), cyclic
    for bands in [(-1.0, 3.0, -1.0), (1.0, -4.0, 7.0, -4.0, 1.0)]:
        b = bs.Batch.from_array(lib, rhs)
        make(lib, bands, n).solve(b)
        full = [np.full(n, v) for v in bands]
        if len(bands) == 3:
            full[0][0] = 0.0
            full[2][-1] = 0.0
            res = lib.tri_residual(*full, b, bs.Batch.from_array(lib, rhs), cyclic=True)
        else:
            full[0][:2] = 0.0
            full[1][0] = 0.0
            full[3][-1] = 0.0
            full[4][-2:] = 0.0
            res = lib.pent_residual(*full, b, bs.Batch.from_array(lib, rhs), cyclic=True)
        assert res <= 1e-12, (bands, res)
    # zero RHS -> zero; constant RHS -> 1 / row sum (test_periodic.cpp:59-76)
    p = bs.PeriodicTri(lib, -0.5, 2.0, -0.5, 12)
    z = bs.Batch.from_array(lib, np.zeros((12, 4)))
    p.solve(z)
    assert np.all(z.array == 0.0)
    c = bs.Batch.from_array(lib, np.ones((12, 2)))
    p.solve(c)
    np.testing.assert_allclose(c.array, 1.0, rtol=1e-13)
    q = bs.PeriodicPent(lib, 0.25, -1.0, 2.5, -1.0, 0.25, 12)
    c = bs.Batch.from_array(lib, np.ones((12, 2)))
    q.solve(c)
    np.testing.assert_allclose(c.array, 1.0, rtol=1e-13)


@pytest.mark.gpu
def test_gpu_periodic_shape_mismatch(lib, cuda_device):
    p = bs.PeriodicTri(lib, -0.5, 2.0, -0.5, 16)
    b = bs.Batch(lib, 15, 2)
    with pytest.raises(bs.BandsolveError) as e:
        p.solve(b)
    assert e.value.status == bs.ERR_SHAPE_MISMATCH


@pytest.mark.gpu
@pytest.mark.parametrize("wg", [None, "64", "96", "128"])
def test_gpu_periodic_fused_fast_within_tolerance(lib, oracle, cuda_device, wg):
    """Fast mode fuses the correction into the sweep (y_0, y_1 from dot products
    of the forward outputs): within the 1e-12 fp64 tolerance of the reference."""
    torch = cuda_device
    set_plan(lib, ("stream", wg) if wg else None)
    lib.set_mode(bs.MODE_FAST)
    rng = np.random.default_rng(21)
    try:
        for n, m in [(6, 5), (33, 70), (256, 300), (512, 1000), (1024, 130)]:
            x = rng.uniform(-1, 1, (n, m))
            for bands in [(-1.0, 3.0, -1.0), (-0.3, 1.9, -0.5), (1.0, -4.0, 7.0, -4.0, 1.0),
                          (0.2, -0.8, 3.1, -0.7, 0.1)]:
                p = make(lib, bands, n)
                for ld in (m, m + (m % 2) + 2):
                    buf = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
                    buf[:, :m] = torch.from_numpy(x).cuda()
                    p.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
                    torch.cuda.synchronize()
                    got = buf[:, :m].cpu().numpy()
                    want = oracle_solve(oracle, bands, x)
                    assert per_system_max_rel(got, want) <= 1e-12, (wg, n, m, ld, bands)
    finally:
        lib.set_mode(bs.MODE_EXACT)
        set_plan(lib, None)


@pytest.mark.gpu
def test_gpu_fresh_handles_host_api_regression(lib, cuda_device):
    """Round-1 driver failure: the first host-API solve with a fresh handle read
    device constants (factor records, z vectors) whose pageable upload had not
    landed, because the staged solve runs on non-blocking streams. Every fresh
    handle's first solve must meet the reference's residual (periodic.cpp:131-214,
    pent_solver.cpp:223-273) -- 50 fresh periodic and plain handles in a row."""
    n, m = 512, 4096
    rng = np.random.default_rng(5)
    rhs = rng.uniform(-1, 1, (n, m))
    hyper = (1.0, -4.0, 7.0, -4.0, 1.0)
    full = [np.full(n, v) for v in hyper]
    full[0][:2] = 0.0
    full[1][0] = 0.0
    full[3][-1] = 0.0
    full[4][-2:] = 0.0
    ref = bs.Batch.from_array(lib, rhs)
    for k in range(50):
        b = bs.Batch.from_array(lib, rhs)
        bs.PeriodicPent(lib, *hyper, n).solve(b)
        res = lib.pent_residual(*full, b, ref, cyclic=True)
        assert res <= 1e-12, (k, "periodic", res)
        b = bs.Batch.from_array(lib, rhs)
        bs.PentFactor(lib, *full).solve(b)
        res = lib.pent_residual(*full, b, ref, cyclic=False)
        assert res <= 1e-12, (k, "plain", res)
