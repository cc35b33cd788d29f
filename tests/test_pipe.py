"""Pipelined on-chip sequential sweep (csrc/sweep_pipe.cuh).

Every forward intermediate stays on chip (TMEM + shared memory) and each warp
interleaves the backward sweep of one group with the forward sweep of the
next in the same storage slots. In exact mode it must reproduce the
reference's bits (tri_solver.cpp:25-47, pent_solver.cpp:19-62) for every
shape it takes — one and several TMEM-only / TMEM + smem chunk counts, ragged
groups (masked stores), padded pitches, 2..4 compute warps — and stay within
1e-12 in fast mode. The tuning key PIPE=1 forces it below its many-systems
threshold; =0 disables it.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import bitwise_equal, per_system_max_rel
from paper_1909_04539_b200 import bandsolve as bs

pytestmark = pytest.mark.gpu


def _random_tri(rng, n):
    sub = rng.uniform(-1, 1, n); sub[0] = 0
    sup = rng.uniform(-1, 1, n); sup[-1] = 0
    diag = np.abs(sub) + np.abs(sup) + rng.uniform(0.5, 1.5, n)
    return sub, diag, sup


def _random_pent(rng, n):
    a = rng.uniform(-1, 1, n); a[:2] = 0
    b = rng.uniform(-1, 1, n); b[0] = 0
    d = rng.uniform(-1, 1, n); d[-1] = 0
    e = rng.uniform(-1, 1, n); e[-2:] = 0
    c = np.abs(a) + np.abs(b) + np.abs(d) + np.abs(e) + rng.uniform(0.5, 1.5, n)
    return a, b, c, d, e


def _dev_solve(lib, torch, factor, rhs, ld):
    n, m = rhs.shape
    buf = torch.full((n, ld), float("nan"), dtype=torch.float64, device="cuda")
    buf[:, :m] = torch.from_numpy(rhs).cuda()
    before = lib.kernel_launches()
    factor.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    out = buf.cpu().numpy()
    assert np.all(np.isnan(out[:, m:]))
    return out[:, :m], lib.kernel_launches() - before


@pytest.mark.parametrize("mode", [bs.MODE_EXACT, bs.MODE_FAST])
@pytest.mark.parametrize("n", [32, 48, 256, 272, 320, 512, 784, 1024, 1296, 2048, 4096])
def test_pipe_matches_oracle(lib, oracle, cuda_device, mode, n):
    torch = cuda_device
    lib.tune("PIPE", "1")
    lib.tune("SPIKE", "0")
    lib.tune("PARTITION", "0")
    lib.set_mode(mode)
    rng = np.random.default_rng(n + mode)
    try:
        for m, ld in [(2, 2), (64, 66), (330, 330), (1000, 1002)]:
            rhs = rng.uniform(-1, 1, (n, m))
            for name, cls, bands in [("tri", bs.TriFactor, _random_tri(rng, n)),
                                     ("diff", bs.TriFactor, bs.diffusion_bands(1.0, n)),
                                     ("pent", bs.PentFactor, _random_pent(rng, n)),
                                     ("hyper", bs.PentFactor, bs.hyper_bands(1.0, n))]:
                pent = cls is bs.PentFactor
                if pent and n > 3072:
                    continue  # the pentadiagonal records of 4096 rows exceed shared memory
                assert lib.describe_plan(1 if pent else 0, n, m, ld).startswith("pipe"), (n, m)
                want = (oracle.pent_solve(oracle.pent_prefactor(*bands), rhs.copy()) if pent
                        else oracle.tri_solve(oracle.tri_prefactor(*bands), rhs.copy()))
                got, launches = _dev_solve(lib, torch, cls(lib, *bands), rhs, ld)
                assert launches == 1
                if mode == bs.MODE_EXACT:
                    assert bitwise_equal(got, want), (name, n, m, ld)
                else:
                    assert per_system_max_rel(got, want) <= 1e-12, (name, n, m, ld)
    finally:
        lib.set_mode(bs.MODE_EXACT)


def test_pipe_planner(lib, cuda_device):
    """Taken in exact mode for many systems of n % 16 == 0, n <= 4096 (beyond
    512 rows with the cp.async-staged L2 tier: 3 warps + registers up to 1024
    rows, then 2 warps)."""
    assert lib.describe_plan(1, 512, 1 << 20).startswith("pipe")
    assert lib.describe_plan(0, 256, 1 << 20).startswith("pipe")
    assert "l2-rows=0" in lib.describe_plan(1, 512, 1 << 20)               # every row on chip
    s = lib.describe_plan(1, 1024, 1 << 21)                               # configs[4]'s shard
    assert s.startswith("pipe Wg=96") and "l2-rows=0" not in s and "reg-rows=64" in s, s  # the L2 tier
    assert lib.describe_plan(0, 2048, 1 << 20).startswith("pipe Wg=64")
    assert lib.describe_plan(0, 4096, 1 << 20).startswith("pipe Wg=64")
    assert not lib.describe_plan(1, 4096, 1 << 20).startswith("pipe")     # pent records > smem
    assert not lib.describe_plan(0, 4112, 1 << 20).startswith("pipe")     # > 4096 rows
    lib.tune("PIPE_MAX_N", "512")
    assert not lib.describe_plan(1, 528, 1 << 20).startswith("pipe")
    lib.tune("PIPE_MAX_N", None)
    assert not lib.describe_plan(1, 500, 1 << 20).startswith("pipe")      # not whole chunks
    assert not lib.describe_plan(1, 512, (1 << 20) - 1, 1 << 20).startswith("pipe")  # odd batch
    assert not lib.describe_plan(1, 512, 100).startswith("pipe")          # under one wave
    lib.tune("PIPE", "0")
    assert not lib.describe_plan(1, 512, 1 << 20).startswith("pipe")


@pytest.mark.parametrize("n", [32, 256, 320, 512, 1024, 2048])
def test_pipe_periodic_exact_bitwise(lib, oracle, cuda_device, n):
    """Exact periodic solves with the correction fused: a first backward pass
    over the on-chip intermediates finds y_0, y_1, y_{n-2}, y_{n-1}, the
    second recomputes y and stores x = y - w z in the reference's order
    (periodic.cpp:57-95, :172-214) — bitwise, one launch."""
    torch = cuda_device
    lib.tune("PIPE", "1")
    rng = np.random.default_rng(n + 7)
    for m, ld in [(64, 64), (330, 332)]:
        x = rng.uniform(-1, 1, (n, m))
        for bands in [(-1.0, 3.0, -1.0), (-0.3, 1.9, -0.5), (1.0, -4.0, 7.0, -4.0, 1.0), (0.2, -0.8, 3.1, -0.7, 0.1)]:
            p = bs.PeriodicTri(lib, *bands, n) if len(bands) == 3 else bs.PeriodicPent(lib, *bands, n)
            got, launches = _dev_solve(lib, torch, p, x, ld)
            assert launches == 1, (n, m, bands)
            if len(bands) == 3:
                want = oracle.periodic_tri_solve(oracle.periodic_tri_prepare(*bands, n), x.copy())
            else:
                want = oracle.periodic_pent_solve(oracle.periodic_pent_prepare(*bands, n), x.copy())
            assert bitwise_equal(got, want), (n, m, ld, bands)


@pytest.mark.parametrize("n", [32, 256, 512])
def test_pipe_cn_step_exact_bitwise(lib, oracle, cuda_device, n):
    """Crank-Nicolson step in one pipe launch: the explicit periodic stencil
    in the reference's operation order (pde.cpp:85 / :108, halo rows carried
    across chunks and the wrap), the sequential sweep and the fused exact
    correction — bitwise equal to assemble-then-solve; the old field is left
    untouched."""
    torch = cuda_device
    lib.tune("PIPE", "1")
    lib.tune("PIPE_CN", "1")
    rng = np.random.default_rng(n + 9)
    for prob in (0, 1):
        for m, ld in [(64, 64), (330, 332)]:
            s = 0.61
            u = rng.uniform(-1, 1, (n, m))
            if prob == 0:
                h = bs.PeriodicTri(lib, -s, 1 + 2 * s, -s, n)
                want = oracle.periodic_tri_solve(oracle.periodic_tri_prepare(-s, 1 + 2 * s, -s, n),
                                                 oracle.cn_rhs(0, s, u))
            else:
                h = bs.PeriodicPent(lib, s, -4 * s, 1 + 6 * s, -4 * s, s, n)
                want = oracle.periodic_pent_solve(oracle.periodic_pent_prepare(s, -4 * s, 1 + 6 * s, -4 * s, s, n),
                                                  oracle.cn_rhs(1, s, u))
            du = torch.full((n, ld), float("nan"), dtype=torch.float64, device="cuda")
            du[:, :m] = torch.from_numpy(u).cuda()
            do = torch.full_like(du, float("nan"))
            before = lib.kernel_launches()
            h.cn_step_dev(s, du.data_ptr(), do.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            assert lib.kernel_launches() - before == 1, (prob, n, m)
            out = do.cpu().numpy()
            assert np.all(np.isnan(out[:, m:]))
            assert bitwise_equal(out[:, :m], want), (prob, n, m, ld)
            assert np.array_equal(du[:, :m].cpu().numpy(), u)


@pytest.mark.parametrize("mode", [bs.MODE_EXACT, bs.MODE_FAST])
@pytest.mark.parametrize("n", [32, 256, 512, 1024, 2048])
def test_pipe_fp32_pairs(lib, oracle, cuda_device, mode, n):
    """fp32 batches through the pipelined kernel, two systems per lane
    (float2, packed FMUL2/FADD2/FFMA2): in exact mode the same bits as the
    scalar fp32 sequential sweep (the streaming kernel, PIPE=0), and within
    the 1e-5 fp32 contract of the fp64 reference solution in both modes."""
    torch = cuda_device
    lib.tune("SPIKE", "0")
    lib.set_mode(mode)
    rng = np.random.default_rng(n + 11 + mode)
    try:
        for m, ld in [(64, 64), (328, 332), (1000, 1000)]:
            rhs = rng.uniform(-1, 1, (n, m)).astype(np.float32)
            for cls, bands in [(bs.TriFactor, _random_tri(rng, n)), (bs.TriFactor, bs.diffusion_bands(1.0, n)),
                               (bs.PentFactor, _random_pent(rng, n)), (bs.PentFactor, bs.hyper_bands(1.0, n))]:
                pent = cls is bs.PentFactor
                fac = cls(lib, *bands)
                outs = []
                for force in ("1", "0"):
                    lib.tune("PIPE", force)
                    plan = lib.describe_plan(1 if pent else 0, n, m, ld, True)
                    assert plan.startswith("pipe") == (force == "1"), plan
                    if force == "1":
                        assert "fp32 pairs" in plan, plan
                    buf = torch.full((n, ld), float("nan"), dtype=torch.float32, device="cuda")
                    buf[:, :m] = torch.from_numpy(rhs).cuda()
                    before = lib.kernel_launches()
                    fac.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream,
                                  f32=True)
                    torch.cuda.synchronize()
                    if force == "1":
                        assert lib.kernel_launches() - before == 1
                    out = buf.cpu().numpy()
                    assert np.all(np.isnan(out[:, m:]))
                    outs.append(out[:, :m])
                if mode == bs.MODE_EXACT:
                    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32)), (n, m, ld, pent)
                want = (oracle.pent_solve(oracle.pent_prefactor(*bands), rhs.astype(np.float64))
                        if pent else oracle.tri_solve(oracle.tri_prefactor(*bands), rhs.astype(np.float64)))
                assert per_system_max_rel(outs[0].astype(np.float64), want) <= 1e-5, (n, m, pent)
    finally:
        lib.set_mode(bs.MODE_EXACT)
