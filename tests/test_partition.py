"""Partitioned (SPIKE) fast-mode path for few long systems (csrc/partition.cu).

Fast mode promises the reference's answer within a per-system max-norm
relative error of 1e-12; the partitioned path reorders the
arithmetic (block sweeps + a dense interface solve + spike update), so it is
held to that same bound against the oracle, over ragged block splits, padded
pitches and every band structure. The tuning key PARTITION=1 forces the path even
where the planner would not pick it; =0 disables it.
"""
from __future__ import annotations


import numpy as np
import pytest

from oracle.oracle import per_system_max_rel
from paper_1909_04539_b200 import bandsolve as bs

pytestmark = pytest.mark.gpu

TOL_F64 = 1e-12


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


@pytest.fixture(autouse=True)
def _fast_mode(lib):
    lib.set_mode(bs.MODE_FAST)
    lib.tune("PLAN", None)
    yield
    lib.set_mode(bs.MODE_EXACT)
    lib.tune("PARTITION", None)


def _dev_solve(torch, factor, rhs, ld=None):
    n, m = rhs.shape
    ld = m if ld is None else ld
    buf = torch.full((n, ld), float("nan"), dtype=torch.float64, device="cuda")
    buf[:, :m] = torch.from_numpy(rhs).cuda()
    factor.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    out = buf.cpu().numpy()
    if ld > m:
        assert np.all(np.isnan(out[:, m:]))
    return out[:, :m]


@pytest.mark.parametrize("forced", ["1", None])
def test_partition_within_tolerance(lib, oracle, cuda_device, forced):
    torch = cuda_device
    if forced:
        lib.tune("PARTITION", forced)
    rng = np.random.default_rng(77)
    for n, m in [(128, 5), (200, 33), (1000, 64), (1023, 257), (4096, 128), (4099, 96)]:
        rhs = rng.uniform(-1, 1, (n, m))
        tb = _random_tri(rng, n)
        want = oracle.tri_solve(oracle.tri_prefactor(*tb), rhs.copy())
        for ld in (m, m + 3):
            got = _dev_solve(torch, bs.TriFactor(lib, *tb), rhs, ld)
            assert per_system_max_rel(got, want) <= TOL_F64, ("tri", n, m, ld)
        db = bs.diffusion_bands(1.0, n)
        want = oracle.tri_solve(oracle.tri_prefactor(*db), rhs.copy())
        assert per_system_max_rel(_dev_solve(torch, bs.TriFactor(lib, *db), rhs), want) <= TOL_F64, ("diff", n)
        pb = _random_pent(rng, n)
        want = oracle.pent_solve(oracle.pent_prefactor(*pb), rhs.copy())
        for ld in (m, m + 1):
            got = _dev_solve(torch, bs.PentFactor(lib, *pb), rhs, ld)
            assert per_system_max_rel(got, want) <= TOL_F64, ("pent", n, m, ld)
        hb = bs.hyper_bands(1.0, n)
        want = oracle.pent_solve(oracle.pent_prefactor(*hb), rhs.copy())
        assert per_system_max_rel(_dev_solve(torch, bs.PentFactor(lib, *hb), rhs), want) <= TOL_F64, ("hyper", n)
        u = bs.UniformPentFactor(lib, 1.0, -4.0, 7.0, -4.0, 1.0, n)
        want = oracle.pent_solve(oracle.uniform_prefactor(1.0, -4.0, 7.0, -4.0, 1.0, n), rhs.copy())
        assert per_system_max_rel(_dev_solve(torch, u, rhs), want) <= TOL_F64, ("uniform", n)


def test_partition_long_systems_two_launches(lib, oracle, cuda_device):
    """Few long systems (an ADI axis: 4096-row systems) take the partitioned
    path: two launches (block forward sweeps; interface solve + block
    backward sweeps)."""
    torch = cuda_device
    n, m = 4096, 1024
    bands = bs.diffusion_bands(1.0, n)
    f = bs.TriFactor(lib, *bands)
    x = torch.empty((n, m), dtype=torch.float64, device="cuda")
    lib.fill_rhs_dev(x.data_ptr(), n, m, m, seed=42)
    rhs = x.clone()
    f.solve_dev(x.data_ptr(), n, m)  # warm (plan + upload)
    torch.cuda.synchronize()
    x.copy_(rhs)
    before = lib.kernel_launches()
    f.solve_dev(x.data_ptr(), n, m)
    torch.cuda.synchronize()
    assert lib.kernel_launches() - before == 2
    res = lib.tri_residual_dev(*bands, x.data_ptr(), rhs.data_ptr(), m, m)
    assert 0.0 <= res <= TOL_F64, res
    cols = np.arange(0, m, 17)
    want = oracle.tri_solve(oracle.tri_prefactor(*bands), rhs.cpu().numpy()[:, cols].copy())
    assert per_system_max_rel(x.cpu().numpy()[:, cols], want) <= TOL_F64


def test_partition_disabled_matches_sequential(lib, oracle, cuda_device):
    torch = cuda_device
    rng = np.random.default_rng(5)
    n, m = 512, 200
    pb = _random_pent(rng, n)
    rhs = rng.uniform(-1, 1, (n, m))
    f = bs.PentFactor(lib, *pb)
    lib.tune("PARTITION", "1")
    part = _dev_solve(torch, f, rhs)
    lib.tune("PARTITION", "0")
    seq = _dev_solve(torch, f, rhs)
    assert per_system_max_rel(part, seq) <= TOL_F64


@pytest.mark.parametrize("forced", ["1", None])
def test_partition_periodic_fused_within_tolerance(lib, oracle, cuda_device, forced):
    """The periodic (Woodbury) correction fused into the partitioned path's
    backward pass: within 1e-12 of the reference's periodic solve."""
    torch = cuda_device
    if forced:
        lib.tune("PARTITION", forced)
    rng = np.random.default_rng(31)
    # m a multiple of 128: every CTA solves one block (rows staged in shared memory)
    for n, m in [(130, 7), (1024, 130), (2050, 64), (4096, 33), (1024, 256), (4096, 128)]:
        x = rng.uniform(-1, 1, (n, m))
        for bands in [(-1.0, 3.0, -1.0), (-0.3, 1.9, -0.5), (1.0, -4.0, 7.0, -4.0, 1.0), (0.2, -0.8, 3.1, -0.7, 0.1)]:
            if len(bands) == 3:
                p = bs.PeriodicTri(lib, *bands, n)
                want = oracle.periodic_tri_solve(oracle.periodic_tri_prepare(*bands, n), x.copy(), False)
            else:
                p = bs.PeriodicPent(lib, *bands, n)
                want = oracle.periodic_pent_solve(oracle.periodic_pent_prepare(*bands, n), x.copy(), False)
            for ld in (m, m + 2):
                buf = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
                buf[:, :m] = torch.from_numpy(x).cuda()
                p.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                got = buf[:, :m].cpu().numpy()
                assert per_system_max_rel(got, want) <= TOL_F64, (n, m, ld, bands)


def test_partition_through_host_api(lib, oracle, cuda_device):
    """The reference-facing host call (pinned batch staged in column chunks)
    takes the partitioned path per chunk in fast mode; within 1e-12."""
    rng = np.random.default_rng(91)
    n, m = 2048, 700
    rhs = rng.uniform(-1, 1, (n, m))
    tb = _random_tri(rng, n)
    b = bs.Batch.from_array(lib, rhs)
    bs.TriFactor(lib, *tb).solve(b)
    want = oracle.tri_solve(oracle.tri_prefactor(*tb), rhs.copy())
    assert per_system_max_rel(b.array, want) <= TOL_F64
    pb = _random_pent(rng, n)
    b = bs.Batch.from_array(lib, rhs)
    bs.PentFactor(lib, *pb).solve(b)
    want = oracle.pent_solve(oracle.pent_prefactor(*pb), rhs.copy())
    assert per_system_max_rel(b.array, want) <= TOL_F64
    lib.tune("HOST_CHUNK_MIB", "1")  # many small chunks: m per chunk = 64
    try:
        # the planner must pick the partitioned path for a chunk's shape, and
        # every chunk must launch exactly its two partitioned passes
        assert lib.describe_plan(bs.KIND_PENT, n, 64).startswith("partition"), lib.describe_plan(bs.KIND_PENT, n, 64)
        chunks = -(-m // 64)
        b = bs.Batch.from_array(lib, rhs)
        f = bs.PentFactor(lib, *pb)
        before = lib.kernel_launches()
        f.solve(b)
        assert lib.kernel_launches() - before == 2 * chunks
        assert per_system_max_rel(b.array, want) <= TOL_F64
    finally:
        lib.tune("HOST_CHUNK_MIB", None)


def test_partition_rejects_growing_block_pivots(lib, oracle, cuda_device):
    """A block that is not a leading principal submatrix may meet a tiny pivot
    even when the sequential factor is well conditioned: a near-zero diagonal
    entry at a block start. The plan must be rejected (sequential
    sweep instead), so the answer stays within 1e-12 of the reference."""
    torch = cuda_device
    lib.tune("PARTITION", "1")
    rng = np.random.default_rng(17)
    n, m = 2048, 256
    sub = np.full(n, -1.0); sub[0] = 0
    sup = np.full(n, -1.0); sup[-1] = 0
    diag = np.full(n, 3.0)
    for s in range(n // 16, n, n // 16):  # every candidate block start of K <= 16
        diag[s] = 1e-14
    rhs = rng.uniform(-1, 1, (n, m))
    want = oracle.tri_solve(oracle.tri_prefactor(sub, diag, sup), rhs.copy())
    before = lib.kernel_launches()
    got = _dev_solve(torch, bs.TriFactor(lib, sub, diag, sup), rhs)
    assert per_system_max_rel(got, want) <= TOL_F64
    assert lib.kernel_launches() - before == 1  # the sequential sweep, not the 2 partitioned passes
