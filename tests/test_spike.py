"""One-pass partitioned sweep for many long systems (csrc/sweep_spike.cuh).

Fast mode promises the reference's answer within a per-system max-norm
relative error of 1e-12; the one-pass kernel reorders the
arithmetic exactly like the two-launch partitioned path (block sweeps, a
dense interface solve, the left-coupling update), so it is held to the same
bound against the oracle: K = 4 and 8 blocks, ragged batch widths (TMA
zero-fill + masked stores), padded pitches, every band structure, and a
column sample at configs[4] scale (pent N = 1024). The tuning key SPIKE=1
forces the kernel below its many-systems threshold; =0 disables it.
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
    yield
    lib.set_mode(bs.MODE_EXACT)


def _dev_solve(lib, torch, factor, rhs, ld=None):
    n, m = rhs.shape
    ld = m if ld is None else ld
    buf = torch.full((n, ld), float("nan"), dtype=torch.float64, device="cuda")
    buf[:, :m] = torch.from_numpy(rhs).cuda()
    before = lib.kernel_launches()
    factor.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    launches = lib.kernel_launches() - before
    out = buf.cpu().numpy()
    if ld > m:
        assert np.all(np.isnan(out[:, m:]))
    return out[:, :m], launches


@pytest.mark.parametrize("n", [320, 512, 768, 1024, 1536, 2048, 4096])
def test_spike_within_tolerance(lib, oracle, cuda_device, n):
    """K <= 8 blocks in one CTA; K = 16 / 32 blocks across a cluster of
    2 / 4 CTAs (interface values through distributed shared memory)."""
    torch = cuda_device
    lib.tune("SPIKE", "1")
    rng = np.random.default_rng(n)
    K = {320: 4, 512: 4, 768: 8, 1024: 8, 1536: 16, 2048: 16, 4096: 32}[n]
    for m, ld in [(38, 40), (64, 64), (300, 302)]:
        rhs = rng.uniform(-1, 1, (n, m))
        cases = [("tri", bs.TriFactor, _random_tri(rng, n)), ("diff", bs.TriFactor, bs.diffusion_bands(1.0, n)),
                 ("pent", bs.PentFactor, _random_pent(rng, n)), ("hyper", bs.PentFactor, bs.hyper_bands(1.0, n))]
        for name, cls, bands in cases:
            pent = cls is bs.PentFactor
            assert lib.describe_plan(1 if pent else 0, n, m, ld).startswith(f"spike K={K}")
            want = (oracle.pent_solve(oracle.pent_prefactor(*bands), rhs.copy()) if pent
                    else oracle.tri_solve(oracle.tri_prefactor(*bands), rhs.copy()))
            got, launches = _dev_solve(lib, torch, cls(lib, *bands), rhs, ld)
            assert launches == 1, (name, n, m)
            assert per_system_max_rel(got, want) <= TOL_F64, (name, n, m, ld)


def test_spike_planner_threshold(lib, cuda_device):
    """Without the override the kernel is taken for many systems only, in
    fast mode only, and never for odd pitches (TMA 16-byte rule)."""
    sms = cuda_device.cuda.get_device_properties(0).multi_processor_count
    assert lib.describe_plan(1, 1024, 1 << 20).startswith("spike K=8")
    assert lib.describe_plan(0, 512, 1 << 20).startswith("spike K=4")
    assert lib.describe_plan(0, 2048, 1 << 20).startswith("spike K=16")
    assert lib.describe_plan(1, 4096, 1 << 20).startswith("spike K=32")
    assert not lib.describe_plan(1, 1024, sms * 32 - 2).startswith("spike")
    assert lib.describe_plan(0, 256, 4096).startswith("spike K=8")  # configs[0]: few systems, short blocks
    assert not lib.describe_plan(1, 1024, (1 << 20) - 1, 1 << 20).startswith("spike")  # odd batch width
    assert not lib.describe_plan(1, 1024, 1 << 20, (1 << 20) + 1).startswith("spike")
    assert not lib.describe_plan(1, 1000, 1 << 20).startswith("spike")  # 1000 / 4 is not a chunk multiple
    lib.tune("SPIKE", "0")
    assert not lib.describe_plan(1, 1024, 1 << 20).startswith("spike")
    lib.tune("SPIKE", None)
    lib.set_mode(bs.MODE_EXACT)
    assert not lib.describe_plan(1, 1024, 1 << 20).startswith("spike")


def test_spike_breakdown_falls_back(lib, oracle, cuda_device):
    """A block whose unpivoted elimination grows (tiny diagonal at a block
    start) is rejected by the plan; the sequential sweep answers instead."""
    torch = cuda_device
    lib.tune("SPIKE", "1")
    n, m = 512, 64
    rng = np.random.default_rng(5)
    sub, diag, sup = _random_tri(rng, n)
    sub[256], sup[255] = 1.0, 1.0
    diag[256] = 1e-14  # block 1 starts here: a near-zero pivot for the block factor
    diag[255] = 4.0
    rhs = rng.uniform(-1, 1, (n, m))
    want = oracle.tri_solve(oracle.tri_prefactor(sub, diag, sup), rhs.copy())
    got, _ = _dev_solve(lib, torch, bs.TriFactor(lib, sub, diag, sup), rhs)
    assert per_system_max_rel(got, want) <= TOL_F64


def test_spike_configs4_column_sample(lib, oracle, cuda_device):
    """configs[4] shape (pent N = 1024, hyperdiffusion sigma_x = 1) through the
    planner's own choice at 2^20 systems: residual over the whole batch and
    a column sample against the oracle, both within the fast-mode bound."""
    torch = cuda_device
    n, m = 1024, 1 << 20
    assert lib.describe_plan(1, n, m).startswith("spike K=8")
    bands = bs.hyper_bands(1.0, n)
    stream = torch.cuda.current_stream().cuda_stream
    x = torch.empty((n, m), dtype=torch.float64, device="cuda")
    lib.fill_rhs_dev(x.data_ptr(), n, m, m, 42, 0, stream)
    rhs = x.clone()
    fac = bs.PentFactor(lib, *bands)
    fac.solve_dev(x.data_ptr(), n, m, ld=m, stream=stream)
    res = lib.pent_residual_dev(*bands, x.data_ptr(), rhs.data_ptr(), m, m, stream=stream)
    assert res <= 1e-12
    cols = np.random.default_rng(3).choice(m, 512, replace=False)
    cols.sort()
    idx = torch.from_numpy(cols).cuda()
    got = x.index_select(1, idx).cpu().numpy()
    b = rhs.index_select(1, idx).cpu().numpy()
    want = oracle.pent_solve(oracle.pent_prefactor(*bands), b.copy())
    assert per_system_max_rel(got, want) <= TOL_F64


@pytest.mark.parametrize("n", [320, 512, 1024, 2048, 4096])
def test_spike_periodic_fused_within_tolerance(lib, oracle, cuda_device, n):
    """Cyclic systems: the Woodbury correction rides in the spike kernel's
    backward sweep (its coefficients need x_0, x_1, x_{n-2}, x_{n-1}, which
    are interface unknowns) — one launch, within 1e-12 of the reference's
    periodic solve (periodic.cpp:57-95, :172-214)."""
    torch = cuda_device
    lib.tune("SPIKE", "1")
    rng = np.random.default_rng(n + 1)
    for m, ld in [(64, 64), (300, 302)]:
        x = rng.uniform(-1, 1, (n, m))
        for bands in [(-1.0, 3.0, -1.0), (-0.3, 1.9, -0.5), (1.0, -4.0, 7.0, -4.0, 1.0),
                      (0.2, -0.8, 3.1, -0.7, 0.1)]:
            p = bs.PeriodicTri(lib, *bands, n) if len(bands) == 3 else bs.PeriodicPent(lib, *bands, n)
            buf = torch.full((n, ld), float("nan"), dtype=torch.float64, device="cuda")
            buf[:, :m] = torch.from_numpy(x).cuda()
            before = lib.kernel_launches()
            p.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            assert lib.kernel_launches() - before == 1, (n, m, bands)
            out = buf.cpu().numpy()
            assert np.all(np.isnan(out[:, m:]))
            if len(bands) == 3:
                want = oracle.periodic_tri_solve(oracle.periodic_tri_prepare(*bands, n), x.copy())
            else:
                want = oracle.periodic_pent_solve(oracle.periodic_pent_prepare(*bands, n), x.copy())
            assert per_system_max_rel(out[:, :m], want) <= TOL_F64, (n, m, ld, bands)


@pytest.mark.parametrize("n", [320, 512, 1024, 4096])
def test_spike_cn_step_within_tolerance(lib, oracle, cuda_device, n):
    """Crank-Nicolson step u_new = A^-1 (B u) in one spike launch: the
    explicit periodic stencil (pde.cpp:73-114) is formed from the ring boxes
    plus halo rows across block edges and the wrap, then the partitioned
    sweep and the Woodbury correction. Within 1e-12 of the reference's
    assemble-then-solve; the old field is left untouched."""
    torch = cuda_device
    lib.tune("SPIKE", "1")
    rng = np.random.default_rng(n + 2)
    for prob in (0, 1):
        for m, ld in [(64, 64), (300, 302)]:
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
            assert per_system_max_rel(out[:, :m], want) <= TOL_F64, (prob, n, m, ld)
            assert np.array_equal(du[:, :m].cpu().numpy(), u)


@pytest.mark.parametrize("n", [256, 512, 1024, 2048, 4096])
def test_spike_fp32_within_tolerance(lib, oracle, cuda_device, n):
    """fp32 batches: the same plan rounded to float (records, R^-1, TMEM
    storage of up to 256 fp32 rows per lane), within the 1e-5 fp32 contract
    of the fp64 reference solution."""
    torch = cuda_device
    lib.tune("SPIKE", "1")
    rng = np.random.default_rng(n + 3)
    for m, ld in [(64, 64), (300, 304)]:
        rhs = rng.uniform(-1, 1, (n, m))
        for cls, bands in [(bs.TriFactor, bs.diffusion_bands(1.0, n)), (bs.TriFactor, _random_tri(rng, n)),
                           (bs.PentFactor, bs.hyper_bands(1.0, n)), (bs.PentFactor, _random_pent(rng, n))]:
            pent = cls is bs.PentFactor
            assert lib.describe_plan(1 if pent else 0, n, m, ld, True).startswith("spike"), (n, m)
            want = (oracle.pent_solve(oracle.pent_prefactor(*bands), rhs.copy()) if pent
                    else oracle.tri_solve(oracle.tri_prefactor(*bands), rhs.copy()))
            buf = torch.full((n, ld), float("nan"), dtype=torch.float32, device="cuda")
            buf[:, :m] = torch.from_numpy(rhs.astype(np.float32)).cuda()
            before = lib.kernel_launches()
            cls(lib, *bands).solve_dev(buf.data_ptr(), n, m, ld=ld, stream=torch.cuda.current_stream().cuda_stream,
                                       f32=True)
            torch.cuda.synchronize()
            assert lib.kernel_launches() - before == 1
            out = buf.cpu().numpy()
            assert np.all(np.isnan(out[:, m:]))
            assert per_system_max_rel(out[:, :m].astype(np.float64), want) <= 1e-5, (n, m, pent)


@pytest.mark.parametrize("n", [512, 1024, 2048])
def test_spike_decay_cutoffs(lib, oracle, cuda_device, n):
    """Pentadiagonal decay cut-offs (sweep_spike.cuh SpikePer::dp / df):
    strongly dominant bands (fast decay: most chunks skip the interface and
    coupling FMAs) and weakly dominant ones (slow decay: few or none skip)
    stay within 1e-12 of the reference, and the strongly dominant result is
    within 1e-15 of the same kernel with the cut-offs disabled (SPIKE_CUT=0)."""
    torch = cuda_device
    lib.tune("SPIKE", "1")
    rng = np.random.default_rng(7 * n)
    m = 96
    rhs = rng.uniform(-1, 1, (n, m))
    strong = (np.full(n, 0.1), np.full(n, -0.2), np.full(n, 4.0), np.full(n, -0.2), np.full(n, 0.1))
    weak = (np.full(n, 1.0), np.full(n, -4.0), np.full(n, 6.2), np.full(n, -4.0), np.full(n, 1.0))
    for name, bands in [("strong", strong), ("weak", weak), ("hyper", bs.hyper_bands(1.0, n))]:
        a, b, c, d, e = (np.array(v, dtype=np.float64) for v in bands)
        a[:2] = 0; b[0] = 0; d[-1] = 0; e[-2:] = 0
        bands = (a, b, c, d, e)
        want = oracle.pent_solve(oracle.pent_prefactor(*bands), rhs.copy())
        got, _ = _dev_solve(lib, torch, bs.PentFactor(lib, *bands), rhs)
        assert per_system_max_rel(got, want) <= TOL_F64, (name, n)
        lib.tune("SPIKE_CUT", "0")
        try:
            full, _ = _dev_solve(lib, torch, bs.PentFactor(lib, *bands), rhs)
        finally:
            lib.tune("SPIKE_CUT", None)
        assert per_system_max_rel(full, want) <= TOL_F64, (name, n)
        if name == "strong":
            assert per_system_max_rel(got, full) <= 1e-15, n
