"""GPU parity: the sm_100a sweeps against the pinned CPU oracle and the
reference's golden outputs.

Bar (BASELINE.json north_star): exact mode is bitwise equal to the
reference; fast mode and fp32 are within the stated per-system max-norm
tolerance (fp64 1e-12, fp32 1e-5); residual ||Ax-b||/||b|| <= 1e-12 (fp64).
All solves go through the C ABI of libbandsolve_b200.so.
"""
from __future__ import annotations


import numpy as np
import pytest

from oracle.oracle import bitwise_equal, per_system_max_rel
from paper_1909_04539_b200 import bandsolve as bs

pytestmark = pytest.mark.gpu

TOL_F64 = 1e-12
TOL_F32 = 1e-5


@pytest.fixture(autouse=True)
def _exact_mode(lib):
    lib.set_mode(bs.MODE_EXACT)
    yield
    lib.set_mode(bs.MODE_EXACT)


# ---- helpers -------------------------------------------------------------------
def random_tri(rng, n):
    """oracles.cpp:9-17 distribution (strictly diagonally dominant)."""
    sub = rng.uniform(-1, 1, n); sub[0] = 0
    sup = rng.uniform(-1, 1, n); sup[-1] = 0
    diag = np.abs(sub) + np.abs(sup) + rng.uniform(0.5, 1.5, n)
    return sub, diag, sup


def random_pent(rng, n):
    """oracles.cpp:19-30 distribution."""
    a = rng.uniform(-1, 1, n); a[:2] = 0
    b = rng.uniform(-1, 1, n); b[0] = 0
    d = rng.uniform(-1, 1, n); d[-1] = 0
    e = rng.uniform(-1, 1, n); e[-2:] = 0
    c = np.abs(a) + np.abs(b) + np.abs(d) + np.abs(e) + rng.uniform(0.5, 1.5, n)
    return a, b, c, d, e


def dev_solve(torch, factor, rhs: np.ndarray, ld: int | None = None, f32: bool = False) -> np.ndarray:
    """Device-pointer entry point on a (n, ld) device array; returns (n, m)."""
    n, m = rhs.shape
    ld = m if ld is None else ld
    dt = torch.float32 if f32 else torch.float64
    buf = torch.full((n, ld), float("nan"), dtype=dt, device="cuda")
    buf[:, :m] = torch.from_numpy(rhs.astype(np.float32 if f32 else np.float64)).cuda()
    stream = torch.cuda.current_stream().cuda_stream
    factor.solve_dev(buf.data_ptr(), n, m, ld=ld, stream=stream, f32=f32)
    torch.cuda.synchronize()
    out = buf.cpu().numpy()
    if ld > m:  # padding columns are never touched
        assert np.all(np.isnan(out[:, m:]))
    return out[:, :m].astype(np.float64)


# ---- golden cases through the reference-facing host API ---------------------------
def test_golden_tri_host_api_bitwise(lib, golden, cuda_device):
    names = [c for c in golden.cases if c.startswith("tri_") or c.startswith("kat_tri")]
    before = lib.kernel_launches()
    for name in names:
        g = golden.case(name)
        f = bs.TriFactor(lib, g["sub"], g["diag"], g["sup"])
        b = bs.Batch.from_array(lib, g["rhs"])
        f.solve(b)
        assert bitwise_equal(b.array, g["x"]), name
        r = lib.tri_residual(g["sub"], g["diag"], g["sup"], b, bs.Batch.from_array(lib, g["rhs"]))
        assert r == g["residual"], name  # GPU residual in the reference's order
    assert lib.kernel_launches() > before  # the native kernels ran


def test_golden_pent_host_api_bitwise(lib, golden, cuda_device):
    names = [c for c in golden.cases if c.startswith("pent_") or c.startswith("kat_pent") or c.endswith("_shared")]
    for name in names:
        g = golden.case(name)
        f = bs.PentFactor(lib, g["a"], g["b"], g["c"], g["d"], g["e"])
        b = bs.Batch.from_array(lib, g["rhs"])
        f.solve(b)
        assert bitwise_equal(b.array, g["x"]), name
        r = lib.pent_residual(g["a"], g["b"], g["c"], g["d"], g["e"], b, bs.Batch.from_array(lib, g["rhs"]))
        assert r == g["residual"], name


def test_golden_uniform_host_api_bitwise(lib, golden, cuda_device):
    for name in [c for c in golden.cases if c.startswith("uniform_") and not c.endswith("_shared")]:
        g = golden.case(name)
        f = bs.UniformPentFactor(lib, *g["bands"], g["n"])
        b = bs.Batch.from_array(lib, g["rhs"])
        f.solve(b)
        assert bitwise_equal(b.array, g["x"]), name


def test_capi_residual_bounds(lib, cuda_device):
    # test_capi.cpp:49-83 and :102-141 through our ABI
    n = 8
    sub, diag, sup = bs.diffusion_bands(0.5, n)
    f = bs.TriFactor(lib, sub, diag, sup)
    rhs = np.sin(0.7 * np.arange(2 * n)).reshape(n, 2)
    x = bs.Batch.from_array(lib, rhs)
    f.solve(x)
    assert lib.tri_residual(sub, diag, sup, x, bs.Batch.from_array(lib, rhs)) <= 1e-12
    n = 12
    bands = bs.hyper_bands(0.25, n)
    pf = bs.PentFactor(lib, *bands)
    uf = bs.UniformPentFactor(lib, 0.25, -1.0, 2.5, -1.0, 0.25, n)
    rhs = np.cos(0.3 * np.arange(3 * n)).reshape(n, 3)
    xs, xu = bs.Batch.from_array(lib, rhs), bs.Batch.from_array(lib, rhs)
    pf.solve(xs)
    uf.solve(xu)
    assert bitwise_equal(xs.array, xu.array)
    assert lib.pent_residual(*bands, xs, bs.Batch.from_array(lib, rhs)) <= 1e-12


def test_cyclic_residual_matches_oracle(lib, oracle, cuda_device):
    rng = np.random.default_rng(9)
    n, m = 16, 5
    x, rhs = rng.uniform(-1, 1, (n, m)), rng.uniform(-1, 1, (n, m))
    sub, diag, sup = np.full(n, -0.3), np.full(n, 2.0), np.full(n, -0.7)
    got = lib.tri_residual(sub, diag, sup, bs.Batch.from_array(lib, x), bs.Batch.from_array(lib, rhs), cyclic=True)
    assert got == oracle.tri_residual(sub, diag, sup, x, rhs, cyclic=True)
    bands = [np.full(n, v) for v in (0.2, -0.9, 3.0, -0.8, 0.1)]
    got = lib.pent_residual(*bands, bs.Batch.from_array(lib, x), bs.Batch.from_array(lib, rhs), cyclic=True)
    assert got == oracle.pent_residual(*bands, x, rhs, cyclic=True)


# ---- device entry points over every plan and edge shape -----------------------------
SHAPES = [(2, 1), (3, 2), (5, 3), (31, 7), (32, 16), (33, 17), (64, 8), (65, 40), (100, 33), (257, 130),
          (512, 64), (1024, 48)]
# plan overrides: (BANDSOLVE_PLAN, BANDSOLVE_PWARPS, BANDSOLVE_PTAIL) for the persist/smem/global
# plans; "stream" takes (BANDSOLVE_SWG, BANDSOLVE_STAIL, BANDSOLVE_SKB, BANDSOLVE_SV, BANDSOLVE_SKR,
# BANDSOLVE_SRC, BANDSOLVE_SSEG, BANDSOLVE_TM8): group width, smem tail rows, ring slots, systems
# per lane, reload-ring slots, recomputed rows, recompute segment chunks, TMEM with 5..8 warps.
PLANS = [None, ("global",), ("smemW8",), ("smemW16",), ("smemW32",), ("persist", "1", "0"),
         ("persist", "2", "48"), ("persist", "3", "100000"),
         ("stream", "64", "0", "4", "2"), ("stream", "64", "16", "2", "1"), ("stream", "128", "40", "4", "2"),
         ("stream", "256", "100000", "4", "1"), ("stream", "192", "33", "2", "2"), ("stream", "96", "48", "3", "1"),
         ("stream", "32", "0", "4", "1"), ("stream", "96", "48", "4", "1", "4"),
         ("stream", "64", "8", "3", "2", "2"), ("stream", "96", "16", "4", "1", "4"), ("stream", "128", "40", "4", "1", "4"),
         ("stream", "32", "0", "2", "1", "2"),
         # recompute tier: segments re-streamed and re-run from checkpoints (bitwise like every plan)
         ("stream", "128", "32", "4", "1", "4", "64", "2"), ("stream", "64", "16", "2", "1", "2", "100000", "3"),
         ("stream", "96", "0", "3", "1", "0", "100000", "1"), ("stream", "32", "48", "4", "1", "4", "100000", "16"),
         ("stream", "256", "16", "4", "1", "4", "48", "4", "1"), ("stream", "192", "32", "3", "1", "2", "100000", "8", "1")]
STREAM_KEYS = ("SWG", "STAIL", "SKB", "SV", "SKR", "SRC", "SSEG", "TM8")


def set_plan(lib, plan):
    """Force a plan through the tuning table (bandsolve_tune_set)."""
    lib.tune_reset()
    if not plan:
        return
    if plan[0] == "stream":
        lib.tune("PLAN", "stream")
        for k, v in zip(STREAM_KEYS, plan[1:]):
            lib.tune(k, v)
    else:
        for k, v in zip(("PLAN", "PWARPS", "PTAIL"), plan):
            lib.tune(k, v)


@pytest.mark.parametrize("plan", PLANS)
def test_tri_device_plans_bitwise(lib, oracle, cuda_device, plan):
    torch = cuda_device
    rng = np.random.default_rng(100)
    set_plan(lib, plan)
    for n, m in SHAPES:
        bands = random_tri(rng, n)
        f = bs.TriFactor(lib, *bands)
        ref_f = oracle.tri_prefactor(*bands)
        rhs = rng.uniform(-1, 1, (n, m))
        want = oracle.tri_solve(ref_f, rhs.copy())
        for ld in (m, m + (m % 2) + 2):
            got = dev_solve(torch, f, rhs, ld=ld)
            assert bitwise_equal(got, want), (plan, n, m, ld)


@pytest.mark.parametrize("plan", PLANS)
def test_pent_device_plans_bitwise(lib, oracle, cuda_device, plan):
    torch = cuda_device
    rng = np.random.default_rng(200)
    set_plan(lib, plan)
    for n, m in SHAPES:
        if n < 5:
            continue
        bands = random_pent(rng, n)
        f = bs.PentFactor(lib, *bands)
        rhs = rng.uniform(-1, 1, (n, m))
        want = oracle.pent_solve(oracle.pent_prefactor(*bands), rhs.copy())
        for ld in (m, m + (m % 2) + 2):
            got = dev_solve(torch, f, rhs, ld=ld)
            assert bitwise_equal(got, want), (plan, n, m, ld)
        u = bs.UniformPentFactor(lib, 1.0, -4.0, 7.0, -4.0, 1.0, n)
        want_u = oracle.pent_solve(oracle.uniform_prefactor(1.0, -4.0, 7.0, -4.0, 1.0, n), rhs.copy())
        assert bitwise_equal(dev_solve(torch, u, rhs), want_u), (plan, n, m)


@pytest.mark.parametrize("plan", [None, ("global",), ("persist", "2", "0"), ("stream", "64", "48", "4", "2"),
                                  ("stream", "96", "48", "4", "1"), ("stream", "128", "32", "4", "1", "4", "100000", "4")])
def test_fast_mode_within_tolerance(lib, oracle, cuda_device, plan):
    torch = cuda_device
    rng = np.random.default_rng(300)
    set_plan(lib, plan)
    lib.set_mode(bs.MODE_FAST)
    for n, m in [(2, 3), (33, 17), (256, 64), (512, 96), (2048, 32)]:
        tb = random_tri(rng, n)
        rhs = rng.uniform(-1, 1, (n, m))
        want = oracle.tri_solve(oracle.tri_prefactor(*tb), rhs.copy())
        got = dev_solve(torch, bs.TriFactor(lib, *tb), rhs)
        assert per_system_max_rel(got, want) <= TOL_F64, (n, m)
        if n >= 5:
            pb = random_pent(rng, n)
            want = oracle.pent_solve(oracle.pent_prefactor(*pb), rhs.copy())
            got = dev_solve(torch, bs.PentFactor(lib, *pb), rhs)
            assert per_system_max_rel(got, want) <= TOL_F64, (n, m)
            hb = bs.hyper_bands(1.0, n)
            want = oracle.pent_solve(oracle.pent_prefactor(*hb), rhs.copy())
            got = dev_solve(torch, bs.PentFactor(lib, *hb), rhs)
            assert per_system_max_rel(got, want) <= TOL_F64, (n, m)


@pytest.mark.parametrize("mode", [bs.MODE_EXACT, bs.MODE_FAST])
def test_f32_within_tolerance(lib, oracle, cuda_device, mode):
    torch = cuda_device
    lib.set_mode(mode)
    rng = np.random.default_rng(400)
    for n, m in [(64, 64), (256, 100), (1024, 256), (4096, 64)]:
        db = bs.diffusion_bands(1.0, n)
        rhs = rng.uniform(-1, 1, (n, m)).astype(np.float32).astype(np.float64)
        want = oracle.tri_solve(oracle.tri_prefactor(*db), rhs.copy())
        got = dev_solve(torch, bs.TriFactor(lib, *db), rhs, f32=True)
        assert per_system_max_rel(got, want) <= TOL_F32, (n, m)
        hb = bs.hyper_bands(1.0, n)
        want = oracle.pent_solve(oracle.pent_prefactor(*hb), rhs.copy())
        got = dev_solve(torch, bs.PentFactor(lib, *hb), rhs, f32=True)
        assert per_system_max_rel(got, want) <= TOL_F32, (n, m)


# ---- reference behaviours --------------------------------------------------------------
def test_identity_lhs_leaves_batch_unchanged(lib, cuda_device):
    # test_tri_solver.cpp:13-20, test_pent_solver.cpp:22-29, :179-187
    rng = np.random.default_rng(1)
    rhs = rng.uniform(-1, 1, (9, 4))
    for f in (bs.TriFactor(lib, np.zeros(9), np.ones(9), np.zeros(9)),
              bs.PentFactor(lib, *[np.zeros(9)] * 2, np.ones(9), *[np.zeros(9)] * 2),
              bs.UniformPentFactor(lib, 0, 0, 1, 0, 0, 9)):
        b = bs.Batch.from_array(lib, rhs)
        f.solve(b)
        assert bitwise_equal(b.array, rhs)


def test_repeat_solve_purity(lib, cuda_device):
    # test_tri_solver.cpp:133-146
    rng = np.random.default_rng(31)
    f = bs.TriFactor(lib, *random_tri(rng, 20))
    first = rng.uniform(-1, 1, (20, 4))
    b1, b2, other = bs.Batch.from_array(lib, first), bs.Batch.from_array(lib, first), \
        bs.Batch.from_array(lib, rng.uniform(-1, 1, (20, 4)))
    f.solve(b1)
    f.solve(other)
    f.solve(b2)
    assert bitwise_equal(b1.array, b2.array)


def test_device_shape_mismatch_and_empty(lib, cuda_device):
    torch = cuda_device
    f = bs.TriFactor(lib, *bs.diffusion_bands(0.5, 8))
    buf = torch.zeros((9, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(bs.BandsolveError) as e:
        f.solve_dev(buf.data_ptr(), 9, 4)
    assert e.value.status == bs.ERR_SHAPE_MISMATCH
    f.solve_dev(buf.data_ptr(), 8, 0)  # m = 0 is a no-op


def test_shard_invariance(lib, oracle, cuda_device):
    """Columns are partition independent (parallel.hpp:20-23): solving
    contiguous shards in place gives the full solve bit for bit (the
    multi-GPU split of bench.py, emulated on one device)."""
    torch = cuda_device
    n, m = 512, 6000
    f = bs.PentFactor(lib, *bs.hyper_bands(1.0, n))
    full = torch.empty((n, m), dtype=torch.float64, device="cuda")
    lib.fill_rhs_dev(full.data_ptr(), n, m, m, seed=42)
    sharded = full.clone()
    f.solve_dev(full.data_ptr(), n, m)
    bounds = [0, 1500, 3002, 4498, m]  # shards share the pitch m; even offsets keep 16-byte alignment
    for j0, j1 in zip(bounds[:-1], bounds[1:]):
        f.solve_dev(sharded.data_ptr() + 8 * j0, n, j1 - j0, ld=m)
    torch.cuda.synchronize()
    assert torch.equal(full.view(torch.int64), sharded.view(torch.int64))


# ---- configs at full size ----------------------------------------------------------------
def _check_config(lib, oracle, torch, kind, n, m, bands, sample_cols=256):
    f = bs.TriFactor(lib, *bands) if kind == "tri" else bs.PentFactor(lib, *bands)
    x = torch.empty((n, m), dtype=torch.float64, device="cuda")
    lib.fill_rhs_dev(x.data_ptr(), n, m, m, seed=42)
    rhs = x.clone()
    f.solve_dev(x.data_ptr(), n, m)
    torch.cuda.synchronize()
    if kind == "tri":
        res = lib.tri_residual_dev(*bands, x.data_ptr(), rhs.data_ptr(), m, m)
    else:
        res = lib.pent_residual_dev(*bands, x.data_ptr(), rhs.data_ptr(), m, m)
    assert 0.0 <= res <= TOL_F64, res
    # bitwise vs the oracle on a column sample (columns are independent)
    cols = np.unique(np.concatenate([np.arange(min(64, m)), np.linspace(0, m - 1, sample_cols).astype(int)]))
    sub_rhs = rhs[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    sub_x = x[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    ref_f = oracle.tri_prefactor(*bands) if kind == "tri" else oracle.pent_prefactor(*bands)
    want = oracle.tri_solve(ref_f, sub_rhs.copy()) if kind == "tri" else oracle.pent_solve(ref_f, sub_rhs.copy())
    assert bitwise_equal(sub_x, want)
    assert bitwise_equal(sub_rhs, oracle.rhs(42, n, m)[:, cols])  # device generator == host generator


def test_config1_tri_n256_m4096(lib, oracle, cuda_device):
    _check_config(lib, oracle, cuda_device, "tri", 256, 4096, bs.diffusion_bands(1.0, 256), sample_cols=4096)


def test_config2_pent_n512_m65536(lib, oracle, cuda_device):
    _check_config(lib, oracle, cuda_device, "pent", 512, 65536, bs.hyper_bands(1.0, 512))
    rng = np.random.default_rng(2)
    _check_config(lib, oracle, cuda_device, "pent", 512, 65536, random_pent(rng, 512))


@pytest.mark.parametrize("n", [64, 512, 4096])
def test_config3_tri_batch_2p20(lib, oracle, cuda_device, n):
    m = 1 << 20 if n <= 512 else 1 << 18  # N=4096 x 2^18 keeps the test under 10 GiB
    _check_config(lib, oracle, cuda_device, "tri", n, m, bs.diffusion_bands(1.0, n), sample_cols=64)


def test_pent_n512_batch_2p20(lib, oracle, cuda_device):
    _check_config(lib, oracle, cuda_device, "pent", 512, 1 << 20, bs.hyper_bands(1.0, 512), sample_cols=64)


def test_config5_pent_n1024_batch_2p24(lib, oracle, cuda_device):
    """configs[4] at its full single-GPU size: pent N=1024, 2^24 systems
    (128 GiB in place, the bench's default workload). Exact mode bitwise and
    fast mode <= 1e-12 against the oracle on a column sample spread over the
    whole batch (pent_solver.cpp:15-81), plus the sample's residual."""
    torch = cuda_device
    free, _ = torch.cuda.mem_get_info()
    n, m = 1024, 1 << 24
    if free < n * m * 8 + (4 << 30):
        pytest.skip(f"needs {n * m * 8 / 2**30:.0f} GiB of device memory, {free / 2**30:.0f} GiB free")
    bands = bs.hyper_bands(1.0, n)
    f = bs.PentFactor(lib, *bands)
    ref_f = oracle.pent_prefactor(*bands)
    rng = np.random.default_rng(5)
    cols = np.unique(np.concatenate([np.arange(64), np.arange(m - 64, m), rng.integers(0, m, 128)]))
    rhs = np.concatenate([oracle.rhs(42, n, 1, j_offset=int(c)) for c in cols], axis=1)
    want = oracle.pent_solve(ref_f, rhs.copy())
    x = torch.empty((n, m), dtype=torch.float64, device="cuda")
    idx = torch.from_numpy(cols).cuda()
    try:
        for mode in (bs.MODE_EXACT, bs.MODE_FAST):
            lib.set_mode(mode)
            lib.fill_rhs_dev(x.data_ptr(), n, m, m, seed=42)
            f.solve_dev(x.data_ptr(), n, m)
            torch.cuda.synchronize()
            got = x[:, idx].cpu().numpy()
            if mode == bs.MODE_EXACT:
                assert bitwise_equal(got, want)
            else:
                assert per_system_max_rel(got, want) <= TOL_F64
            sx, sr = bs.Batch.from_array(lib, got), bs.Batch.from_array(lib, rhs)
            assert lib.pent_residual(*bands, sx, sr) <= TOL_F64
    finally:
        del x
        torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", [bs.MODE_EXACT, bs.MODE_FAST])
@pytest.mark.parametrize("n", [64, 512, 1024, 4096])
def test_config3_tri_f32_batch_2p20(lib, oracle, cuda_device, mode, n):
    """configs[2] in fp32 at its full batch (2^20 systems; N = 4096 at 2^18):
    the fp32 plans (system pairs per lane) within north_star's fp32
    tolerance of the reference solving the same fp32-rounded right-hand
    sides, on a column sample spread over the batch, plus its residual."""
    torch = cuda_device
    lib.set_mode(mode)
    m = 1 << 20 if n <= 1024 else 1 << 18
    bands = bs.diffusion_bands(1.0, n)
    f = bs.TriFactor(lib, *bands)
    x64 = torch.empty((n, m), dtype=torch.float64, device="cuda")
    lib.fill_rhs_dev(x64.data_ptr(), n, m, m, seed=42)
    x = x64.float()
    del x64
    rng = np.random.default_rng(n)
    cols = np.unique(np.concatenate([np.arange(64), np.arange(m - 64, m), rng.integers(0, m, 128)]))
    idx = torch.from_numpy(cols).cuda()
    rhs = x[:, idx].double().cpu().numpy()
    try:
        f.solve_dev(x.data_ptr(), n, m, f32=True)
        torch.cuda.synchronize()
        got = x[:, idx].double().cpu().numpy()
        want = oracle.tri_solve(oracle.tri_prefactor(*bands), rhs.copy())
        assert per_system_max_rel(got, want) <= TOL_F32, (n, m)
        sx, sr = bs.Batch.from_array(lib, got), bs.Batch.from_array(lib, rhs)
        assert lib.tri_residual(*bands, sx, sr) <= TOL_F32
    finally:
        lib.set_mode(bs.MODE_EXACT)
        del x
        torch.cuda.empty_cache()
