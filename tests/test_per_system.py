"""Per-system baselines and IBAT files — SURVEY.md §8(f) row 4.

* The oracle's per-system restatement is pinned bit for bit to the reference
  library built from its sources (oracle/_ref), over every array the
  reference destroys, including breakdown statuses (CPU).
* IBAT files: the product writes files byte-identical to the reference's, each
  reads the other's, and malformed files get the reference's statuses (CPU:
  IBAT is host I/O).
* The GPU per-system kernels (csrc/per_system.cu) equal the oracle bit for bit
  through the host C-ABI and the device entry points (GPU).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle.oracle import bitwise_equal
from paper_1909_04539_b200 import bandsolve as bs


def random_tri_columns(rng, n, m):
    a = rng.uniform(-1, 1, (n, m)); a[0] = 0
    c = rng.uniform(-1, 1, (n, m)); c[-1] = 0
    b = np.abs(a) + np.abs(c) + rng.uniform(0.5, 1.5, (n, m))
    d = rng.uniform(-1, 1, (n, m))
    return a, b, c, d


def random_pent_columns(rng, n, m):
    a = rng.uniform(-1, 1, (n, m)); a[:2] = 0
    b = rng.uniform(-1, 1, (n, m)); b[0] = 0
    d = rng.uniform(-1, 1, (n, m)); d[-1] = 0
    e = rng.uniform(-1, 1, (n, m)); e[-2:] = 0
    c = np.abs(a) + np.abs(b) + np.abs(d) + np.abs(e) + rng.uniform(0.5, 1.5, (n, m))
    f = rng.uniform(-1, 1, (n, m))
    return a, b, c, d, e, f


def run_lib_per_system(lib, arrays, pent):
    """Through the reference-facing host ABI; returns (status, destroyed arrays b.. )."""
    batches = [bs.Batch.from_array(lib, v) for v in arrays]
    fn = lib.lib.bandsolve_pent_solve_per_system if pent else lib.lib.bandsolve_tri_solve_per_system
    st = fn(*[b.handle for b in batches])
    out = [b.array.copy() for b in batches[1:]]
    for b in batches:
        b.close()
    return st, out


# ---- oracle pinned to the reference (CPU) ------------------------------------------
@pytest.mark.parametrize("pent", [False, True])
def test_oracle_per_system_matches_reference(oracle, reflib, pent):
    rng = np.random.default_rng(8)
    for n, m in [(5, 1), (6, 3), (64, 17), (300, 40)]:
        arrays = random_pent_columns(rng, n, m) if pent else random_tri_columns(rng, n, m)
        st_ref, ref_out = run_lib_per_system(reflib, arrays, pent)
        got = oracle.pent_per_system(*arrays) if pent else oracle.tri_per_system(*arrays)
        assert st_ref == got[0] == bs.OK
        for r, g in zip(ref_out, got[1:]):
            assert bitwise_equal(r, g), (n, m)


@pytest.mark.parametrize("pent", [False, True])
def test_oracle_per_system_statuses_match_reference(oracle, reflib, pent):
    rng = np.random.default_rng(9)
    n, m = 8, 4
    arrays = [v.copy() for v in (random_pent_columns(rng, n, m) if pent else random_tri_columns(rng, n, m))]
    diag = arrays[2] if pent else arrays[1]
    diag[0, 1] = 0.0  # zero first pivot in column 1
    st_ref, _ = run_lib_per_system(reflib, arrays, pent)
    got = oracle.pent_per_system(*arrays) if pent else oracle.tri_per_system(*arrays)
    assert st_ref == got[0] == bs.ERR_FACTORIZATION_BREAKDOWN
    small = [v[: (4 if pent else 1)] for v in arrays]
    st_ref, _ = run_lib_per_system(reflib, small, pent)
    assert st_ref == bs.ERR_BAD_ARG
    assert (oracle.pent_per_system(*small) if pent else oracle.tri_per_system(*small))[0] == bs.ERR_BAD_ARG


# ---- IBAT (host I/O, CPU) ------------------------------------------------------------------
def test_ibat_byte_identical_and_cross_readable(lib, reflib, tmp_path):
    rng = np.random.default_rng(10)
    x = rng.standard_normal((7, 5))
    x[0, 0] = -0.0
    x[1, 1] = np.inf
    x[2, 2] = np.nan
    mine, ref = tmp_path / "mine.ibat", tmp_path / "ref.ibat"
    bm = bs.Batch.from_array(lib, x)
    br = bs.Batch.from_array(reflib, x)
    bm.write_ibat(str(mine))
    br.write_ibat(str(ref))
    assert mine.read_bytes() == ref.read_bytes()
    assert len(mine.read_bytes()) == 24 + 7 * 5 * 8
    for reader, path in [(lib, ref), (reflib, mine), (lib, mine)]:
        b = bs.Batch.read_ibat(reader, str(path))
        assert (b.rows(), b.systems()) == (7, 5)
        assert b.array.tobytes() == x.tobytes()
        b.close()


def test_ibat_error_statuses_match_reference(lib, reflib, tmp_path):
    good = bytearray(b"IBAT" + (1).to_bytes(4, "little") + (2).to_bytes(8, "little") + (3).to_bytes(8, "little"))
    good += bytes(2 * 3 * 8)
    cases = {
        "missing": None,
        "short_header": bytes(good[:10]),
        "bad_magic": b"IBAX" + bytes(good[4:]),
        "bad_version": bytes(good[:4]) + (2).to_bytes(4, "little") + bytes(good[8:]),
        "zero_rows": bytes(good[:8]) + (0).to_bytes(8, "little") + bytes(good[16:]),
        "huge_m": bytes(good[:16]) + ((1 << 28) + 1).to_bytes(8, "little") + bytes(good[24:]),
        "truncated_payload": bytes(good[:-8]),
        "extra_payload": bytes(good) + b"\0",
        "good": bytes(good),
    }
    for name, content in cases.items():
        path = tmp_path / f"{name}.ibat"
        if content is not None:
            path.write_bytes(content)
        sts = []
        for L in (lib, reflib):
            h = bs._vp()
            st = L.lib.bandsolve_batch_read_ibat(str(path).encode(), bs.C.byref(h))
            if st == bs.OK:
                L.lib.bandsolve_batch_destroy(h)
            sts.append(st)
        assert sts[0] == sts[1], (name, sts)
        assert (sts[0] == bs.OK) == (name == "good"), (name, sts)
    b = bs.Batch(lib, 2, 2)
    assert lib.lib.bandsolve_batch_write_ibat(b.handle, str(tmp_path / "no_dir" / "x.ibat").encode()) == bs.ERR_IO
    assert lib.lib.bandsolve_batch_write_ibat(None, b"x") == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_batch_read_ibat(None, None) == bs.ERR_BAD_ARG


# ---- GPU kernels vs the oracle ------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("pent", [False, True])
def test_gpu_per_system_bitwise(lib, oracle, cuda_device, pent):
    rng = np.random.default_rng(11)
    for n, m in [(5, 1), (6, 33), (64, 17), (513, 300), (2048, 129)]:
        arrays = random_pent_columns(rng, n, m) if pent else random_tri_columns(rng, n, m)
        st, got = run_lib_per_system(lib, arrays, pent)
        want = oracle.pent_per_system(*arrays) if pent else oracle.tri_per_system(*arrays)
        assert st == want[0] == bs.OK
        for g, w in zip(got, want[1:]):
            assert bitwise_equal(g, w), (n, m)


@pytest.mark.gpu
@pytest.mark.parametrize("pent", [False, True])
def test_gpu_per_system_device_entry(lib, oracle, cuda_device, pent):
    torch = cuda_device
    rng = np.random.default_rng(12)
    n, m, ld = 300, 70, 72
    arrays = random_pent_columns(rng, n, m) if pent else random_tri_columns(rng, n, m)
    dev = []
    for v in arrays:
        t = torch.full((n, ld), float("nan"), dtype=torch.float64, device="cuda")
        t[:, :m] = torch.from_numpy(v).cuda()
        dev.append(t)
    fn = lib.lib.bandsolve_pent_solve_per_system_dev if pent else lib.lib.bandsolve_tri_solve_per_system_dev
    st = fn(*[t.data_ptr() for t in dev], n, m, ld, torch.cuda.current_stream().cuda_stream)
    assert st == bs.OK
    want = oracle.pent_per_system(*arrays) if pent else oracle.tri_per_system(*arrays)
    for t, w in zip(dev[1:], want[1:]):
        out = t.cpu().numpy()
        assert bitwise_equal(out[:, :m], w)
        assert np.all(np.isnan(out[:, m:]))


@pytest.mark.gpu
@pytest.mark.parametrize("pent", [False, True])
def test_gpu_per_system_statuses(lib, cuda_device, pent):
    rng = np.random.default_rng(13)
    n, m = 16, 8
    arrays = [v.copy() for v in (random_pent_columns(rng, n, m) if pent else random_tri_columns(rng, n, m))]
    (arrays[2] if pent else arrays[1])[0, 5] = 0.0  # zero first pivot in column 5
    st, _ = run_lib_per_system(lib, arrays, pent)
    assert st == bs.ERR_FACTORIZATION_BREAKDOWN
    small = [v[: (4 if pent else 1)] for v in arrays]
    st, _ = run_lib_per_system(lib, small, pent)
    assert st == bs.ERR_BAD_ARG
    mixed = [bs.Batch.from_array(lib, v) for v in arrays]
    mixed[-1] = bs.Batch.from_array(lib, arrays[-1][:, :4])
    fn = lib.lib.bandsolve_pent_solve_per_system if pent else lib.lib.bandsolve_tri_solve_per_system
    assert fn(*[b.handle for b in mixed]) == bs.ERR_SHAPE_MISMATCH
    assert fn(*([None] * (6 if pent else 4))) == bs.ERR_BAD_ARG


# ---- cuSPARSE comparators (gtsv/gpsvInterleavedBatch) ---------------------------------------------
def max_rel_err(got, want):
    """Per-system max-norm relative error, max over systems."""
    return float(np.max(np.max(np.abs(got - want), axis=0) / np.max(np.abs(want), axis=0)))


@pytest.mark.gpu
@pytest.mark.parametrize("pent", [False, True])
def test_gpu_cusparse_comparator_vs_oracle(lib, oracle, cuda_device, pent):
    """The library comparator solves the reference's per-system problems to
    1e-12 of the oracle (different algorithms: Thomas / QR, so not bitwise)."""
    torch = cuda_device
    assert lib.cusparse_available()
    rng = np.random.default_rng(14)
    for n, m in [(5, 1), (64, 17), (513, 300)]:
        arrays = random_pent_columns(rng, n, m) if pent else random_tri_columns(rng, n, m)
        want = (oracle.pent_per_system(*arrays) if pent else oracle.tri_per_system(*arrays))[-1]
        dev = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in arrays]
        lib.cusparse_solve_dev([t.data_ptr() for t in dev[:-1]], dev[-1].data_ptr(), n, m,
                               stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert max_rel_err(dev[-1].cpu().numpy(), want) <= 1e-12, (n, m)


@pytest.mark.gpu
def test_gpu_cusparse_arguments(lib, cuda_device):
    torch = cuda_device
    t = torch.zeros((4, 3), dtype=torch.float64, device="cuda")
    p = t.data_ptr()
    with pytest.raises(bs.BandsolveError) as e:
        lib.cusparse_solve_dev([p, p, p, p, p], p, 4, 3)  # pent needs n >= 5
    assert e.value.status == bs.ERR_BAD_ARG
    with pytest.raises(bs.BandsolveError) as e:
        lib.cusparse_solve_dev([p, p, p], p, 4, 3, algo=7)
    assert e.value.status == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_tri_solve_cusparse_dev(None, None, None, None, 4, 3, 0, None) == bs.ERR_BAD_ARG


@pytest.mark.gpu
@pytest.mark.parametrize("problem", [bs.PROBLEM_DIFFUSION, bs.PROBLEM_HYPERDIFFUSION])
def test_gpu_bench_cusparse_variant_tracks_shared(lib, cuda_device, tmp_path, problem):
    """The cuSPARSE step (same stencil, same correction) evolves the same
    field as the shared step to rounding (pde.cpp run_benchmark protocol)."""
    n, m, steps = 64, 48, 5
    fields = {}
    for v in (bs.VARIANT_SHARED, bs.VARIANT_CUSPARSE):
        prefix = str(tmp_path / f"v{v}")
        r = lib.bench_run(n, m, steps, problem=problem, variant=v, dump_every=steps, dump_prefix=prefix)
        assert r.steps == steps and r.per_step_mean_s > 0
        b = bs.Batch.read_ibat(lib, f"{prefix}_step{steps}.ibat")
        fields[v] = b.array.copy()
        b.close()
    assert np.max(np.abs(fields[bs.VARIANT_SHARED] - fields[bs.VARIANT_CUSPARSE])) <= 1e-12


@pytest.mark.gpu
def test_gpu_acceptance_speedup_trend(lib, cuda_device):
    """Reference acceptance criterion 8 (acceptance_main.cpp:482-510): at
    n = 256, m = 4096, 1000 Crank-Nicolson steps, the shared-LHS step is no
    slower than the per-system step, for both problems (mean of 3 runs)."""
    for problem in (bs.PROBLEM_DIFFUSION, bs.PROBLEM_HYPERDIFFUSION):
        mean = {}
        for v in (bs.VARIANT_SHARED, bs.VARIANT_PER_SYSTEM):
            mean[v] = sum(lib.bench_run(256, 4096, 1000, problem=problem, variant=v).per_step_mean_s
                          for _ in range(3)) / 3
        assert mean[bs.VARIANT_SHARED] <= mean[bs.VARIANT_PER_SYSTEM], (problem, mean)


# ---- the bench command (reference tools/main.cpp run_bench) -----------------------------------------
CLI = os.path.join(os.path.dirname(bs.DEFAULT_LIB), "bandsolve_b200")


def run_cli(*args):
    import subprocess
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_cli_version_and_argument_errors(lib, tmp_path):
    """Argument validation happens before any device work (exit 2, as the
    reference's exit_args); --version prints the library version."""
    assert os.path.exists(CLI), "bandsolve_b200 not built"
    r = run_cli("--version")
    assert r.returncode == 0 and r.stdout.strip() == "1.0.0"
    out = str(tmp_path / "b.csv")
    for bad in (["--problem", "heat"], ["--variants", "shared,fancy"], ["--n", "64,0"], ["--m", "x"],
                ["--steps", "0"], ["--problem", "diffusion", "--variants", "uniform"], ["--bogus", "1"]):
        r = run_cli("bench", "--out", out, *bad)
        assert r.returncode == 2, (bad, r.stderr)
        assert not os.path.exists(out)
    assert run_cli("solve").returncode == 2


@pytest.mark.gpu
def test_gpu_cli_bench_csv_schema(lib, cuda_device, tmp_path):
    out = tmp_path / "bench.csv"
    r = run_cli("bench", "--problem", "both", "--variants", "shared,persystem,cusparse", "--n", "64,128",
                "--m", "64,256", "--steps", "20", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rows = out.read_text().splitlines()
    assert rows[0] == "problem,variant,n,m,steps,threads,wall_s,per_step_mean_s,per_step_std_s,elements"
    assert len(rows) == 1 + 2 * 3 * 2 * 2
    for row in rows[1:]:
        f = row.split(",")
        assert f[0] in ("diffusion", "hyperdiffusion") and f[1] in ("shared", "persystem", "cusparse")
        assert int(f[4]) == 20 and float(f[7]) > 0
    sp = (tmp_path / "bench.speedup.csv").read_text().splitlines()
    assert sp[0] == "problem,n,m,variant,speedup_vs_persystem"
    assert len(sp) == 1 + 2 * 2 * 2 * 2
    spc = (tmp_path / "bench.speedup_cusparse.csv").read_text().splitlines()
    assert spc[0] == "problem,n,m,variant,speedup_vs_cusparse"
