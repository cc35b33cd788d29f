"""Host-side checks of libbandsolve_b200 that need no GPU.

The library loads, exports every entry point include/bandsolve.h declares
(and every in-scope reference entry point), keeps the reference's status
codes and argument checks, and its host prefactor reproduces the
reference's factor arrays bit for bit. No solve is executed here; without a
device a solve must fail loudly (BANDSOLVE_ERR_INTERNAL), never fall back to
the CPU.
"""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

from oracle.oracle import bitwise_equal
from paper_1909_04539_b200 import bandsolve as bs

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "bandsolve.h")
REF_HEADER = "/root/reference/proj/include/bandsolve.h"

# Reference entry points in scope; the rest of the reference
# ABI (periodic, per-system, IBAT, footprint, bench) is out of scope.
IN_SCOPE = [
    "bandsolve_status_string", "bandsolve_version", "bandsolve_get_threads", "bandsolve_set_threads",
    "bandsolve_batch_create", "bandsolve_batch_destroy", "bandsolve_batch_rows", "bandsolve_batch_systems",
    "bandsolve_batch_data", "bandsolve_batch_data_const", "bandsolve_tri_factor_create",
    "bandsolve_tri_factor_destroy", "bandsolve_tri_solve_shared", "bandsolve_pent_factor_create",
    "bandsolve_pent_factor_destroy", "bandsolve_pent_solve_shared", "bandsolve_uniform_pent_factor_create",
    "bandsolve_uniform_pent_factor_destroy", "bandsolve_pent_solve_uniform", "bandsolve_tri_residual",
    "bandsolve_pent_residual",
]


def header_functions(path: str) -> list[str]:
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bandsolve_[a-z0-9_]+)\s*\(", text)))


def exported(path: str) -> set[str]:
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_exports_every_declared_symbol(lib):
    declared = header_functions(HEADER)
    assert len(declared) >= 40
    syms = exported(lib.path)
    missing = [f for f in declared if f not in syms]
    assert not missing, missing
    # nothing but the declared C ABI leaks out of the library
    extra = sorted(s for s in syms if s not in declared)
    assert not extra, extra


def test_in_scope_reference_entry_points_present(lib):
    declared = set(header_functions(HEADER))
    for name in IN_SCOPE:
        assert name in declared
    if os.path.exists(REF_HEADER):
        ref = set(header_functions(REF_HEADER))
        assert set(IN_SCOPE) <= ref  # same names as the reference header
        # the whole reference ABI is declared and exported (periodic, per-system,
        # IBAT, footprint and bench included)
        assert not sorted(ref - declared), sorted(ref - declared)
        assert not sorted(ref - exported(lib.path))


def test_status_strings_and_version(lib):
    # test_capi.cpp:21-27 plus the full capi.cpp:82-97 table
    expected = ["ok", "bad argument", "shape mismatch", "factorization breakdown", "division by zero",
                "singular correction", "singular matrix", "malformed IBAT data", "I/O failure",
                "internal error"]
    for code, text in enumerate(expected):
        assert lib.status_string(code) == text
    assert lib.status_string(42) == "unknown status"
    assert lib.version() == "1.0.0"


def test_status_strings_match_reference(lib, reflib):
    for code in range(11):
        assert lib.status_string(code) == reflib.status_string(code)


def test_thread_control(lib, monkeypatch):
    # test_capi.cpp:29-34, parallel.cpp:17-37
    lib.set_threads(3)
    assert lib.get_threads() == 3
    lib.set_threads(0)
    assert lib.get_threads() >= 1
    monkeypatch.setenv("BANDSOLVE_THREADS", "5")
    assert lib.get_threads() == 5
    lib.set_threads(-2)
    assert lib.get_threads() == 5


def test_batch_lifecycle(lib):
    # test_capi.cpp:36-47
    b = bs.Batch(lib, 4, 3)
    assert b.rows() == 4 and b.systems() == 3
    assert np.all(b.array == 0.0)
    b.array[...] = 1.5
    assert lib.lib.bandsolve_batch_data_const(b.handle)[11] == 1.5
    h = bs._vp()
    assert lib.lib.bandsolve_batch_create(0, 3, bs.C.byref(h)) == bs.ERR_BAD_ARG
    assert not h.value
    assert lib.lib.bandsolve_batch_create(4, 0, bs.C.byref(h)) == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_batch_create(4, 3, None) == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_batch_rows(None) == 0
    assert lib.lib.bandsolve_batch_systems(None) == 0
    assert not lib.lib.bandsolve_batch_data(None)
    lib.lib.bandsolve_batch_destroy(None)  # NULL-safe like the reference


def test_tri_factor_error_codes(lib):
    # test_capi.cpp:85-100
    n = 4
    zero = np.zeros(n)
    with pytest.raises(bs.BandsolveError) as e:
        bs.TriFactor(lib, zero, zero, zero)
    assert e.value.status == bs.ERR_FACTORIZATION_BREAKDOWN
    with pytest.raises(bs.BandsolveError) as e:
        bs.TriFactor(lib, np.ones(n), np.ones(n), zero)
    assert e.value.status == bs.ERR_BAD_ARG
    with pytest.raises(bs.BandsolveError) as e:
        bs.TriFactor(lib, [0.0, 0.0], [1.0, np.inf], [1.0, 0.0])
    assert e.value.status == bs.ERR_BAD_ARG
    with pytest.raises(bs.BandsolveError) as e:
        bs.TriFactor(lib, [0.0], [1.0], [0.0])  # n >= 2
    assert e.value.status == bs.ERR_BAD_ARG
    out = bs._vp(1234)
    d = np.ones(n)
    assert lib.lib.bandsolve_tri_factor_create(None, bs._dptr(d), bs._dptr(d), n, bs.C.byref(out)) == bs.ERR_BAD_ARG
    st = lib.lib.bandsolve_tri_factor_create(bs._dptr(zero), bs._dptr(zero), bs._dptr(zero), n, bs.C.byref(out))
    assert st == bs.ERR_FACTORIZATION_BREAKDOWN and not out.value  # *out = NULL on failure


def test_pent_factor_error_codes(lib):
    with pytest.raises(bs.BandsolveError) as e:
        bs.UniformPentFactor(lib, 0, 0, 1, 0, 0, 4)
    assert e.value.status == bs.ERR_BAD_ARG
    with pytest.raises(bs.BandsolveError) as e:
        bs.UniformPentFactor(lib, 0, 0, 0, 0, 0, 5)
    assert e.value.status == bs.ERR_FACTORIZATION_BREAKDOWN
    a = np.zeros(5); a[1] = 0.5
    with pytest.raises(bs.BandsolveError) as e:
        bs.PentFactor(lib, a, np.zeros(5), np.ones(5), np.zeros(5), np.zeros(5))
    assert e.value.status == bs.ERR_BAD_ARG


def test_tri_factor_arrays_bitwise_golden(lib, golden):
    names = [c for c in golden.cases if c.startswith("tri_") or c.startswith("kat_tri")]
    for name in names:
        g = golden.case(name)
        f = bs.TriFactor(lib, g["sub"], g["diag"], g["sup"]).arrays()
        assert bitwise_equal(f["chat"], g["chat"]), name
        assert bitwise_equal(f["inv_denom"], g["inv_denom"]), name
        assert bitwise_equal(f["sub"], g["sub"]), name


def test_pent_factor_arrays_bitwise_golden(lib, golden):
    names = [c for c in golden.cases if c.startswith("pent_") or c.startswith("kat_pent") or c.endswith("_shared")]
    for name in names:
        g = golden.case(name)
        f = bs.PentFactor(lib, g["a"], g["b"], g["c"], g["d"], g["e"]).arrays()
        for k in ("inv_alpha", "beta", "gamma", "delta", "epsilon"):
            assert bitwise_equal(f[k], g[k]), (name, k)


def test_uniform_factor_arrays_bitwise_golden(lib, golden):
    for name in [c for c in golden.cases if c.startswith("uniform_") and not c.endswith("_shared")]:
        g = golden.case(name)
        f = bs.UniformPentFactor(lib, *g["bands"], g["n"]).arrays()
        for k in ("inv_alpha", "beta", "gamma", "delta"):
            assert bitwise_equal(f[k], g[k]), (name, k)
        assert f["eps_scalar"] == g["eps_scalar"]


def test_factor_arrays_vs_oracle_random(lib, oracle):
    rng = np.random.default_rng(3)
    for n in [2, 3, 17, 512, 4096]:
        sub = rng.uniform(-1, 1, n); sub[0] = 0
        sup = rng.uniform(-1, 1, n); sup[-1] = 0
        diag = np.abs(sub) + np.abs(sup) + rng.uniform(0.5, 1.5, n)
        mine = bs.TriFactor(lib, sub, diag, sup).arrays()
        ref = oracle.tri_prefactor(sub, diag, sup)
        for k in ref:
            assert bitwise_equal(mine[k], ref[k]), (n, k)
    for n in [5, 6, 64, 1024]:
        bands = [rng.uniform(-1, 1, n) for _ in range(5)]
        bands[0][:2] = 0; bands[1][0] = 0; bands[3][-1] = 0; bands[4][-2:] = 0
        bands[2] = sum(np.abs(bands[k]) for k in (0, 1, 3, 4)) + rng.uniform(0.5, 1.5, n)
        mine = bs.PentFactor(lib, *bands).arrays()
        ref = oracle.pent_prefactor(*bands)
        for k in ref:
            assert bitwise_equal(mine[k], ref[k]), (n, k)


def test_modes(lib):
    lib.set_mode(bs.MODE_FAST)
    assert lib.get_mode() == bs.MODE_FAST
    lib.set_mode(bs.MODE_EXACT)
    assert lib.get_mode() == bs.MODE_EXACT
    with pytest.raises(bs.BandsolveError):
        lib.set_mode(7)


def test_plan_description(lib):
    s = lib.describe_plan(bs.KIND_PENT, 512, 65536)
    assert s.startswith("pipe"), s  # configs[1]: every row on chip (TMEM + smem), pipelined across groups
    lib.tune("PIPE", "0")
    s = lib.describe_plan(bs.KIND_PENT, 512, 65536)
    assert s.startswith("stream"), s  # the warp-specialised streaming kernel, head spilled to L2
    assert "head(L2)=0" not in s
    lib.tune("PIPE", None)
    assert "head(L2)=0" in lib.describe_plan(bs.KIND_TRI, 256, 4096)  # config 1 fits smem entirely
    assert "global" in lib.describe_plan(bs.KIND_TRI, 64, 3)  # odd pitch: no TMA
    assert "global" in lib.describe_plan(bs.KIND_TRI, 100000, 1 << 20)  # tile > smem


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="host has a GPU")
def test_solve_without_gpu_fails_loudly(lib):
    n = 8
    sub, diag, sup = bs.diffusion_bands(0.5, n)
    f = bs.TriFactor(lib, sub, diag, sup)
    b = bs.Batch(lib, n, 2)
    with pytest.raises(bs.BandsolveError) as e:
        f.solve(b)
    assert e.value.status == bs.ERR_INTERNAL
    assert "no CUDA device" in str(e.value)


def test_shape_and_null_checks_before_device(lib):
    n = 8
    f = bs.TriFactor(lib, *bs.diffusion_bands(0.5, n))
    wrong = bs.Batch(lib, n + 1, 2)
    with pytest.raises(bs.BandsolveError) as e:
        f.solve(wrong)
    assert e.value.status == bs.ERR_SHAPE_MISMATCH  # test_capi.cpp:77-80
    assert lib.lib.bandsolve_tri_solve_shared(None, wrong.handle) == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_tri_solve_shared(f.handle, None) == bs.ERR_BAD_ARG
    with pytest.raises(bs.BandsolveError) as e:
        f.solve_dev(0, n, 4)
    assert e.value.status == bs.ERR_BAD_ARG
    with pytest.raises(bs.BandsolveError) as e:
        f.solve_dev(4096, n, 4, ld=2)
    assert e.value.status == bs.ERR_BAD_ARG
