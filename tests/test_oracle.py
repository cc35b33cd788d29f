"""Pin the CPU oracle (oracle/bandsolve_oracle.c) before trusting it.

1. Known-answer tables hand-written in the reference's own tests
   (test_banded_core.cpp:35-55, :111-148).
2. Bit-for-bit agreement with the reference's outputs on every golden case
   (tests/golden/reference_cases.npz, produced by the reference build).
3. Live agreement with the reference library (oracle/_ref) on fresh random
   inputs, when that build is present.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import (OracleError, bitwise_equal, dense_from_pent, dense_from_tri,
                           per_system_max_rel)


def test_tri_prefactor_kat(oracle):
    # test_banded_core.cpp:35-55: a = -0.5, b = 2, c = -0.5, n = 4
    n = 4
    sub = np.full(n, -0.5); sub[0] = 0
    sup = np.full(n, -0.5); sup[-1] = 0
    f = oracle.tri_prefactor(sub, np.full(n, 2.0), sup)
    assert f["chat"][0] == -0.25
    np.testing.assert_allclose(f["chat"][1:3], [-0.26666666666666666, -0.26785714285714285], rtol=1e-15)
    assert f["chat"][3] == 0.0
    assert f["inv_denom"][0] == 0.5
    np.testing.assert_allclose(f["inv_denom"][1:],
                               [0.5333333333333333, 0.5357142857142857, 0.5358851674641149], rtol=1e-15)
    np.testing.assert_allclose(f["chat"][:3] / f["inv_denom"][:3], sup[:3], rtol=1e-14)


def test_pent_prefactor_kat(oracle):
    # test_banded_core.cpp:111-148: sigma = 1/4 hyperdiffusion bands, n = 6
    n = 6
    a = np.full(n, 0.25); a[:2] = 0
    b = np.full(n, -1.0); b[0] = 0
    d = np.full(n, -1.0); d[-1] = 0
    e = np.full(n, 0.25); e[-2:] = 0
    f = oracle.pent_prefactor(a, b, np.full(n, 2.5), d, e)
    assert 1.0 / f["inv_alpha"][0] == 2.5
    assert f["gamma"][0] == -0.4 and f["delta"][0] == 0.1
    np.testing.assert_allclose(f["inv_alpha"], [0.4, 0.47619047619047616, 0.4786324786324786,
                                                0.478772378516624, 0.47889279007103774, 0.4789035310679232],
                               rtol=1e-15)
    np.testing.assert_allclose(f["beta"], [0.0, -1.0, -0.9, -0.8928571428571429, -0.8931623931623932,
                                           -0.8930946291560102], rtol=1e-15)
    np.testing.assert_allclose(f["gamma"], [-0.4, -0.42857142857142855, -0.42735042735042733,
                                            -0.42762148337595907, -0.42769657875398054, 0.0], rtol=1e-15)
    np.testing.assert_allclose(f["delta"], [0.1, 0.11904761904761904, 0.11965811965811965,
                                            0.119693094629156, 0.0, 0.0], rtol=1e-15)
    assert bitwise_equal(f["epsilon"], a)


def test_identity_factors(oracle):
    # test_banded_core.cpp:25-33, :99-109
    f = oracle.tri_prefactor(np.zeros(3), np.ones(3), np.zeros(3))
    assert np.all(f["chat"] == 0) and np.all(f["inv_denom"] == 1)
    p = oracle.pent_prefactor(np.zeros(5), np.zeros(5), np.ones(5), np.zeros(5), np.zeros(5))
    assert np.all(p["inv_alpha"] == 1) and not np.any(p["beta"]) and not np.any(p["gamma"])


def test_breakdown_and_validation(oracle):
    # test_banded_core.cpp:81-97, :185-195
    with pytest.raises(OracleError) as e:
        oracle.tri_prefactor([0.0, 0.0], [0.0, 1.0], [1.0, 0.0])
    assert e.value.status == 3
    with pytest.raises(OracleError) as e:
        oracle.tri_prefactor([1.0, 0.0], [1.0, 1.0], [1.0, 0.0])
    assert e.value.status == 1
    with pytest.raises(OracleError) as e:
        oracle.tri_prefactor([0.0, 0.0], [1.0, np.nan], [1.0, 0.0])
    assert e.value.status == 1
    with pytest.raises(OracleError) as e:
        oracle.pent_prefactor(*[np.zeros(5)] * 5)
    assert e.value.status == 3
    bad = np.zeros(5); bad[1] = 0.5
    with pytest.raises(OracleError) as e:
        oracle.pent_prefactor(bad, np.zeros(5), np.ones(5), np.zeros(5), np.zeros(5))
    assert e.value.status == 1
    with pytest.raises(OracleError) as e:
        oracle.uniform_prefactor(0, 0, 1, 0, 0, 4)
    assert e.value.status == 1


def _tri_case_check(oracle, g):
    f = oracle.tri_prefactor(g["sub"], g["diag"], g["sup"])
    assert bitwise_equal(f["chat"], g["chat"])
    assert bitwise_equal(f["inv_denom"], g["inv_denom"])
    x = oracle.tri_solve(f, g["rhs"].copy())
    assert bitwise_equal(x, g["x"])
    r = oracle.tri_residual(g["sub"], g["diag"], g["sup"], x, g["rhs"])
    assert bitwise_equal(np.array([r]), np.array([g["residual"]]))
    if "dense_err" in g:
        err = oracle.max_error_vs_dense(dense_from_tri(g["sub"], g["diag"], g["sup"]), x, g["rhs"])
        assert bitwise_equal(np.array([err]), np.array([g["dense_err"]]))


def _pent_case_check(oracle, g):
    f = oracle.pent_prefactor(g["a"], g["b"], g["c"], g["d"], g["e"])
    for k in ("inv_alpha", "beta", "gamma", "delta", "epsilon"):
        assert bitwise_equal(f[k], g[k]), k
    x = oracle.pent_solve(f, g["rhs"].copy())
    assert bitwise_equal(x, g["x"])
    r = oracle.pent_residual(g["a"], g["b"], g["c"], g["d"], g["e"], x, g["rhs"])
    assert bitwise_equal(np.array([r]), np.array([g["residual"]]))
    if "dense_err" in g:
        err = oracle.max_error_vs_dense(dense_from_pent(g["a"], g["b"], g["c"], g["d"], g["e"]), x, g["rhs"])
        assert bitwise_equal(np.array([err]), np.array([g["dense_err"]]))


def test_golden_tri_cases_bitwise(oracle, golden):
    names = [c for c in golden.cases if c.startswith("tri_") or c == "kat_tri_sigma05_n4"]
    assert len(names) >= 40
    for name in names:
        _tri_case_check(oracle, golden.case(name))


def test_golden_pent_cases_bitwise(oracle, golden):
    names = [c for c in golden.cases
             if (c.startswith("pent_") or c == "kat_pent_sigma025_n6" or c.endswith("_shared"))]
    assert len(names) >= 25
    for name in names:
        _pent_case_check(oracle, golden.case(name))


def test_golden_uniform_cases_bitwise(oracle, golden):
    names = [c for c in golden.cases if c.startswith("uniform_") and not c.endswith("_shared")]
    assert len(names) >= 4
    for name in names:
        g = golden.case(name)
        a, b, c, d, e = g["bands"]
        f = oracle.uniform_prefactor(a, b, c, d, e, g["n"])
        for k in ("inv_alpha", "beta", "gamma", "delta"):
            assert bitwise_equal(f[k], g[k]), (name, k)
        assert f["eps_scalar"] == g["eps_scalar"]
        x = oracle.pent_solve(f, g["rhs"].copy())
        assert bitwise_equal(x, g["x"]), name


def test_uniform_equals_shared_golden(golden):
    # test_pent_solver.cpp:165-177: the reference's uniform == shared bitwise
    u = golden.case("uniform_n32_m4")
    s = golden.case("uniform_n32_m4_shared")
    assert bitwise_equal(u["x"], s["x"])


def test_golden_accuracy_bounds(golden):
    # the reference's own bounds on its own outputs (acceptance_main.cpp:41-88)
    for name in golden.names("tri_accept1_") + golden.names("pent_accept2_"):
        assert golden.case(name)["dense_err"] <= 1e-9
    for name in golden.names("pent_lr_n"):
        assert golden.case(name)["lr_err"] <= 1e-11


def test_rhs_generator_range_and_determinism(oracle):
    x = oracle.rhs(42, 64, 257)
    assert np.all(x >= -1.0) and np.all(x < 1.0)
    assert abs(x.mean()) < 0.05
    y = oracle.rhs(42, 64, 100, j_offset=100)
    assert bitwise_equal(x[:, 100:200], y)  # shards of one global batch agree


@pytest.mark.parametrize("threads", [1, 2, 4])
def test_live_reference_tri(oracle, reflib, threads):
    """Fresh random inputs through the reference library's C ABI vs the oracle."""
    from paper_1909_04539_b200.bandsolve import Batch, TriFactor
    rng = np.random.default_rng(7 + threads)
    reflib.set_threads(threads)
    try:
        for n, m in [(2, 1), (3, 5), (64, 33), (257, 130)]:
            sub = rng.uniform(-1, 1, n); sub[0] = 0
            sup = rng.uniform(-1, 1, n); sup[-1] = 0
            diag = np.abs(sub) + np.abs(sup) + rng.uniform(0.5, 1.5, n)
            rhs = rng.uniform(-1, 1, (n, m))
            fac = TriFactor(reflib, sub, diag, sup)
            bt = Batch.from_array(reflib, rhs)
            fac.solve(bt)
            mine = oracle.tri_solve(oracle.tri_prefactor(sub, diag, sup), rhs.copy())
            assert bitwise_equal(bt.array, mine)
    finally:
        reflib.set_threads(0)


def test_live_reference_pent(oracle, reflib):
    from paper_1909_04539_b200.bandsolve import Batch, PentFactor, UniformPentFactor
    rng = np.random.default_rng(11)
    for n, m in [(5, 1), (6, 7), (97, 40), (512, 64)]:
        a = rng.uniform(-1, 1, n); a[:2] = 0
        b = rng.uniform(-1, 1, n); b[0] = 0
        d = rng.uniform(-1, 1, n); d[-1] = 0
        e = rng.uniform(-1, 1, n); e[-2:] = 0
        c = np.abs(a) + np.abs(b) + np.abs(d) + np.abs(e) + rng.uniform(0.5, 1.5, n)
        rhs = rng.uniform(-1, 1, (n, m))
        fac = PentFactor(reflib, a, b, c, d, e)
        bt = Batch.from_array(reflib, rhs)
        fac.solve(bt)
        mine = oracle.pent_solve(oracle.pent_prefactor(a, b, c, d, e), rhs.copy())
        assert bitwise_equal(bt.array, mine)
        res_ref = reflib.pent_residual(a, b, c, d, e, bt, Batch.from_array(reflib, rhs))
        assert res_ref == oracle.pent_residual(a, b, c, d, e, mine, rhs)
    # uniform, hyperdiffusion sigma = 1 (pde.cpp:67-71), config-2 row count
    u = UniformPentFactor(reflib, 1.0, -4.0, 7.0, -4.0, 1.0, 512)
    rhs = oracle.rhs(42, 512, 8)
    bt = Batch.from_array(reflib, rhs)
    u.solve(bt)
    mine = oracle.pent_solve(oracle.uniform_prefactor(1.0, -4.0, 7.0, -4.0, 1.0, 512), rhs.copy())
    assert bitwise_equal(bt.array, mine)


def test_live_reference_residual_cyclic(oracle, reflib):
    from paper_1909_04539_b200.bandsolve import Batch
    rng = np.random.default_rng(5)
    n, m = 16, 6
    x = rng.uniform(-1, 1, (n, m))
    rhs = rng.uniform(-1, 1, (n, m))
    sub = np.full(n, -0.3); diag = np.full(n, 2.0); sup = np.full(n, -0.7)
    r_ref = reflib.tri_residual(sub, diag, sup, Batch.from_array(reflib, x), Batch.from_array(reflib, rhs),
                                cyclic=True)
    assert r_ref == oracle.tri_residual(sub, diag, sup, x, rhs, cyclic=True)
    bands = [np.full(n, v) for v in (0.2, -0.9, 3.0, -0.8, 0.1)]
    r_ref = reflib.pent_residual(*bands, Batch.from_array(reflib, x), Batch.from_array(reflib, rhs), cyclic=True)
    assert r_ref == oracle.pent_residual(*bands, x, rhs, cyclic=True)


def test_per_system_metric():
    ref = np.array([[1.0, 0.0], [2.0, 0.0]])
    x = np.array([[1.0, 1e-3], [2.2, 0.0]])
    # column 0: 0.2 / 2; column 1 has a zero reference -> absolute error
    assert per_system_max_rel(x, ref) == pytest.approx(0.1)
