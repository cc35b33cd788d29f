"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the CPU oracle.

Wraps oracle/liboracle.so (the plain-C restatement in bandsolve_oracle.c) and
locates the reference build oracle/_ref/libbandsolve_ref.so. Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module; the
product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(ORACLE_DIR, "liboracle.so")
REF_LIB = os.path.join(ORACLE_DIR, "_ref", "libbandsolve_ref.so")
REFERENCE_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t


def build_port() -> str:
    """Build liboracle.so if needed (gcc is in the image on both sides)."""
    src = os.path.join(ORACLE_DIR, "bandsolve_oracle.c")
    if not os.path.exists(PORT_LIB) or os.path.getmtime(PORT_LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", ORACLE_DIR, "port"])
    return PORT_LIB


def build_ref() -> str | None:
    """Build the reference library from /root/reference when that tree exists."""
    if os.path.exists(REF_LIB):
        return REF_LIB
    if not os.path.isdir(REFERENCE_SRC):
        return None
    subprocess.check_call(["make", "-s", "-C", ORACLE_DIR, "-j8", "ref"])
    return REF_LIB


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _arr(v, n=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    if n is not None:
        assert a.shape == (n,), (a.shape, n)
    return a


class OracleError(RuntimeError):
    def __init__(self, status: int):
        super().__init__(f"oracle status {status}")
        self.status = status


class Oracle:
    def __init__(self, path: str | None = None):
        self.lib = C.CDLL(path or build_port())
        L = self.lib
        L.oracle_tri_prefactor.argtypes = [_dp, _dp, _dp, _sz, _dp, _dp, _dp]
        L.oracle_tri_per_system.argtypes = [_dp] * 4 + [_sz, _sz]
        L.oracle_pent_per_system.argtypes = [_dp] * 6 + [_sz, _sz]
        L.oracle_tri_solve_shared.argtypes = [_dp, _dp, _dp, _sz, _sz, _sz, _dp]
        L.oracle_tri_solve_shared.restype = None
        L.oracle_pent_prefactor.argtypes = [_dp] * 5 + [_sz] + [_dp] * 5
        L.oracle_pent_solve.argtypes = [_dp] * 5 + [C.c_double, _sz, _sz, _sz, _dp]
        L.oracle_pent_solve.restype = None
        L.oracle_uniform_pent_prefactor.argtypes = [C.c_double] * 5 + [_sz] + [_dp] * 5
        L.oracle_tri_residual.argtypes = [_dp, _dp, _dp, _sz, C.c_int, _sz, _dp, _dp, _dp]
        L.oracle_pent_residual.argtypes = [_dp] * 5 + [_sz, C.c_int, _sz, _dp, _dp, _dp]
        L.oracle_max_error_vs_dense.argtypes = [_dp, _sz, _sz, _dp, _dp, _dp]
        L.oracle_rhs_value.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.oracle_rhs_value.restype = C.c_double
        L.oracle_fill_rhs.argtypes = [C.c_uint64, _sz, _sz, _sz, _sz, _dp]
        L.oracle_fill_rhs.restype = None
        L.oracle_periodic_tri_prepare.argtypes = [C.c_double] * 3 + [_sz] + [_dp] * 6
        L.oracle_periodic_tri_apply.argtypes = [_dp, C.c_double, C.c_double, _sz, _sz, _dp]
        L.oracle_periodic_tri_apply.restype = None
        L.oracle_periodic_pent_prepare.argtypes = [C.c_double] * 5 + [_sz] + [_dp] * 8
        L.oracle_periodic_pent_apply.argtypes = [_dp, _dp, _dp, _sz, _sz, _dp]
        L.oracle_periodic_pent_apply.restype = None
        L.oracle_default_mode_initial.argtypes = [_sz, _sz, _dp]
        L.oracle_default_mode_initial.restype = None
        L.oracle_cn_rhs.argtypes = [C.c_int, C.c_double, _sz, _sz, _dp, _dp]
        L.oracle_cn_rhs.restype = None

    # -- factors ------------------------------------------------------------
    def tri_prefactor(self, sub, diag, sup) -> dict:
        n = len(diag)
        s, d, u = _arr(sub, n), _arr(diag, n), _arr(sup, n)
        out = {k: np.zeros(n) for k in ("chat", "inv_denom", "sub")}
        st = self.lib.oracle_tri_prefactor(_d(s), _d(d), _d(u), n, _d(out["chat"]), _d(out["inv_denom"]),
                                           _d(out["sub"]))
        if st:
            raise OracleError(st)
        return out

    def pent_prefactor(self, a, b, c, d, e) -> dict:
        n = len(c)
        bands = [_arr(v, n) for v in (a, b, c, d, e)]
        keys = ("inv_alpha", "beta", "gamma", "delta", "epsilon")
        out = {k: np.zeros(n) for k in keys}
        st = self.lib.oracle_pent_prefactor(*[_d(v) for v in bands], n, *[_d(out[k]) for k in keys])
        if st:
            raise OracleError(st)
        return out

    def uniform_prefactor(self, a, b, c, d, e, n) -> dict:
        keys = ("inv_alpha", "beta", "gamma", "delta")
        out = {k: np.zeros(n) for k in keys}
        eps = np.zeros(1)
        st = self.lib.oracle_uniform_pent_prefactor(a, b, c, d, e, n, *[_d(out[k]) for k in keys], _d(eps))
        if st:
            raise OracleError(st)
        out["eps_scalar"] = float(eps[0])
        return out

    # -- sweeps (in place on a C-contiguous (n, m) float64 array) -------------
    def tri_solve(self, f: dict, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, m = x.shape
        self.lib.oracle_tri_solve_shared(_d(f["chat"]), _d(f["inv_denom"]), _d(f["sub"]), n, m, m, _d(x))
        return x

    def pent_solve(self, f: dict, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, m = x.shape
        eps = f.get("epsilon")
        self.lib.oracle_pent_solve(_d(f["inv_alpha"]), _d(f["beta"]), _d(f["gamma"]), _d(f["delta"]),
                                   _d(eps) if eps is not None else None, f.get("eps_scalar", 0.0),
                                   n, m, m, _d(x))
        return x

    # -- per-system baselines (reference tri_solver.cpp:51-112, pent_solver.cpp:131-219)
    def tri_per_system(self, a, b, c, d):
        """Destroys copies of b, c, d as the reference does; returns (status, b, c, d)."""
        arrs = [np.array(v, dtype=np.float64, order="C", copy=True) for v in (a, b, c, d)]
        n, m = arrs[0].shape
        st = self.lib.oracle_tri_per_system(*[_d(v) for v in arrs], n, m)
        return (st, *arrs[1:])

    def pent_per_system(self, a, b, c, d, e, f):
        """Destroys copies of b..f as the reference does; returns (status, b, c, d, e, f)."""
        arrs = [np.array(v, dtype=np.float64, order="C", copy=True) for v in (a, b, c, d, e, f)]
        n, m = arrs[0].shape
        st = self.lib.oracle_pent_per_system(*[_d(v) for v in arrs], n, m)
        return (st, *arrs[1:])

    # -- periodic wrap correction (reference periodic.cpp) -----------------------
    def periodic_tri_prepare(self, a, b, c, n) -> dict:
        f = {k: np.zeros(n) for k in ("chat", "inv_denom", "sub", "z")}
        vl, sc = np.zeros(1), np.zeros(1)
        st = self.lib.oracle_periodic_tri_prepare(a, b, c, n, _d(f["chat"]), _d(f["inv_denom"]), _d(f["sub"]),
                                                  _d(f["z"]), _d(vl), _d(sc))
        if st:
            raise OracleError(st)
        f["v_last"], f["scale"] = float(vl[0]), float(sc[0])
        return f

    def periodic_tri_solve(self, f: dict, x: np.ndarray, correct_only: bool = False) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, m = x.shape
        if not correct_only:
            self.tri_solve(f, x)
        self.lib.oracle_periodic_tri_apply(_d(f["z"]), f["v_last"], f["scale"], n, m, _d(x))
        return x

    def periodic_pent_prepare(self, a, b, c, d, e, n) -> dict:
        keys = ("inv_alpha", "beta", "gamma", "delta", "epsilon", "z1", "z2")
        f = {k: np.zeros(n) for k in keys}
        f["cap_inv"] = np.zeros(4)
        st = self.lib.oracle_periodic_pent_prepare(a, b, c, d, e, n, *[_d(f[k]) for k in keys], _d(f["cap_inv"]))
        if st:
            raise OracleError(st)
        return f

    def periodic_pent_solve(self, f: dict, x: np.ndarray, correct_only: bool = False) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n, m = x.shape
        if not correct_only:
            self.pent_solve(f, x)
        self.lib.oracle_periodic_pent_apply(_d(f["z1"]), _d(f["z2"]), _d(f["cap_inv"]), n, m, _d(x))
        return x

    # -- Crank-Nicolson (reference pde.cpp) ---------------------------------------
    def default_mode_initial(self, n: int, m: int) -> np.ndarray:
        out = np.empty((n, m))
        self.lib.oracle_default_mode_initial(n, m, _d(out))
        return out

    def cn_rhs(self, problem: int, sigma_x: float, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        n, m = u.shape
        out = np.empty_like(u)
        self.lib.oracle_cn_rhs(problem, sigma_x, n, m, _d(u), _d(out))
        return out

    @staticmethod
    def cn_sigma(problem: int, n: int, dt: float = 0.0) -> float:
        """bench_config::sigma_x (pde.cpp:29-46)."""
        dx = 1.0 / n
        pow_dx = dx * dx if problem == 0 else dx * dx * dx * dx
        dtv = dt if dt > 0.0 else 1.0 * 2.0 * pow_dx
        return dtv / (2.0 * pow_dx)

    @staticmethod
    def periodic_modified_bands(consts, n: int) -> list:
        """The strictly banded A' of the periodic splitting (periodic.cpp:11-31 tri,
        :97-129 pent), as the reference's per-system engine replicates it
        (pde.cpp:168-185, :199-221)."""
        if len(consts) == 3:
            a, b, c = consts
            sub, diag, sup = np.full(n, a), np.full(n, b), np.full(n, c)
            sub[0] = 0.0
            sup[n - 1] = 0.0
            diag[0] = 2.0 * b
            diag[n - 1] = b + a * c / b
            return [sub, diag, sup]
        a, b, c, d, e = consts
        av, bv, cv, dv, ev = (np.full(n, v) for v in (a, b, c, d, e))
        av[0] = av[1] = bv[0] = 0.0
        dv[n - 1] = ev[n - 1] = ev[n - 2] = 0.0
        cv[0] = c + b
        dv[0] = d + a
        bv[1] = b + a
        dv[n - 2] = d + e
        bv[n - 1] = b + e
        cv[n - 1] = c + d
        return [av, bv, cv, dv, ev]

    def cn_trajectory(self, problem: int, n: int, m: int, steps: int, dt: float = 0.0, variant: int = 0) -> list:
        """Fields after each step of run_benchmark (pde.cpp:279-343). Shared and
        uniform variants sweep the shared factor (bitwise the same,
        pent_solver.cpp:83-97); the per-system variant (1) rewrites replicated
        band copies of A' every step, solves per system, then applies the
        correction (pde.cpp:168-185, :199-221)."""
        s = self.cn_sigma(problem, n, dt)
        if problem == 0:
            consts = (-s, 1.0 + 2.0 * s, -s)
            f = self.periodic_tri_prepare(*consts, n)
            solve = self.periodic_tri_solve
        else:
            consts = (s, -4.0 * s, 1.0 + 6.0 * s, -4.0 * s, s)
            f = self.periodic_pent_prepare(*consts, n)
            solve = self.periodic_pent_solve
        bands = self.periodic_modified_bands(consts, n)
        u = self.default_mode_initial(n, m)
        out = []
        for _ in range(steps):
            rhs = self.cn_rhs(problem, s, u)
            if variant == 1:
                rep = [np.repeat(b[:, None], m, axis=1) for b in bands]
                res = (self.tri_per_system if problem == 0 else self.pent_per_system)(*rep, rhs)
                if res[0]:
                    raise OracleError(res[0])
                u = solve(f, res[-1], correct_only=True)
            else:
                u = solve(f, rhs)
            out.append(u.copy())
        return out

    def adi_step(self, problem: int, s: float, field: np.ndarray) -> np.ndarray:
        """One periodic Peaceman-Rachford step on an (ny, nx) field: explicit
        along y + implicit along x, then explicit along x + implicit along y,
        each half with the 1D Crank-Nicolson bands / stencil (pde.cpp)."""
        ny, nx = field.shape
        if problem == 0:
            fx = self.periodic_tri_prepare(-s, 1 + 2 * s, -s, nx)
            fy = self.periodic_tri_prepare(-s, 1 + 2 * s, -s, ny)
            solve = self.periodic_tri_solve
        else:
            fx = self.periodic_pent_prepare(s, -4 * s, 1 + 6 * s, -4 * s, s, nx)
            fy = self.periodic_pent_prepare(s, -4 * s, 1 + 6 * s, -4 * s, s, ny)
            solve = self.periodic_pent_solve
        t1 = np.ascontiguousarray(self.cn_rhs(problem, s, field).T)     # rows = x
        t1 = solve(fx, t1)
        t2 = np.ascontiguousarray(self.cn_rhs(problem, s, t1).T)        # rows = y
        return solve(fy, t2)

    # -- checks ---------------------------------------------------------------
    def tri_residual(self, sub, diag, sup, x, rhs, cyclic=False) -> float:
        n = len(diag)
        x = np.ascontiguousarray(x, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.zeros(1)
        st = self.lib.oracle_tri_residual(_d(_arr(sub, n)), _d(_arr(diag, n)), _d(_arr(sup, n)), n,
                                          int(cyclic), x.shape[1], _d(x), _d(rhs), _d(out))
        if st:
            raise OracleError(st)
        return float(out[0])

    def pent_residual(self, a, b, c, d, e, x, rhs, cyclic=False) -> float:
        n = len(c)
        x = np.ascontiguousarray(x, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.zeros(1)
        st = self.lib.oracle_pent_residual(*[_d(_arr(v, n)) for v in (a, b, c, d, e)], n, int(cyclic),
                                           x.shape[1], _d(x), _d(rhs), _d(out))
        if st:
            raise OracleError(st)
        return float(out[0])

    def max_error_vs_dense(self, dense: np.ndarray, x, rhs) -> float:
        dense = np.ascontiguousarray(dense, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        n = dense.shape[0]
        out = np.zeros(1)
        st = self.lib.oracle_max_error_vs_dense(_d(dense), n, x.shape[1], _d(x), _d(rhs), _d(out))
        if st:
            raise OracleError(st)
        return float(out[0])

    def rhs(self, seed: int, n: int, m: int, j_offset: int = 0) -> np.ndarray:
        x = np.empty((n, m))
        self.lib.oracle_fill_rhs(seed, n, m, j_offset, m, _d(x))
        return x


def dense_from_tri(sub, diag, sup) -> np.ndarray:
    """tests/support/oracles.cpp:59-67 (banded -> dense)."""
    n = len(diag)
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = diag[i]
        if i > 0:
            a[i, i - 1] = sub[i]
        if i + 1 < n:
            a[i, i + 1] = sup[i]
    return a


def dense_from_pent(a_, b_, c_, d_, e_) -> np.ndarray:
    """tests/support/oracles.cpp:69-79."""
    n = len(c_)
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = c_[i]
        if i >= 2:
            a[i, i - 2] = a_[i]
        if i >= 1:
            a[i, i - 1] = b_[i]
        if i + 1 < n:
            a[i, i + 1] = d_[i]
        if i + 2 < n:
            a[i, i + 2] = e_[i]
    return a


def per_system_max_rel(x: np.ndarray, ref: np.ndarray) -> float:
    """max_j ||x_j - ref_j||_inf / ||ref_j||_inf (oracles.cpp:104-122 metric)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(x - ref).max(axis=0)
    scale = np.abs(ref).max(axis=0)
    rel = np.where(scale > 0, err / np.where(scale > 0, scale, 1.0), err)
    return float(rel.max()) if rel.size else 0.0


def bitwise_equal(x: np.ndarray, y: np.ndarray) -> bool:
    """Bit-for-bit equality, treating any NaN as equal to any NaN."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.shape != y.shape:
        return False
    same = x.view(np.uint64) == y.view(np.uint64)
    both_nan = np.isnan(x) & np.isnan(y)
    return bool(np.all(same | both_nan))
