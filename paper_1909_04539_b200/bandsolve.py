"""ctypes binding of the bandsolve C ABI (include/bandsolve.h).

The same classes drive either the B200 library (libbandsolve_b200.so, the
default) or any other library exporting the reference ABI
(/root/reference/proj/include/bandsolve.h) — tests and the bench's reference
arm point it at the reference build. Names follow the C entry points; every
non-OK status raises BandsolveError carrying the status and the library's
last-error text, the Python rendering of the reference's status returns
(capi.cpp:38-72).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB = os.path.join(PKG_DIR, "libbandsolve_b200.so")

OK = 0
ERR_BAD_ARG = 1
ERR_SHAPE_MISMATCH = 2
ERR_FACTORIZATION_BREAKDOWN = 3
ERR_DIVISION_BY_ZERO = 4
ERR_SINGULAR_CORRECTION = 5
ERR_SINGULAR_MATRIX = 6
ERR_BAD_FORMAT = 7
ERR_IO = 8
ERR_INTERNAL = 9

MODE_EXACT = 0
MODE_FAST = 1

KIND_TRI = 0
KIND_PENT = 1
KIND_UNIFORM = 2

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_vp = C.c_void_p
_sz = C.c_size_t
_st = C.c_int

class BenchParams(C.Structure):
    """bandsolve_bench_params (ref bandsolve.h:199-208)."""
    _fields_ = [("n", C.c_size_t), ("m", C.c_size_t), ("steps", C.c_long), ("dt", C.c_double),
                ("problem", C.c_int), ("variant", C.c_int), ("dump_every", C.c_long),
                ("dump_prefix", C.c_char_p)]


class BenchResult(C.Structure):
    """bandsolve_bench_result (ref bandsolve.h:210-217)."""
    _fields_ = [("wall_s", C.c_double), ("per_step_mean_s", C.c_double), ("per_step_std_s", C.c_double),
                ("elements", C.c_uint64), ("threads", C.c_int), ("steps", C.c_long)]


PROBLEM_DIFFUSION, PROBLEM_HYPERDIFFUSION = 0, 1
VARIANT_SHARED, VARIANT_PER_SYSTEM, VARIANT_UNIFORM = 0, 1, 2
VARIANT_CUSPARSE = 3  # extension: the per-system step with cuSPARSE as the solver

# (name, restype, argtypes) of the reference ABI subset (ref bandsolve.h)
_REFERENCE_SIGS = [
    ("bandsolve_status_string", C.c_char_p, [_st]),
    ("bandsolve_version", C.c_char_p, []),
    ("bandsolve_get_threads", C.c_int, []),
    ("bandsolve_set_threads", None, [C.c_int]),
    ("bandsolve_batch_create", _st, [_sz, _sz, C.POINTER(_vp)]),
    ("bandsolve_batch_destroy", None, [_vp]),
    ("bandsolve_batch_rows", _sz, [_vp]),
    ("bandsolve_batch_systems", _sz, [_vp]),
    ("bandsolve_batch_data", _dp, [_vp]),
    ("bandsolve_batch_data_const", _dp, [_vp]),
    ("bandsolve_batch_read_ibat", _st, [C.c_char_p, C.POINTER(_vp)]),
    ("bandsolve_batch_write_ibat", _st, [_vp, C.c_char_p]),
    ("bandsolve_tri_solve_per_system", _st, [_vp] * 4),
    ("bandsolve_pent_solve_per_system", _st, [_vp] * 6),
    ("bandsolve_tri_factor_create", _st, [_dp, _dp, _dp, _sz, C.POINTER(_vp)]),
    ("bandsolve_tri_factor_destroy", None, [_vp]),
    ("bandsolve_tri_solve_shared", _st, [_vp, _vp]),
    ("bandsolve_pent_factor_create", _st, [_dp, _dp, _dp, _dp, _dp, _sz, C.POINTER(_vp)]),
    ("bandsolve_pent_factor_destroy", None, [_vp]),
    ("bandsolve_pent_solve_shared", _st, [_vp, _vp]),
    ("bandsolve_uniform_pent_factor_create", _st,
     [C.c_double] * 5 + [_sz, C.POINTER(_vp)]),
    ("bandsolve_uniform_pent_factor_destroy", None, [_vp]),
    ("bandsolve_pent_solve_uniform", _st, [_vp, _vp]),
    ("bandsolve_tri_residual", _st, [_dp, _dp, _dp, _sz, C.c_int, _vp, _vp, _dp]),
    ("bandsolve_pent_residual", _st, [_dp] * 5 + [_sz, C.c_int, _vp, _vp, _dp]),
    ("bandsolve_periodic_tri_create", _st, [C.c_double] * 3 + [_sz, C.POINTER(_vp)]),
    ("bandsolve_periodic_tri_destroy", None, [_vp]),
    ("bandsolve_periodic_tri_solve", _st, [_vp, _vp]),
    ("bandsolve_periodic_tri_modified_bands", _st, [_vp, _dp, _dp, _dp]),
    ("bandsolve_periodic_tri_correct", _st, [_vp, _vp]),
    ("bandsolve_periodic_pent_create", _st, [C.c_double] * 5 + [_sz, C.POINTER(_vp)]),
    ("bandsolve_periodic_pent_destroy", None, [_vp]),
    ("bandsolve_periodic_pent_solve", _st, [_vp, _vp]),
    ("bandsolve_periodic_pent_modified_bands", _st, [_vp] + [_dp] * 5),
    ("bandsolve_periodic_pent_correct", _st, [_vp, _vp]),
    ("bandsolve_footprint", _st, [C.c_int, _sz, _sz, C.POINTER(C.c_uint64), _dp]),
    ("bandsolve_bench_run", _st, [C.POINTER(BenchParams), C.POINTER(BenchResult)]),
]

# B200 extensions (include/bandsolve.h, second part)
_EXTENSION_SIGS = [
    ("bandsolve_set_mode", _st, [C.c_int]),
    ("bandsolve_get_mode", C.c_int, []),
    ("bandsolve_tri_solve_shared_dev", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_tri_solve_shared_dev_f32", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_pent_solve_shared_dev", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_pent_solve_shared_dev_f32", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_pent_solve_uniform_dev", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_tri_solve_per_system_dev", _st, [_vp] * 4 + [_sz, _sz, _sz, _vp]),
    ("bandsolve_pent_solve_per_system_dev", _st, [_vp] * 6 + [_sz, _sz, _sz, _vp]),
    ("bandsolve_pent_solve_uniform_dev_f32", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_cusparse_available", C.c_int, []),
    ("bandsolve_tri_solve_cusparse_dev", _st, [_vp] * 4 + [_sz, _sz, C.c_int, _vp]),
    ("bandsolve_pent_solve_cusparse_dev", _st, [_vp] * 6 + [_sz, _sz, _vp]),
    ("bandsolve_tri_residual_dev", _st,
     [_dp, _dp, _dp, _sz, C.c_int, _vp, _vp, _sz, _sz, _vp, _dp]),
    ("bandsolve_pent_residual_dev", _st,
     [_dp] * 5 + [_sz, C.c_int, _vp, _vp, _sz, _sz, _vp, _dp]),
    ("bandsolve_fill_rhs_dev", _st, [_vp, _sz, _sz, _sz, C.c_uint64, C.c_uint64, _vp]),
    ("bandsolve_fill_rhs_dev_f32", _st, [_vp, _sz, _sz, _sz, C.c_uint64, C.c_uint64, _vp]),
    ("bandsolve_tri_factor_order", _sz, [_vp]),
    ("bandsolve_tri_factor_arrays", _st, [_vp, _dp, _dp, _dp]),
    ("bandsolve_pent_factor_order", _sz, [_vp]),
    ("bandsolve_pent_factor_arrays", _st, [_vp, _dp, _dp, _dp, _dp, _dp]),
    ("bandsolve_uniform_pent_factor_order", _sz, [_vp]),
    ("bandsolve_uniform_pent_factor_arrays", _st, [_vp, _dp, _dp, _dp, _dp, _dp]),
    ("bandsolve_periodic_tri_solve_dev", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_periodic_tri_correct_dev", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_periodic_pent_solve_dev", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_periodic_pent_correct_dev", _st, [_vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_periodic_tri_cn_step_dev", _st, [_vp, C.c_double, _vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_periodic_pent_cn_step_dev", _st, [_vp, C.c_double, _vp, _vp, _sz, _sz, _sz, _vp]),
    ("bandsolve_adi_create", _st, [C.c_int, C.c_double, _sz, _sz, C.POINTER(_vp)]),
    ("bandsolve_adi_destroy", None, [_vp]),
    ("bandsolve_adi_step_dev", _st, [_vp, _vp, _vp, _sz, _vp]),
    ("bandsolve_describe_plan", _st, [C.c_int, _sz, _sz, _sz, C.c_int, C.c_char_p, _sz]),
    ("bandsolve_set_devices", _st, [C.POINTER(C.c_int), C.c_int]),
    ("bandsolve_get_devices", C.c_int, [C.POINTER(C.c_int), C.c_int]),
    ("bandsolve_tune_set", _st, [C.c_char_p, C.c_char_p]),
    ("bandsolve_tune_get", _st, [C.c_char_p, C.c_char_p, _sz]),
    ("bandsolve_tune_reset", None, []),
    ("bandsolve_kernel_launches", C.c_uint64, []),
    ("bandsolve_last_error", C.c_char_p, []),
]

REFERENCE_SYMBOLS = [s[0] for s in _REFERENCE_SIGS]
EXTENSION_SYMBOLS = [s[0] for s in _EXTENSION_SIGS]


class BandsolveError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{message} (status {status})")
        self.status = status


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(v, n: Optional[int] = None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    if n is not None and a.shape != (n,):
        raise ValueError(f"band must have length {n}")
    return a


class Library:
    """One loaded bandsolve-ABI shared library."""

    def __init__(self, path: str = DEFAULT_LIB, mode: int = C.RTLD_LOCAL):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is missing: build it first (python -c 'import __graft_entry__ as g; g.build()')")
        self.path = path
        self.lib = C.CDLL(path, mode=mode)
        for name, res, args in _REFERENCE_SIGS:
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args
        self.has_extensions = hasattr(self.lib, "bandsolve_set_mode")
        if self.has_extensions:
            for name, res, args in _EXTENSION_SIGS:
                fn = getattr(self.lib, name)
                fn.restype = res
                fn.argtypes = args

    # -- status plumbing ----------------------------------------------------
    def check(self, status: int, what: str = "") -> None:
        if status != OK:
            msg = self.lib.bandsolve_status_string(status).decode()
            if self.has_extensions:
                detail = self.lib.bandsolve_last_error().decode()
                if detail:
                    msg = f"{msg}: {detail}"
            raise BandsolveError(status, f"{what}: {msg}" if what else msg)

    def status_string(self, status: int) -> str:
        return self.lib.bandsolve_status_string(status).decode()

    def version(self) -> str:
        return self.lib.bandsolve_version().decode()

    def get_threads(self) -> int:
        return self.lib.bandsolve_get_threads()

    def set_threads(self, n: int) -> None:
        self.lib.bandsolve_set_threads(n)

    # -- extensions ---------------------------------------------------------
    def set_mode(self, mode: int) -> None:
        self.check(self.lib.bandsolve_set_mode(mode), "set_mode")

    def get_mode(self) -> int:
        return self.lib.bandsolve_get_mode()

    def set_devices(self, devices) -> None:
        """Device list of the host-batch solves ([] = the current device)."""
        ids = (C.c_int * max(1, len(devices)))(*devices)
        self.check(self.lib.bandsolve_set_devices(ids if devices else None, len(devices)), "set_devices")

    def get_devices(self) -> list[int]:
        n = self.lib.bandsolve_get_devices(None, 0)
        ids = (C.c_int * max(1, n))()
        self.lib.bandsolve_get_devices(ids, n)
        return list(ids[:n])

    def tune(self, key: str, value=None) -> None:
        """Set (value not None) or unset a tuning override (bandsolve_tune_set)."""
        v = None if value is None else str(value).encode()
        self.check(self.lib.bandsolve_tune_set(key.encode(), v), f"tune {key}")

    def tune_get(self, key: str) -> Optional[str]:
        buf = C.create_string_buffer(256)
        if self.lib.bandsolve_tune_get(key.encode(), buf, 256) != 0:
            return None
        return buf.value.decode()

    def tune_reset(self) -> None:
        self.lib.bandsolve_tune_reset()

    def kernel_launches(self) -> int:
        return int(self.lib.bandsolve_kernel_launches())

    def describe_plan(self, kind: int, n: int, m: int, ld: Optional[int] = None, f32: bool = False) -> str:
        buf = C.create_string_buffer(256)
        self.check(self.lib.bandsolve_describe_plan(kind, n, m, ld if ld is not None else m,
                                                    int(f32), buf, 256), "describe_plan")
        return buf.value.decode()

    def fill_rhs_dev(self, ptr: int, n: int, m: int, ld: int, seed: int, j_offset: int = 0,
                     stream: int = 0, f32: bool = False) -> None:
        fn = self.lib.bandsolve_fill_rhs_dev_f32 if f32 else self.lib.bandsolve_fill_rhs_dev
        self.check(fn(ptr, n, m, ld, seed, j_offset, stream), "fill_rhs_dev")

    def cusparse_available(self) -> bool:
        return bool(self.lib.bandsolve_cusparse_available())

    def cusparse_solve_dev(self, band_ptrs: Sequence[int], x_ptr: int, n: int, m: int, algo: int = 0,
                           stream: int = 0) -> None:
        """cuSPARSE gtsv/gpsvInterleavedBatch comparator on per-system device
        bands (3 tri / 5 pent pointers, n x m each, pitch m)."""
        if len(band_ptrs) == 3:
            st = self.lib.bandsolve_tri_solve_cusparse_dev(*band_ptrs, x_ptr, n, m, algo, stream)
        elif len(band_ptrs) == 5:
            st = self.lib.bandsolve_pent_solve_cusparse_dev(*band_ptrs, x_ptr, n, m, stream)
        else:
            raise ValueError("3 (tri) or 5 (pent) band pointers")
        self.check(st, "cusparse_solve_dev")

    # -- residuals ----------------------------------------------------------
    def footprint(self, variant: int, n: int, m: int) -> tuple[int, float]:
        el, red = C.c_uint64(), C.c_double()
        self.check(self.lib.bandsolve_footprint(variant, n, m, C.byref(el), C.byref(red)), "footprint")
        return int(el.value), float(red.value)

    def bench_run(self, n: int, m: int, steps: int, problem: int = PROBLEM_DIFFUSION,
                  variant: int = VARIANT_SHARED, dt: float = 0.0, dump_every: int = 0,
                  dump_prefix: Optional[str] = None) -> BenchResult:
        """bandsolve_bench_run (ref bandsolve.h:219-220): Crank-Nicolson stepping."""
        p = BenchParams(n, m, steps, dt, problem, variant, dump_every,
                        dump_prefix.encode() if dump_prefix else None)
        r = BenchResult()
        self.check(self.lib.bandsolve_bench_run(C.byref(p), C.byref(r)), "bench_run")
        return r

    def tri_residual(self, sub, diag, sup, x: "Batch", rhs: "Batch", cyclic: bool = False) -> float:
        n = len(diag)
        s, d, u = _f64(sub, n), _f64(diag, n), _f64(sup, n)
        out = C.c_double(-1.0)
        self.check(self.lib.bandsolve_tri_residual(_dptr(s), _dptr(d), _dptr(u), n, int(cyclic),
                                                   x.handle, rhs.handle, C.byref(out)), "tri_residual")
        return out.value

    def pent_residual(self, a, b, c, d, e, x: "Batch", rhs: "Batch", cyclic: bool = False) -> float:
        n = len(c)
        bands = [_f64(v, n) for v in (a, b, c, d, e)]
        out = C.c_double(-1.0)
        self.check(self.lib.bandsolve_pent_residual(*[_dptr(v) for v in bands], n, int(cyclic),
                                                    x.handle, rhs.handle, C.byref(out)), "pent_residual")
        return out.value

    def tri_residual_dev(self, sub, diag, sup, x_ptr: int, rhs_ptr: int, m: int, ld: int,
                         cyclic: bool = False, stream: int = 0) -> float:
        n = len(diag)
        s, d, u = _f64(sub, n), _f64(diag, n), _f64(sup, n)
        out = C.c_double(-1.0)
        self.check(self.lib.bandsolve_tri_residual_dev(_dptr(s), _dptr(d), _dptr(u), n, int(cyclic),
                                                       x_ptr, rhs_ptr, m, ld, stream, C.byref(out)),
                   "tri_residual_dev")
        return out.value

    def pent_residual_dev(self, a, b, c, d, e, x_ptr: int, rhs_ptr: int, m: int, ld: int,
                          cyclic: bool = False, stream: int = 0) -> float:
        n = len(c)
        bands = [_f64(v, n) for v in (a, b, c, d, e)]
        out = C.c_double(-1.0)
        self.check(self.lib.bandsolve_pent_residual_dev(*[_dptr(v) for v in bands], n, int(cyclic),
                                                        x_ptr, rhs_ptr, m, ld, stream, C.byref(out)),
                   "pent_residual_dev")
        return out.value


class Batch:
    """Owning bandsolve_batch handle with a numpy (n, m) view of its data."""

    def __init__(self, lib: Library, n: int, m: int, _handle: Optional[_vp] = None):
        self.lib = lib
        h = _handle
        if h is None:
            h = _vp()
            lib.check(lib.lib.bandsolve_batch_create(n, m, C.byref(h)), "batch_create")
        self.handle = h
        self.n, self.m = n, m
        ptr = lib.lib.bandsolve_batch_data(h)
        self.array = np.ctypeslib.as_array(ptr, shape=(n, m))

    @classmethod
    def read_ibat(cls, lib: Library, path: str) -> "Batch":
        """bandsolve_batch_read_ibat (ref batch.cpp:172-218)."""
        h = _vp()
        lib.check(lib.lib.bandsolve_batch_read_ibat(str(path).encode(), C.byref(h)), "batch_read_ibat")
        return cls(lib, lib.lib.bandsolve_batch_rows(h), lib.lib.bandsolve_batch_systems(h), _handle=h)

    def write_ibat(self, path: str) -> None:
        """bandsolve_batch_write_ibat (ref batch.cpp:146-170)."""
        self.lib.check(self.lib.lib.bandsolve_batch_write_ibat(self.handle, str(path).encode()), "batch_write_ibat")

    @classmethod
    def from_array(cls, lib: Library, arr) -> "Batch":
        a = np.asarray(arr, dtype=np.float64)
        if a.ndim == 1:
            a = a.reshape(-1, 1)
        b = cls(lib, a.shape[0], a.shape[1])
        b.array[...] = a
        return b

    def rows(self) -> int:
        return self.lib.lib.bandsolve_batch_rows(self.handle)

    def systems(self) -> int:
        return self.lib.lib.bandsolve_batch_systems(self.handle)

    def close(self) -> None:
        if self.handle:
            self.lib.lib.bandsolve_batch_destroy(self.handle)
            self.handle = None
            self.array = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tri_solve_per_system(lib: Library, a: Batch, b: Batch, c: Batch, d: Batch) -> None:
    """bandsolve_tri_solve_per_system (ref tri_solver.cpp:51-112): a/b/c consumed, d -> x."""
    lib.check(lib.lib.bandsolve_tri_solve_per_system(a.handle, b.handle, c.handle, d.handle),
              "tri_solve_per_system")


def pent_solve_per_system(lib: Library, a: Batch, b: Batch, c: Batch, d: Batch, e: Batch, f: Batch) -> None:
    """bandsolve_pent_solve_per_system (ref pent_solver.cpp:131-219): b..e consumed, f -> x."""
    lib.check(lib.lib.bandsolve_pent_solve_per_system(a.handle, b.handle, c.handle, d.handle, e.handle, f.handle),
              "pent_solve_per_system")


class _Factor:
    _destroy = ""
    _solve = ""
    _solve_dev = ""
    _order = ""

    def __init__(self, lib: Library, handle: _vp, n: int):
        self.lib, self.handle, self.n = lib, handle, n

    def solve(self, batch: Batch) -> None:
        self.lib.check(getattr(self.lib.lib, self._solve)(self.handle, batch.handle), self._solve)

    def solve_dev(self, ptr: int, n: int, m: int, ld: Optional[int] = None, stream: int = 0,
                  f32: bool = False) -> None:
        name = self._solve_dev + ("_f32" if f32 else "")
        self.lib.check(getattr(self.lib.lib, name)(self.handle, ptr, n, m, m if ld is None else ld, stream),
                       name)

    def close(self) -> None:
        if self.handle:
            getattr(self.lib.lib, self._destroy)(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TriFactor(_Factor):
    """bandsolve_tri_factor (ref bandsolve.h:67-78)."""
    _destroy = "bandsolve_tri_factor_destroy"
    _solve = "bandsolve_tri_solve_shared"
    _solve_dev = "bandsolve_tri_solve_shared_dev"

    def __init__(self, lib: Library, sub, diag, sup):
        n = len(diag)
        s, d, u = _f64(sub, n), _f64(diag, n), _f64(sup, n)
        h = _vp()
        lib.check(lib.lib.bandsolve_tri_factor_create(_dptr(s), _dptr(d), _dptr(u), n, C.byref(h)),
                  "tri_factor_create")
        super().__init__(lib, h, n)

    def arrays(self) -> dict:
        out = {k: np.empty(self.n) for k in ("chat", "inv_denom", "sub")}
        self.lib.check(self.lib.lib.bandsolve_tri_factor_arrays(
            self.handle, _dptr(out["chat"]), _dptr(out["inv_denom"]), _dptr(out["sub"])), "tri_factor_arrays")
        return out


class PentFactor(_Factor):
    """bandsolve_pent_factor (ref bandsolve.h:91-100)."""
    _destroy = "bandsolve_pent_factor_destroy"
    _solve = "bandsolve_pent_solve_shared"
    _solve_dev = "bandsolve_pent_solve_shared_dev"

    def __init__(self, lib: Library, a, b, c, d, e):
        n = len(c)
        bands = [_f64(v, n) for v in (a, b, c, d, e)]
        h = _vp()
        lib.check(lib.lib.bandsolve_pent_factor_create(*[_dptr(v) for v in bands], n, C.byref(h)),
                  "pent_factor_create")
        super().__init__(lib, h, n)

    def arrays(self) -> dict:
        keys = ("inv_alpha", "beta", "gamma", "delta", "epsilon")
        out = {k: np.empty(self.n) for k in keys}
        self.lib.check(self.lib.lib.bandsolve_pent_factor_arrays(self.handle, *[_dptr(out[k]) for k in keys]),
                       "pent_factor_arrays")
        return out


class UniformPentFactor(_Factor):
    """bandsolve_uniform_pent_factor (ref bandsolve.h:105-113)."""
    _destroy = "bandsolve_uniform_pent_factor_destroy"
    _solve = "bandsolve_pent_solve_uniform"
    _solve_dev = "bandsolve_pent_solve_uniform_dev"

    def __init__(self, lib: Library, a: float, b: float, c: float, d: float, e: float, n: int):
        h = _vp()
        lib.check(lib.lib.bandsolve_uniform_pent_factor_create(a, b, c, d, e, n, C.byref(h)),
                  "uniform_pent_factor_create")
        super().__init__(lib, h, n)

    def arrays(self) -> dict:
        keys = ("inv_alpha", "beta", "gamma", "delta")
        out = {k: np.empty(self.n) for k in keys}
        eps = C.c_double()
        self.lib.check(self.lib.lib.bandsolve_uniform_pent_factor_arrays(
            self.handle, *[_dptr(out[k]) for k in keys], C.byref(eps)), "uniform_pent_factor_arrays")
        out["eps_scalar"] = eps.value
        return out


# ---- LHS definitions used by the configs (ref pde.cpp:62-71) ---------------
class _Periodic(_Factor):
    _correct = ""
    _correct_dev = ""

    def correct(self, batch: Batch) -> None:
        """The wrap correction alone (caller already solved A' y = d)."""
        self.lib.check(getattr(self.lib.lib, self._correct)(self.handle, batch.handle), self._correct)

    def correct_dev(self, ptr: int, n: int, m: int, ld: Optional[int] = None, stream: int = 0) -> None:
        self.lib.check(getattr(self.lib.lib, self._correct_dev)(self.handle, ptr, n, m, m if ld is None else ld,
                                                                  stream), self._correct_dev)


def read_ibat(path: str) -> np.ndarray:
    """IBAT file (batch.cpp:146-218): 'IBAT', u32 version 1, u64 n, u64 m, n*m LE binary64."""
    with open(path, "rb") as f:
        blob = f.read()
    if blob[:4] != b"IBAT" or int.from_bytes(blob[4:8], "little") != 1:
        raise ValueError(f"not an IBAT v1 file: {path}")
    n, m = int.from_bytes(blob[8:16], "little"), int.from_bytes(blob[16:24], "little")
    return np.frombuffer(blob, dtype="<f8", count=n * m, offset=24).reshape(n, m).astype(np.float64)


class PeriodicTri(_Periodic):
    """bandsolve_periodic_tri (ref bandsolve.h:118-131): cyclic constant-band
    tridiagonal system, rank-1 wrap correction."""
    _destroy = "bandsolve_periodic_tri_destroy"
    _solve = "bandsolve_periodic_tri_solve"
    _solve_dev = "bandsolve_periodic_tri_solve_dev"
    _correct = "bandsolve_periodic_tri_correct"
    _correct_dev = "bandsolve_periodic_tri_correct_dev"

    def __init__(self, lib: Library, a: float, b: float, c: float, n: int):
        h = _vp()
        lib.check(lib.lib.bandsolve_periodic_tri_create(a, b, c, n, C.byref(h)), "periodic_tri_create")
        super().__init__(lib, h, n)

    def cn_step_dev(self, sigma_x: float, u_ptr: int, out_ptr: int, n: int, m: int, ld: Optional[int] = None,
                    stream: int = 0) -> None:
        self.lib.check(self.lib.lib.bandsolve_periodic_tri_cn_step_dev(self.handle, sigma_x, u_ptr, out_ptr, n, m,
                                                                        m if ld is None else ld, stream),
                       "periodic_tri_cn_step_dev")

    def modified_bands(self):
        out = [np.empty(self.n) for _ in range(3)]
        self.lib.check(self.lib.lib.bandsolve_periodic_tri_modified_bands(self.handle, *[_dptr(v) for v in out]),
                       "periodic_tri_modified_bands")
        return out


class PeriodicPent(_Periodic):
    """bandsolve_periodic_pent (ref bandsolve.h:133-146): cyclic constant-band
    pentadiagonal system, rank-2 (Woodbury) wrap correction."""
    _destroy = "bandsolve_periodic_pent_destroy"
    _solve = "bandsolve_periodic_pent_solve"
    _solve_dev = "bandsolve_periodic_pent_solve_dev"
    _correct = "bandsolve_periodic_pent_correct"
    _correct_dev = "bandsolve_periodic_pent_correct_dev"

    def __init__(self, lib: Library, a: float, b: float, c: float, d: float, e: float, n: int):
        h = _vp()
        lib.check(lib.lib.bandsolve_periodic_pent_create(a, b, c, d, e, n, C.byref(h)), "periodic_pent_create")
        super().__init__(lib, h, n)

    def cn_step_dev(self, sigma_x: float, u_ptr: int, out_ptr: int, n: int, m: int, ld: Optional[int] = None,
                    stream: int = 0) -> None:
        self.lib.check(self.lib.lib.bandsolve_periodic_pent_cn_step_dev(self.handle, sigma_x, u_ptr, out_ptr, n, m,
                                                                         m if ld is None else ld, stream),
                       "periodic_pent_cn_step_dev")

    def modified_bands(self):
        out = [np.empty(self.n) for _ in range(5)]
        self.lib.check(self.lib.lib.bandsolve_periodic_pent_modified_bands(self.handle, *[_dptr(v) for v in out]),
                       "periodic_pent_modified_bands")
        return out


class ADI:
    """bandsolve_adi (B200 extension): periodic 2D Peaceman-Rachford ADI step."""

    def __init__(self, lib: Library, problem: int, sigma_x: float, nx: int, ny: int):
        self.lib, self.nx, self.ny = lib, nx, ny
        h = _vp()
        lib.check(lib.lib.bandsolve_adi_create(problem, sigma_x, nx, ny, C.byref(h)), "adi_create")
        self.handle = h

    def step_dev(self, field_ptr: int, work_ptr: int, ld: Optional[int] = None, stream: int = 0) -> None:
        self.lib.check(self.lib.lib.bandsolve_adi_step_dev(self.handle, field_ptr, work_ptr,
                                                           self.nx if ld is None else ld, stream), "adi_step_dev")

    def close(self) -> None:
        if self.handle:
            self.lib.lib.bandsolve_adi_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def diffusion_bands(sigma: float, n: int):
    """Crank-Nicolson diffusion LHS (-s, 1+2s, -s), structural zeros applied."""
    sub = np.full(n, -sigma)
    diag = np.full(n, 1.0 + 2.0 * sigma)
    sup = np.full(n, -sigma)
    sub[0] = 0.0
    sup[-1] = 0.0
    return sub, diag, sup


def hyper_bands(sigma: float, n: int):
    """Crank-Nicolson hyperdiffusion LHS (s, -4s, 1+6s, -4s, s)."""
    a = np.full(n, sigma)
    b = np.full(n, -4.0 * sigma)
    c = np.full(n, 1.0 + 6.0 * sigma)
    d = np.full(n, -4.0 * sigma)
    e = np.full(n, sigma)
    a[0] = a[1] = b[0] = 0.0
    d[-1] = e[-1] = e[-2] = 0.0
    return a, b, c, d, e


_default: Optional[Library] = None


def load(path: Optional[str] = None) -> Library:
    """The B200 library (cached). Raises if the .so has not been built."""
    global _default
    if path is not None:
        return Library(path)
    if _default is None:
        _default = Library(DEFAULT_LIB)
    return _default
