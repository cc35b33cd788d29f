"""Shared fixtures. `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "reference_cases.npz")
PRODUCT_LIB = os.path.join(REPO, "paper_1909_04539_b200", "libbandsolve_b200.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs under gpurun)")


def _build_product() -> None:
    if not os.path.exists(PRODUCT_LIB):
        subprocess.check_call(["make", "-s", "-C", os.path.join(REPO, "paper_1909_04539_b200", "csrc")])


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    """The reference library built from /root/reference sources, or skip."""
    from oracle.oracle import build_ref
    from paper_1909_04539_b200.bandsolve import Library
    path = build_ref()
    if path is None or not os.path.exists(path):
        pytest.skip("reference build unavailable (no /root/reference and no prebuilt oracle/_ref)")
    return Library(path)


@pytest.fixture(scope="session")
def _product_lib():
    _build_product()
    from paper_1909_04539_b200.bandsolve import Library
    return Library(PRODUCT_LIB)


@pytest.fixture
def lib(_product_lib):
    """The product library with a clean tuning table (bandsolve_tune_reset)
    and the default device list around every test: overrides never leak
    between tests."""
    _product_lib.tune_reset()
    _product_lib.set_devices([])
    yield _product_lib
    _product_lib.tune_reset()
    _product_lib.set_devices([])


class Golden:
    """Case-indexed view of tests/golden/reference_cases.npz."""

    def __init__(self, path: str):
        self.npz = np.load(path)
        self.cases = sorted({k.split("/")[0] for k in self.npz.files})

    def case(self, name: str) -> dict:
        prefix = name + "/"
        out = {k[len(prefix):]: self.npz[k] for k in self.npz.files if k.startswith(prefix)}
        n, m = int(out["n"][0]), int(out["m"][0])
        out["n"], out["m"] = n, m
        for key in ("rhs", "x"):
            if key in out:
                out[key] = out[key].reshape(n, m)
        for key in ("residual", "dense_err", "lr_err", "eps_scalar"):
            if key in out:
                out[key] = float(out[key][0])
        return out

    def names(self, prefix: str) -> list[str]:
        return [c for c in self.cases if c.startswith(prefix)]


@pytest.fixture(scope="session")
def golden():
    return Golden(GOLDEN)


@pytest.fixture(scope="session")
def cuda_device():
    """torch CUDA context for device-pointer tests (plumbing only)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    return torch
