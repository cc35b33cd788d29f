"""A compiled C program as the ABI's consumer (tests/c/capi_consumer.c).

It includes only include/bandsolve.h and links against the library through
the reference's SONAME, libbandsolve.so.1 (the drop-in relink of
INTEGRATION.md), then runs the assertions of the reference's C-API suite
(test_capi.cpp:21-141). Without a GPU every solve must report
BANDSOLVE_ERR_INTERNAL (no CPU fallback); on a B200 every solve must succeed
with the reference's residual bounds.
"""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_1909_04539_b200", "libbandsolve_b200.so")


@pytest.fixture(scope="module")
def consumer(tmp_path_factory, _product_lib):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    d = tmp_path_factory.mktemp("cabi")
    os.symlink(LIB, d / "libbandsolve.so.1")  # what a binary linked against the reference asks for
    exe = d / "capi_consumer"
    subprocess.check_call([cc, "-std=c11", "-Wall", "-Wextra", "-Werror", "-O1",
                           "-I", os.path.join(REPO, "include"), os.path.join(REPO, "tests", "c", "capi_consumer.c"),
                           "-o", str(exe), f"-L{d}", "-l:libbandsolve.so.1", f"-Wl,-rpath,{d}", "-lm"])
    needed = subprocess.run(["readelf", "-d", str(exe)], capture_output=True, text=True).stdout
    assert "libbandsolve.so.1" in needed  # the reference's DT_NEEDED name
    return exe


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_library_soname_is_the_reference_one(_product_lib):
    out = subprocess.run(["readelf", "-d", LIB], capture_output=True, text=True).stdout
    assert "Library soname: [libbandsolve.so.1]" in out


def test_c_consumer_without_gpu(consumer):
    if _has_gpu():
        pytest.skip("a GPU is present: the gpu variant covers this")
    r = subprocess.run([str(consumer), "nogpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_consumer_on_gpu(consumer):
    r = subprocess.run([str(consumer), "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
