"""Multi-device host-batch solves (SURVEY.md §8(b) device/partition setter,
§8(e) column split): bandsolve_set_devices spreads a host batch's columns over
a device list with the reference's split j0 = m*g/G (parallel.cpp:53-54).
Columns are independent, so any device list must give the single-device
result bit for bit (the analogue of test_tri_solver.cpp:148-164, where any
worker count gives the same bits). On a one-GPU box the list repeats device
0: every shard still gets its own staging pipeline."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1909_04539_b200 import bandsolve as bs


def test_device_list_roundtrip_and_validation(lib):
    assert lib.get_devices() == []
    lib.set_devices([0, 0, 1])
    assert lib.get_devices() == [0, 0, 1]
    lib.set_devices([])
    assert lib.get_devices() == []
    assert lib.lib.bandsolve_set_devices(None, 2) == bs.ERR_BAD_ARG
    assert lib.lib.bandsolve_set_devices(None, -1) == bs.ERR_BAD_ARG
    neg = (bs.C.c_int * 1)(-3)
    assert lib.lib.bandsolve_set_devices(neg, 1) == bs.ERR_BAD_ARG
    assert lib.get_devices() == []


def test_device_list_without_gpu_still_fails_loudly(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib.set_devices([0, 0])
    f = bs.TriFactor(lib, *bs.diffusion_bands(1.0, 16))
    b = bs.Batch(lib, 16, 100)
    with pytest.raises(bs.BandsolveError) as e:
        f.solve(b)
    assert e.value.status == bs.ERR_INTERNAL


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0] * 8])
def test_split_is_bitwise_invariant(lib, cuda_device, devices):
    rng = np.random.default_rng(11)
    for kind, n, m in [("tri", 256, 4099), ("pent", 512, 70001), ("pent", 64, 5)]:
        bands = bs.diffusion_bands(1.0, n) if kind == "tri" else bs.hyper_bands(1.0, n)
        f = bs.TriFactor(lib, *bands) if kind == "tri" else bs.PentFactor(lib, *bands)
        rhs = rng.uniform(-1, 1, (n, m))
        one = bs.Batch.from_array(lib, rhs)
        lib.set_devices([])
        f.solve(one)
        many = bs.Batch.from_array(lib, rhs)
        lib.set_devices(devices)
        before = lib.kernel_launches()
        f.solve(many)
        launched = lib.kernel_launches() - before
        lib.set_devices([])
        assert one.array.tobytes() == many.array.tobytes(), (kind, n, m, devices)
        assert launched >= min(m, len(devices))  # every non-empty shard ran its own sweep


@pytest.mark.gpu
def test_split_periodic_and_missing_device(lib, cuda_device):
    torch = cuda_device
    n, m = 128, 3001
    rng = np.random.default_rng(12)
    rhs = rng.uniform(-1, 1, (n, m))
    per = bs.PeriodicPent(lib, 1.0, -4.0, 7.0, -4.0, 1.0, n)
    a = bs.Batch.from_array(lib, rhs)
    per.solve(a)
    lib.set_devices([0, 0, 0])
    b = bs.Batch.from_array(lib, rhs)
    per.solve(b)
    assert a.array.tobytes() == b.array.tobytes()
    lib.set_devices([torch.cuda.device_count()])  # one past the last device
    with pytest.raises(bs.BandsolveError) as e:
        per.solve(b)
    assert e.value.status == bs.ERR_BAD_ARG
