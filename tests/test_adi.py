"""2D ADI step — BASELINE configs[3], SURVEY.md §8(f) rank 3 (no reference
counterpart: SPEC.md:464 lists ADI as a non-goal of the reference). Checked
against the oracle's composition of the pinned 1D pieces (periodic stencil,
cyclic solve, exact transposes): bitwise in exact mode, 1e-12 in fast mode.
"""
from __future__ import annotations


import numpy as np
import pytest

from oracle.oracle import bitwise_equal, per_system_max_rel
from paper_1909_04539_b200 import bandsolve as bs


def test_adi_create_statuses(lib):
    for args, st in [((0, 1.0, 2, 8), bs.ERR_BAD_ARG), ((1, 1.0, 8, 5), bs.ERR_BAD_ARG),
                     ((3, 1.0, 8, 8), bs.ERR_BAD_ARG), ((0, 0.0, 8, 8), bs.ERR_BAD_ARG)]:
        with pytest.raises(bs.BandsolveError) as e:
            bs.ADI(lib, *args)
        assert e.value.status == st, args
    bs.ADI(lib, 1, 0.5, 16, 12).close()
    assert lib.lib.bandsolve_adi_step_dev(None, None, None, 0, None) == bs.ERR_BAD_ARG


@pytest.mark.gpu
def test_gpu_adi_step(lib, oracle, cuda_device):
    torch = cuda_device
    rng = np.random.default_rng(41)
    stream = torch.cuda.current_stream().cuda_stream
    for problem, ny, nx in [(0, 8, 5), (0, 33, 70), (0, 256, 300), (1, 6, 9), (1, 64, 40), (1, 512, 130)]:
        s = 0.7
        c = rng.uniform(-1, 1, (ny, nx))
        want = oracle.adi_step(problem, s, c)
        adi = bs.ADI(lib, problem, s, nx, ny)
        for mode in (bs.MODE_EXACT, bs.MODE_FAST):
            lib.set_mode(mode)
            try:
                for ld in (nx, nx + (nx % 2) + 2):
                    f = torch.zeros((ny, ld), dtype=torch.float64, device="cuda")
                    f[:, :nx] = torch.from_numpy(c).cuda()
                    w = torch.zeros_like(f)
                    adi.step_dev(f.data_ptr(), w.data_ptr(), ld=ld, stream=stream)
                    torch.cuda.synchronize()
                    got = f[:, :nx].cpu().numpy()
                    if mode == bs.MODE_EXACT:
                        assert bitwise_equal(got, want), (problem, ny, nx, ld)
                    else:
                        assert per_system_max_rel(got, want) <= 1e-12, (problem, ny, nx, ld)
            finally:
                lib.set_mode(bs.MODE_EXACT)
    # the periodic operators conserve the mean (row sums 1)
    f = torch.from_numpy(rng.uniform(-1, 1, (128, 96))).cuda()
    mean0 = float(f.mean())
    adi = bs.ADI(lib, 0, 1.0, 96, 128)
    w = torch.zeros_like(f)
    for _ in range(5):
        adi.step_dev(f.data_ptr(), w.data_ptr(), stream=stream)
    torch.cuda.synchronize()
    assert abs(float(f.mean()) - mean0) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("fuse_pent", [False, True])
def test_gpu_adi_fast_partitioned_fused_stencil(lib, oracle, cuda_device, fuse_pent):
    """Fast mode on grids large enough for the partitioned path (both axes
    >= 1024): the explicit half is fused into the partitioned forward pass
    (tri; pent with tuning key ADI_FUSE_PENT), the correction into the
    backward pass. Within 1e-12 of the oracle's ADI step; an odd pitch and a
    system count that is not a multiple of 32 take the unfused route."""
    torch = cuda_device
    rng = np.random.default_rng(43)
    stream = torch.cuda.current_stream().cuda_stream
    if fuse_pent:
        lib.tune("ADI_FUSE_PENT", "1")
    lib.set_mode(bs.MODE_FAST)
    try:
        for problem, ny, nx in [(0, 1024, 1056), (1, 1088, 1024), (0, 1030, 1024)]:
            s = 0.9
            c = rng.uniform(-1, 1, (ny, nx))
            want = oracle.adi_step(problem, s, c)
            adi = bs.ADI(lib, problem, s, nx, ny)
            for ld in (nx, nx + 1, nx + 2):
                f = torch.zeros((ny, ld), dtype=torch.float64, device="cuda")
                f[:, :nx] = torch.from_numpy(c).cuda()
                w = torch.zeros_like(f)
                adi.step_dev(f.data_ptr(), w.data_ptr(), ld=ld, stream=stream)
                torch.cuda.synchronize()
                assert per_system_max_rel(f[:, :nx].cpu().numpy(), want) <= 1e-12, (problem, ny, nx, ld)
    finally:
        lib.set_mode(bs.MODE_EXACT)
        lib.tune("ADI_FUSE_PENT", None)


@pytest.mark.gpu
@pytest.mark.parametrize("problem", [0, 1])
def test_gpu_adi_configs3_full_size(lib, oracle, cuda_device, problem):
    """configs[3] itself: one ADI step on the 4096 x 4096 field, every point
    against the oracle's composition — bitwise in exact mode, within 1e-12
    in fast mode (fused partitioned pass for tri, transpose + cluster spike
    kernel for pent)."""
    torch = cuda_device
    rng = np.random.default_rng(44 + problem)
    stream = torch.cuda.current_stream().cuda_stream
    n = 4096
    s = 1.0
    c = rng.uniform(-1, 1, (n, n))
    want = oracle.adi_step(problem, s, c)
    adi = bs.ADI(lib, problem, s, n, n)
    try:
        for mode in (bs.MODE_EXACT, bs.MODE_FAST):
            lib.set_mode(mode)
            f = torch.from_numpy(c).cuda()
            w = torch.zeros_like(f)
            adi.step_dev(f.data_ptr(), w.data_ptr(), stream=stream)
            torch.cuda.synchronize()
            got = f.cpu().numpy()
            if mode == bs.MODE_EXACT:
                assert bitwise_equal(got, want), problem
            else:
                assert per_system_max_rel(got, want) <= 1e-12, problem
    finally:
        lib.set_mode(bs.MODE_EXACT)
