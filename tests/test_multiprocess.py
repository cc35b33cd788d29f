"""Multi-GPU sharding across processes: world-size-2 gloo groups.

Each rank takes its shard of one global synthetic batch (partition.py, the
reference's j0 = M*g/G split, which bench.py uses for its strong-scaling
shards), solves it, and the shards reassembled on rank 0 must equal the
single-process solve bit for bit (ref parallel.hpp:20-23: columns are
partition independent). On CPU the oracle stands in for each rank's GPU (the
host logic: split, gather, max-over-ranks reduction); the gpu-marked variant
solves every shard through the product library.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_1909_04539_b200.partition import shard_range, weak_shard


def test_shard_range_covers_and_aligns():
    for m in (1, 31, 32, 4096, 65536, 100003):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(m, g, world) for g in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0 and a0 <= a1
            for j0, _ in ranges:
                assert j0 % 32 == 0
    assert weak_shard(65536, 3) == (196608, 262144)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_1909_04539_b200 import bandsolve as bs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        n, m = 96, 1000
        bands = bs.hyper_bands(1.0, n)
        f = orc.pent_prefactor(*bands)
        j0, j1 = shard_range(m, rank, world)
        shard = orc.rhs(42, n, j1 - j0, j_offset=j0)  # this rank's columns of the global batch
        x = orc.pent_solve(f, shard)
        # gather the shards to rank 0
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([j1 - j0], dtype=torch.int64))
        width = int(max(s.item() for s in sizes))
        buf = torch.zeros((n, width), dtype=torch.float64)
        buf[:, : j1 - j0] = torch.from_numpy(x)
        parts = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        # max-over-ranks of a per-rank "device time", as bench.py does
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            full = np.concatenate([p.numpy()[:, : int(s.item())] for p, s in zip(parts, sizes)], axis=1)
            ref = orc.pent_solve(f, orc.rhs(42, n, m))
            q.put((full.tobytes() == ref.tobytes(), float(t.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_reassemble_bitwise():
    mp = pytest.importorskip("torch.multiprocessing")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    same, tmax = q.get(timeout=5)
    assert same
    assert tmax == 2.0


def _gpu_worker(rank: int, world: int, port: int, q) -> None:
    """bench.py's strong-scaling split through the product: each rank
    generates and solves its shard [j0, j1) of the global batch on the GPU
    (both ranks share cuda:0 on a one-GPU box), rank 0 reassembles."""
    import torch
    import torch.distributed as dist

    from paper_1909_04539_b200 import bandsolve as bs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lib = bs.load()
        n, m = 1024, 40000
        f = bs.PentFactor(lib, *bs.hyper_bands(1.0, n))
        j0, j1 = shard_range(m, rank, world)
        x = torch.empty((n, j1 - j0), dtype=torch.float64, device="cuda")
        lib.fill_rhs_dev(x.data_ptr(), n, j1 - j0, j1 - j0, 42, j0)
        f.solve_dev(x.data_ptr(), n, j1 - j0)
        torch.cuda.synchronize()
        width = max(shard_range(m, g, world)[1] - shard_range(m, g, world)[0] for g in range(world))
        buf = torch.zeros((n, width), dtype=torch.float64)
        buf[:, : j1 - j0] = x.cpu()
        parts = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        if rank == 0:
            full = torch.empty((n, m), dtype=torch.float64, device="cuda")
            lib.fill_rhs_dev(full.data_ptr(), n, m, m, 42, 0)
            f.solve_dev(full.data_ptr(), n, m)
            torch.cuda.synchronize()
            got = np.concatenate([p.numpy()[:, : shard_range(m, g, world)[1] - shard_range(m, g, world)[0]]
                                  for g, p in enumerate(parts)], axis=1)
            q.put(got.tobytes() == full.cpu().numpy().tobytes())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_product_split_bitwise_on_gpu():
    mp = pytest.importorskip("torch.multiprocessing")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5)
