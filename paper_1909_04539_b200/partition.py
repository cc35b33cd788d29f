"""Batch partitioner across GPUs.

Systems are independent (ref parallel.hpp:20-23), so a batch of M systems
splits into contiguous column ranges with no exchange. The split follows the
reference's worker formula j0 = M*g/G (ref parallel.cpp:53-54), with the cut
points rounded down to a multiple of `align` systems so every shard starts
on a 32-system tile (and a 16-byte boundary for TMA).
"""
from __future__ import annotations


def shard_range(m: int, rank: int, world: int, align: int = 32) -> tuple[int, int]:
    """[j0, j1) of the systems rank `rank` of `world` solves."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if m < 0 or align < 1:
        raise ValueError("bad batch size or alignment")

    def cut(g: int) -> int:
        if g >= world:
            return m
        return (m * g // world) // align * align

    return cut(rank), cut(rank + 1)


def weak_shard(m_per_gpu: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank owns a fixed-size shard of the global batch."""
    return rank * m_per_gpu, (rank + 1) * m_per_gpu
