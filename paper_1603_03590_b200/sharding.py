"""Multi-GPU plumbing for the flow path: one process per GPU, pairs sharded
across ranks, no collective on the data path.

Frame pairs are independent (the reference computes each pair's flow from
that pair alone, ``dis_flow`` pipeline.py:150-163), so the work partitions by
pair: a rank takes a contiguous block of pairs, runs it through its own
``FlowEngine`` and, when the caller wants the flows in one place, the blocks
are gathered afterwards (host side, outside any timed region).  A video
sequence of F frames has F-1 consecutive pairs; a rank owning pairs
[a, b) needs frames [a, b] — one frame overlaps with the next rank.

``torch.distributed`` is used only for plumbing: the barrier around a timed
region, the max-over-ranks of the step time, and the optional gather.
Everything here runs with the ``gloo`` backend on CPU as well as ``nccl``.
"""

from __future__ import annotations

import numpy as np


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of ``n_items`` owned by ``rank``: sizes
    differ by at most one, lower ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if n_items < 0:
        raise ValueError("n_items must be >= 0")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def sequence_frames_for_rank(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Frames [f0, f1) a rank needs for its share of the n_frames-1
    consecutive pairs of a sequence (pair i = frames i, i+1)."""
    a, b = shard_range(max(0, n_frames - 1), rank, world)
    return (a, b + 1) if b > a else (a, a)


def shard_sequence(frames: np.ndarray, rank: int, world: int):
    """(frames1, frames2) of a rank's consecutive pairs of a (F, H, W) sequence."""
    f0, f1 = sequence_frames_for_rank(frames.shape[0], rank, world)
    part = frames[f0:f1]
    return part[:-1], part[1:]


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def barrier() -> None:
    d = _dist()
    if d is not None and d.get_world_size() > 1:
        d.barrier()


def max_over_ranks(value: float, device=None) -> float:
    """The maximum of a per-rank scalar (step time) over all ranks."""
    import torch

    d = _dist()
    if d is None or d.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    d.all_reduce(t, op=d.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch

    d = _dist()
    if d is None or d.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    d.all_reduce(t, op=d.ReduceOp.SUM)
    return float(t.item())


def gather_flows(local: np.ndarray, n_items: int, dst: int = 0):
    """Collect every rank's (n_local, H, W, 2) flow block on rank ``dst`` in
    pair order (host arrays; after the computation, not part of it).
    Returns the full (n_items, H, W, 2) array on dst, None elsewhere."""
    d = _dist()
    if d is None or d.get_world_size() == 1:
        return local
    world, rank = d.get_world_size(), d.get_rank()
    blocks = [None] * world if rank == dst else None
    d.gather_object(np.ascontiguousarray(local), blocks, dst=dst)
    if rank != dst:
        return None
    out = np.concatenate([b for b in blocks if b is not None and b.shape[0] > 0]) if n_items else local[:0]
    if out.shape[0] != n_items:
        raise RuntimeError(f"gathered {out.shape[0]} flows, expected {n_items}")
    return out
