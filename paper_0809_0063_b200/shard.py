"""Data-parallel sharding of the hot path across GPUs (one process per GPU).

Only where the path shards naturally:
* matmul (cfg3/4/5): A is split into row blocks, B is broadcast ONCE from
  the source rank over NCCL (NVLink/NVSwitch), every rank computes its C
  rows; there is no reduction collective.
* batched polymul / dots (cfg1/cfg2): the batch is split, no collective.

The compute callable is the CUDA engine in production (bench.py) and may be
any function of (a_rows, b) -- the multi-process CPU tests drive this module
over gloo with the CPU oracle as the compute to check the partitioning and
the broadcast.
"""

from __future__ import annotations

from typing import Callable, Optional, Tuple


def row_block(n_rows: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, stop) of rank's block; blocks differ in size by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(n_rows, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def broadcast_once(b, src: int = 0, group=None):
    """Broadcast the B operand (uint8 coefficients, in place) from `src`."""
    dist = _dist()
    if dist is not None and dist.get_world_size(group) > 1:
        dist.broadcast(b, src=src, group=group)
    return b


def sharded_matmul(a_rows, b, compute: Callable, src: int = 0, group=None):
    """This rank's rows of A @ B: B broadcast once from `src`, then a local
    product; no reduction.  `b` must be allocated on every rank (filled on
    `src`)."""
    broadcast_once(b, src=src, group=group)
    return compute(a_rows, b)


def gather_rows(c_rows, group=None):
    """All-gather the row blocks (test/verification helper, equal blocks)."""
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return c_rows
    import torch

    parts = [torch.empty_like(c_rows) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, c_rows, group=group)
    return torch.cat(parts, dim=0)
