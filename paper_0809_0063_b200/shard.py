"""Data-parallel sharding of the hot path across GPUs (one process per GPU).

Only where the path shards naturally:
* matmul (cfg3/4/5): C is split into an R x Cc grid of blocks (`grid2d`):
  rank (i, j) computes C[rows_i, cols_j] = A[rows_i] B[:, cols_j] with no
  collective in the step.  B reaches the ranks by ONE broadcast over NCCL
  (NVLink/NVSwitch) at set-up, after which each rank keeps its column block.
  The grid (rather than row blocks only) splits the per-call operand
  conversion of B as well as A's: with row blocks every rank would re-convert
  all of B (the evaluation planes), which caps 8-GPU efficiency near 60%;
  a 2 x 4 grid leaves A/2 + B/4 per rank.  R = 1 gives plain row blocks of C^T
  (column blocks), Cc = 1 plain row blocks.
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


def grid2d(world: int) -> Tuple[int, int]:
    """(R, Cc) with R * Cc = world: R the largest divisor <= sqrt(world), so the
    B (column) side gets the finer split -- 2 -> (1, 2), 4 -> (2, 2), 8 -> (2, 4)."""
    if world < 1:
        raise ValueError("bad world")
    r = 1
    for d in range(1, int(world ** 0.5) + 1):
        if world % d == 0:
            r = d
    return r, world // r


def block2d(m: int, n: int, world: int, rank: int) -> Tuple[int, int, int, int]:
    """(r0, r1, c0, c1): rank's block of an m x n output on the grid2d(world) grid
    (rank = i * Cc + j)."""
    if not 0 <= rank < world:
        raise ValueError("bad world/rank")
    R, C = grid2d(world)
    i, j = divmod(rank, C)
    r0, r1 = row_block(m, R, i)
    c0, c1 = row_block(n, C, j)
    return r0, r1, c0, c1


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


def gather_blocks(c_block, m: int, n: int, group=None):
    """Assemble the full m x n (x k) output from every rank's grid2d block
    (test/verification helper; blocks are padded to the largest for the
    all-gather)."""
    dist = _dist()
    world = dist.get_world_size(group) if dist is not None else 1
    if world == 1:
        return c_block
    import torch

    shapes = [block2d(m, n, world, r) for r in range(world)]
    hmax = max(r1 - r0 for r0, r1, _, _ in shapes)
    wmax = max(c1 - c0 for _, _, c0, c1 in shapes)
    pad = torch.zeros((hmax, wmax) + tuple(c_block.shape[2:]), dtype=c_block.dtype, device=c_block.device)
    pad[:c_block.shape[0], :c_block.shape[1]] = c_block
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = torch.empty((m, n) + tuple(c_block.shape[2:]), dtype=c_block.dtype, device=c_block.device)
    for (r0, r1, c0, c1), part in zip(shapes, parts):
        out[r0:r1, c0:c1] = part[:r1 - r0, :c1 - c0]
    return out


def gather_rows(c_rows, group=None):
    """All-gather the row blocks (test/verification helper, equal blocks)."""
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return c_rows
    import torch

    parts = [torch.empty_like(c_rows) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, c_rows, group=group)
    return torch.cat(parts, dim=0)
