"""Data-parallel sharding of the hot path across GPUs (one process per GPU).

Only where the path shards naturally (the sharded operation is
GFqField.matmul / right_cmm, reference src/gfext.py:311-345, src/cmm.py:244-276):

* matmul (cfg3/4/5), the default partition (`RowBlockStep`): rank r owns the
  row block A[rows_r] (resident) and computes C[rows_r] = A[rows_r] B.  B lives
  on the source rank in column-panel-major order and is broadcast over NCCL
  (NVLink / NVSwitch) INSIDE every step, one column panel at a time on a
  communication stream; the product of panel j starts on the compute stream as
  soon as panel j has landed, so the broadcast of panel j+1 overlaps the
  product of panel j.  No reduction collective: each rank's C rows are final.
  C is kept per panel ([rows, N_j, k] blocks).
* the 2-D grid option (`grid2d` / `block2d`): rank (i, j) computes
  C[rows_i, cols_j] with A[rows_i] and B[:, cols_j] resident after ONE
  broadcast at set-up -- no collective in a step.  It splits the per-step
  operand conversion of B as well as A's (with row blocks every rank converts
  all of B), at the price of B never moving inside the step.
* batched polymul / dots (cfg1/cfg2): the batch is split, no collective.

The compute callable is the CUDA engine in production (bench.py) and may be
any function (a_rows, b_panel, out) -- the multi-process CPU tests drive the
same step over gloo with the CPU oracle as the compute.
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


def panel_bounds(n: int, panels: int):
    """[(j0, j1)] of `panels` near-equal column panels of an n-column operand."""
    panels = max(1, min(panels, n)) if n else 1
    return [row_block(n, panels, j) for j in range(panels)]


def split_panels(b, panels: int):
    """Column panels of B [K, N, ...] as contiguous copies (the source rank's
    panel-major layout; works for numpy arrays and torch tensors)."""
    bounds = panel_bounds(b.shape[1], panels)
    if hasattr(b, "contiguous"):
        return [b[:, j0:j1].contiguous() for j0, j1 in bounds]
    import numpy as np

    return [np.ascontiguousarray(b[:, j0:j1]) for j0, j1 in bounds]


class RowBlockStep:
    """One step of the row-block sharded product C[rows_r] = A[rows_r] @ B.

    b_panels: B's column panels, allocated on every rank and filled on `src`
    (the other ranks' contents are overwritten by the broadcast every step).
    c_panels: this rank's output blocks, c_panels[j] = A[rows_r] @ b_panels[j].
    compute(a_rows, b_panel, out, j): the local product of panel j (writes
    `out`; j lets the engine keep A's converted operand across the sweep).

    On CUDA tensors the broadcasts run on a dedicated stream (NCCL async ops,
    one event per panel) and the compute stream waits on each panel's event
    only, so panel j+1 travels while panel j is multiplied.  On CPU tensors
    (gloo) the same schedule runs synchronously.  `stage(j)` (optional) runs
    on the source rank before panel j is sent -- the e2e step uses it to copy
    the panel in from host memory."""

    def __init__(self, a_rows, b_panels, c_panels, compute: Callable, src: int = 0, group=None,
                 stage: Optional[Callable] = None):
        if len(b_panels) != len(c_panels):
            raise ValueError("one output block per B panel")
        self.a_rows, self.b_panels, self.c_panels = a_rows, list(b_panels), list(c_panels)
        self.compute, self.src, self.group, self.stage = compute, src, group, stage
        dist = _dist()
        self.world = dist.get_world_size(group) if dist is not None else 1
        self.rank = dist.get_rank(group) if dist is not None else 0
        self.cuda = getattr(a_rows, "is_cuda", False)
        self.comm = None
        if self.cuda:
            import torch

            self.comm = torch.cuda.Stream(device=a_rows.device)

    def bytes_broadcast(self) -> int:
        return sum(b.numel() * b.element_size() for b in self.b_panels) if self.world > 1 else 0

    def __call__(self):
        dist = _dist()
        if not self.cuda:
            for j, (bp, cp) in enumerate(zip(self.b_panels, self.c_panels)):
                if self.stage is not None and self.rank == self.src:
                    self.stage(j)
                if dist is not None and self.world > 1:
                    dist.broadcast(bp, src=self.src, group=self.group)
                self.compute(self.a_rows, bp, cp, j)
            return self.c_panels
        import torch

        cur = torch.cuda.current_stream()
        self.comm.wait_stream(cur)  # the previous step's products no longer read the panel buffers
        events = []
        with torch.cuda.stream(self.comm):
            for j, bp in enumerate(self.b_panels):
                if self.stage is not None and self.rank == self.src:
                    self.stage(j)
                if dist is not None and self.world > 1:
                    dist.broadcast(bp, src=self.src, group=self.group, async_op=True).wait()
                ev = torch.cuda.Event()
                ev.record(self.comm)
                events.append(ev)
        for j, (ev, bp, cp) in enumerate(zip(events, self.b_panels, self.c_panels)):
            cur.wait_event(ev)
            self.compute(self.a_rows, bp, cp, j)
        return self.c_panels


def assemble_panels(c_panels, axis: int = 1):
    """Concatenate per-panel output blocks along the column axis."""
    if hasattr(c_panels[0], "contiguous"):
        import torch

        return torch.cat(list(c_panels), dim=axis)
    import numpy as np

    return np.concatenate(list(c_panels), axis=axis)
