"""World-size-2 gloo tests (CPU) of the multi-GPU partitioning: row blocks
of A, B broadcast once from rank 0, no reduction; batch sharding for the
batched configs.  The compute is the CPU oracle here (the CUDA engine on
the GPU box)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0809_0063_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import qadic_oracle as O
        from paper_0809_0063_b200 import workloads as W

        if kind == "gf":
            c = W.CONFIGS[5]
            x = W.make_inputs(c, (37, 50, 23))  # ragged: 37 rows over 2 ranks
            f = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
            s0, s1 = shard.row_block(37, world, rank)
            a_rows = torch.from_numpy(x["a"][s0:s1])
            b = torch.from_numpy(x["b"].copy()) if rank == 0 else torch.zeros(x["b"].shape, dtype=torch.uint8)
            c_rows = shard.sharded_matmul(
                a_rows, b, lambda ar, bb: torch.from_numpy(O.gf_matmul_folded(f, ar.numpy(), bb.numpy(), 9)))
            ok_b = torch.equal(b, torch.from_numpy(x["b"]))
            full = O.gf_matmul_planes(f, x["a"], x["b"])
            ok = ok_b and np.array_equal(c_rows.numpy(), full[s0:s1])
        elif kind == "cmm":
            c = W.CONFIGS[4]
            a = W.make_inputs(c, (64,))["a"]
            s0, s1 = shard.row_block(64, world, rank)
            full_t = torch.from_numpy(a.copy()) if rank == 0 else torch.zeros(a.shape, dtype=torch.uint8)
            shard.broadcast_once(full_t)
            rows = full_t[s0:s1]
            c_rows = torch.from_numpy(O.right_cmm(rows.numpy(), full_t.numpy(), 3, 17, 2))
            gathered = shard.gather_rows(c_rows)
            ok = np.array_equal(gathered.numpy(), O.modmatmul_planes(a, a, 3))
        elif kind == "grid":  # 2-D block grid: B broadcast once at set-up, no collective per product
            c = W.CONFIGS[5]
            m, kd, n = 37, 50, 45
            x = W.make_inputs(c, (m, kd, n))
            f = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
            b = torch.from_numpy(x["b"].copy()) if rank == 0 else torch.zeros(x["b"].shape, dtype=torch.uint8)
            shard.broadcast_once(b)
            r0, r1, c0, c1 = shard.block2d(m, n, world, rank)
            blk = torch.from_numpy(O.gf_matmul_planes(f, x["a"][r0:r1], b.numpy()[:, c0:c1]))
            full = shard.gather_blocks(blk, m, n)
            ok = np.array_equal(full.numpy(), O.gf_matmul_planes(f, x["a"], x["b"]))
        elif kind == "grid_cmm":  # A^2 mod 3 on the grid: rank needs A rows_i and A cols_j
            c = W.CONFIGS[4]
            n = 40
            a = W.make_inputs(c, (n,))["a"]
            r0, r1, c0, c1 = shard.block2d(n, n, world, rank)
            blk = torch.from_numpy(O.right_cmm(a[r0:r1], np.ascontiguousarray(a[:, c0:c1]), 3, 17, 2))
            full = shard.gather_blocks(blk, n, n)
            ok = np.array_equal(full.numpy(), O.modmatmul_planes(a, a, 3))
        elif kind == "rowpanel":  # the bench's default step: B panels broadcast inside the step
            c = W.CONFIGS[5]
            m, kd, n = 37, 50, 45
            x = W.make_inputs(c, (m, kd, n))
            f = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
            r0, r1 = shard.row_block(m, world, rank)
            bounds = shard.panel_bounds(n, 3)
            if rank == 0:
                b_panels = [torch.from_numpy(p) for p in shard.split_panels(x["b"], 3)]
            else:
                b_panels = [torch.zeros((kd, j1 - j0, 3), dtype=torch.uint8) for j0, j1 in bounds]
            c_panels = [torch.zeros((r1 - r0, j1 - j0, 3), dtype=torch.uint8) for j0, j1 in bounds]

            def compute(ar, bp, cp, j=0):
                cp.copy_(torch.from_numpy(O.gf_matmul_folded(f, ar.numpy(), bp.numpy(), 9)))

            stepper = shard.RowBlockStep(torch.from_numpy(x["a"][r0:r1]), b_panels, c_panels, compute)
            ok = True
            for _ in range(2):  # two steps: the second re-broadcasts into the same buffers
                for bp in (b_panels if rank else []):
                    bp.zero_()
                stepper()
                mine = shard.assemble_panels([cp.numpy() for cp in c_panels])
                ok = ok and np.array_equal(mine, O.gf_matmul_planes(f, x["a"], x["b"])[r0:r1])
            ok = ok and stepper.bytes_broadcast() == x["b"].nbytes
        elif kind == "rowpanel_cmm":  # A^2 mod 3: rank 0 sends A's column panels as B
            c = W.CONFIGS[4]
            n = 40
            a = W.make_inputs(c, (n,))["a"]
            r0, r1 = shard.row_block(n, world, rank)
            bounds = shard.panel_bounds(n, 4)
            b_panels = [torch.from_numpy(p) for p in shard.split_panels(a, 4)] if rank == 0 else \
                [torch.zeros((n, j1 - j0), dtype=torch.uint8) for j0, j1 in bounds]
            c_panels = [torch.zeros((r1 - r0, j1 - j0), dtype=torch.uint8) for j0, j1 in bounds]

            def compute(ar, bp, cp, j=0):
                cp.copy_(torch.from_numpy(O.right_cmm(ar.numpy(), bp.numpy(), 3, 17, 2)))

            shard.RowBlockStep(torch.from_numpy(a[r0:r1]), b_panels, c_panels, compute)()
            rows = torch.from_numpy(shard.assemble_panels([cp.numpy() for cp in c_panels]))
            ok = np.array_equal(rows.numpy(), O.modmatmul_planes(a, a, 3)[r0:r1])
        else:  # batch sharding, no collective
            c = W.CONFIGS[1]
            x = W.make_inputs(c, (1001,))
            s0, s1 = shard.row_block(1001, world, rank)
            got = O.polymul_batch(x["a"][s0:s1], x["b"][s0:s1], 3, 5)
            ok = np.array_equal(got, O.polymul_batch(x["a"], x["b"], 3, 5)[s0:s1])
        result_q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _spawn(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("kind", ["gf", "cmm", "batch", "grid", "grid_cmm", "rowpanel", "rowpanel_cmm"])
def test_world2(kind):
    assert _spawn(2, kind) == {0: True, 1: True}


@pytest.mark.parametrize("kind", ["grid", "grid_cmm"])
def test_world4_grid(kind):
    """2 x 2 block grid over four gloo ranks."""
    assert _spawn(4, kind) == {r: True for r in range(4)}


def test_grid2d_blocks_tile_the_output():
    for world in (1, 2, 3, 4, 6, 8):
        R, C = shard.grid2d(world)
        assert R * C == world and R <= C
        for m, n in ((8192, 8192), (37, 45), (5, 3)):
            cover = np.zeros((m, n), np.int32)
            for r in range(world):
                r0, r1, c0, c1 = shard.block2d(m, n, world, r)
                cover[r0:r1, c0:c1] += 1
            assert (cover == 1).all()
    assert shard.grid2d(8) == (2, 4) and shard.grid2d(4) == (2, 2) and shard.grid2d(2) == (1, 2)


def test_row_block_partition():
    for n in (1, 7, 8192, 16384, 37):
        for w in (1, 2, 3, 4, 8):
            spans = [shard.row_block(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


@pytest.mark.parametrize("kind", ["rowpanel", "rowpanel_cmm"])
def test_world4_rowpanel(kind):
    """the bench's default multi-GPU step over four gloo ranks (ragged row blocks)."""
    assert _spawn(4, kind) == {r: True for r in range(4)}


def test_panel_bounds_and_split():
    for n, p in ((8192, 4), (45, 3), (5, 8), (1, 4)):
        b = shard.panel_bounds(n, p)
        assert b[0][0] == 0 and b[-1][1] == n and len(b) == min(p, n)
        arr = np.arange(7 * n).reshape(7, n)
        assert np.array_equal(shard.assemble_panels(shard.split_panels(arr, p)), arr)


def test_bench_gpus_flag_never_silently_single(tmp_path):
    """`bench.py --gpus 2` on a box with fewer GPUs must fail loudly, not measure one."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "--gpus 2" in r.stderr
    env["WORLD_SIZE"] = "4"
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=4" in r.stderr
