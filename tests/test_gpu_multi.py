"""The multi-GPU row-block step on one GPU: B's column panels swept against one
A (the fp4k engine keeps A's evaluation planes across the sweep) and
shard.RowBlockStep's stream/event schedule with CUDA tensors.  The collective
itself is exercised over gloo in tests/test_dist_cpu.py (one GPU per run)."""

import numpy as np
import pytest
import torch

from oracle import qadic_oracle as O
from paper_0809_0063_b200 import shard, workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,m,kd,n,panels", [(5, 300, 1000, 903, 4), (3, 257, 777, 1200, 3), (5, 64, 8192, 512, 2)])
def test_column_panel_sweep(cfg, m, kd, n, panels):
    c = W.CONFIGS[cfg]
    f = W.field_for(c)
    irr = list(c.irreducible)
    of = O.build_field(c.p, c.k, irreducible=irr, max_dot_length=c.dot_bound)
    g = W.rng(m + n)
    a = g.integers(0, c.p, (m, kd, c.k), dtype=np.uint8)
    b = g.integers(0, c.p, (kd, n, c.k), dtype=np.uint8)
    da = torch.from_numpy(a).cuda()
    outs = []
    for j, bp in enumerate(shard.split_panels(torch.from_numpy(b).cuda(), panels)):
        outs.append(f.matmul_coeffs(da, bp, engine="fp4k", col_panel=j))
    got = shard.assemble_panels(outs).cpu().numpy()
    assert np.array_equal(got, O.gf_matmul_planes(of, a, b))


def test_rowblock_step_cuda_streams():
    c = W.CONFIGS[5]
    f = W.field_for(c)
    of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
    m, kd, n = 200, 500, 777
    x = W.make_inputs(c, (m, kd, n))
    dev = torch.device("cuda", 0)
    a = torch.from_numpy(x["a"]).to(dev)
    b_panels = [p.to(dev) for p in shard.split_panels(torch.from_numpy(x["b"]), 3)]
    c_panels = [torch.zeros((m, p.shape[1], 3), dtype=torch.uint8, device=dev) for p in b_panels]

    def compute(ar, bp, cp, j):
        f.matmul_coeffs(ar, bp, out=cp, col_panel=j)

    step = shard.RowBlockStep(a, b_panels, c_panels, compute)
    want = O.gf_matmul_planes(of, x["a"], x["b"])
    for _ in range(3):
        for cp in c_panels:
            cp.zero_()
        step()
        torch.cuda.synchronize()
        assert np.array_equal(shard.assemble_panels(c_panels).cpu().numpy(), want)
