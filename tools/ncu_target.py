"""Small deterministic driver for ncu: runs `--reps` steps of one config's
hot path (reduced shapes allowed) through the public API.  Used as

    python tools/ncu_target.py --config 5 && \
    ncu --set full -k regex:gemm -c 1 -o gpurun_out/prof python tools/ncu_target.py --config 5
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="5", help="1..5, or polylong / polylong3")
    ap.add_argument("--engine", default="auto")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--scale", type=int, default=1, help="divide every dimension")
    args = ap.parse_args()
    import torch

    import paper_0809_0063_b200 as Q
    from paper_0809_0063_b200 import workloads as W

    if args.config.startswith("polylong"):
        import numpy as np

        from paper_0809_0063_b200.params import fqt_params

        prm = fqt_params(3, 3 if args.config == "polylong3" else 1)
        g = np.random.default_rng(7)
        a = torch.from_numpy(g.integers(0, 3, (16, 16384 // args.scale), dtype=np.uint8)).cuda()
        b = torch.from_numpy(g.integers(0, 3, (16, 16384 // args.scale), dtype=np.uint8)).cuda()
        for _ in range(args.reps):
            Q.polymul.polymul_fqt_long_batch(a, b, prm)
        torch.cuda.synchronize()
        print("ok")
        return
    c = W.CONFIGS[int(args.config)]
    shape = W.scaled_shape(c, args.scale)
    x = {k: torch.from_numpy(v).cuda() for k, v in W.make_inputs(c, shape).items()}
    for _ in range(args.reps):
        if c.cfg == 1:
            Q.polymul.polymul_fqt_batch(x["a"], x["b"], W.params_for(c))
        elif c.cfg == 2:
            W.field_for(c).fgdp_batch_coeffs(x["v1"], x["v2"])
        elif c.cfg in (3, 5):
            W.field_for(c).matmul_coeffs(x["a"], x["b"], engine=args.engine)
        else:
            prm = Q.cmm_params(3, shape[0], strict=True)
            Q.cmm.right_cmm(x["a"], Q.cmm.compress_rows(x["a"], prm), engine=args.engine)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
