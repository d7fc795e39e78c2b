import time, numpy as np, sys
sys.path.insert(0, "/root/repo")
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import workloads as W
for cfg in (3, 5):
    c = W.CONFIGS[cfg]
    of = O.build_field(c.p, c.k, irreducible=list(c.irreducible), max_dot_length=c.dot_bound)
    x = W.make_inputs(c)
    t = time.perf_counter(); r = O.gf_matmul_planes(of, x["a"], x["b"]); print(cfg, "plane oracle full: %.1f s" % (time.perf_counter() - t), flush=True)
c = W.CONFIGS[4]; a = W.make_inputs(c)["a"]
t = time.perf_counter(); r = O.modmatmul_planes(a, a, 3); print(4, "full: %.1f s" % (time.perf_counter() - t), flush=True)
