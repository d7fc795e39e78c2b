"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the qadic hot path.

Nothing in the product package (`paper_0809_0063_b200`) may import, call or
link anything under this directory.  Only `tests/`, `__graft_entry__.smoke()`
and the `cpu_baseline` / `--impl reference` legs of `bench.py` use it, and
only as the checker or as the timed CPU baseline, never as the measured path.

Contents
--------
qadic_oracle.py   numpy restatement of the reference algorithm (citations
                  file:line into /root/reference/pkg/src/qadic)
oracle_kernels.c  plain-C restatement of the reference's native kernels
                  (src/_kernels/_speed.pyx), OpenMP over rows; built into
                  oracle/liboracle.so by oracle/Makefile
_ref/             (git-ignored) the reference's own Cython kernel module
                  `_speed` compiled from /root/reference by `make -C oracle ref`

Parity pinning: the restatement is checked against golden vectors generated
by importing the reference package in the build container
(tests/golden/make_golden.py) and, when oracle/_ref is built, against the
reference's compiled kernels directly (tests/test_oracle.py).
"""
