"""B200-native packed small-field arithmetic (arXiv 0809.0063), drop-in for
the reference package `qadic` on its hot path.

    import paper_0809_0063_b200 as qadic

exposes the same module names and signatures as the reference
(/root/reference/pkg/src/qadic/__init__.py:28-57): params, dqt, redq, fdiv,
polymul, gfext, cmm, _kernels.  Every array operation runs as a hand-written
sm_100a CUDA kernel in libqadic_b200.so (C ABI: include/qadic_b200.h):

  DQT pack/unpack          qadic_pack_rows_u8 / in-register packing
  packed products          tcgen05 INT8 plane GEMM | FP64 DMMA word GEMM,
                           batched FP64 polymul / GF dots
  REDQ                     FP64 reciprocal division + 32-bit digit trick
  GF(p^k) fold             L/H tables in shared memory | folded B planes

Additive batched APIs the benchmark configs use: polymul.polymul_fqt_batch
(cfg1), GFqField.fgdp_batch_coeffs (cfg2), GFqField.matmul_coeffs (cfg3,
cfg5), cmm.right_cmm (cfg4).
"""

from . import _kernels, bench, cli, cmm, costs, dqt, fdiv, gfext, params, polymul, redq, shard, workloads
from ._native import launch_count
from .errors import (
    DimensionMismatch,
    Infeasible,
    MemoryBudgetExceeded,
    NoGeneratorFound,
    NotIrreducible,
    PackOverflow,
    ParamsViolation,
    QadicError,
    TooLarge,
)
from .params import (
    FullCompressionParams,
    PackingParams,
    cmm_params,
    delayed_bound,
    dqt_params,
    fqt_params,
    full_cmm_params,
)

__version__ = "0.1.0"

kernel_backend = _kernels.get_backend
