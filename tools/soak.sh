#!/bin/bash
# Parity soak on the GPU box: the seeded random sweeps of tests/test_gpu_parity.py under N
# fresh seed offsets (QADIC_SWEEP_SEED), every draw bit-exact against the CPU oracle.
# Usage: bash tools/soak.sh [first] [last]   -> gpurun_out/soak.log
F=${1:-1}; L=${2:-10}
: > gpurun_out/soak.log
for s in $(seq $F $L); do
  QADIC_SWEEP_SEED=$s python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_sweep -p no:cacheprovider -rf 2>&1 | tail -4 | sed "s/^/seed $s: /" >> gpurun_out/soak.log
done
grep -c passed gpurun_out/soak.log; grep -i "fail\|error" gpurun_out/soak.log | head -20
tail -3 gpurun_out/soak.log
