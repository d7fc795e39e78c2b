# fp4k GEMM epilogue: 32-bit reciprocal mod p (IMAD.HI + IMAD) vs the 64-bit multiply-high (QADIC_EPI_MOD64=1)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py -m gpu -q -k "GFMatmul or sweep_matmul or RightCMM or fp4k or sweep_right" -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2 3; do for v in 1 0; do for c in 5 3 4; do
QADIC_EPI_MOD64=$v python bench.py --config $c --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab40.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('mod64=$v cfg$c',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step'],d['clocks']['sm_mhz'])"
done; done; done
