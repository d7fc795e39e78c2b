# FP4 GEMM instantiations without the (int8-only) convolution / Toeplitz code paths vs the previous build
python -m pytest tests/test_gpu_parity.py tests/test_gpu_domain.py tests/test_gpu_exactness.py -m gpu -q -k "GFMatmul or sweep_matmul or RightCMM or long or toeplitz or sweep_long or matmul_u64 or i8k or fp4" -p no:cacheprovider 2>&1 | tail -2
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for rep in 1 2 3; do for v in prev keep; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
for c in 5 4 3; do
python bench.py --config $c --steps 30 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab46.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v cfg$c',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step']['fp4k gemm'])"
done; done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
