# fused-combine GEMM epilogue (cfg3): offset add compiled out for non-negative representatives vs the previous build
python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py -m gpu -q -k "GFMatmul or sweep_matmul or fused" -p no:cacheprovider 2>&1 | tail -2
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for rep in 1 2 3; do for v in prev keep; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
python bench.py --config 3 --steps 30 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab45.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v cfg3',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step'])"
done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
