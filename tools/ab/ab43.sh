# HEAD (L2-hint code removed, epilogue trimmed) vs the campaign commit eae6cd8 on one box
nvidia-smi --query-gpu=serial --format=csv,noheader
python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py -m gpu -q -k "GFMatmul or sweep_matmul or RightCMM or fp4k or sweep_right or i8k" -p no:cacheprovider 2>&1 | tail -2
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for rep in 1 2; do for v in c0 keep; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
for c in 5 4 3; do
python bench.py --config $c --steps 30 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab43.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v cfg$c',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step'])"
done; done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
for e in i8k; do python bench.py --config 5 --engine $e --steps 30 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>>gpurun_out/ab43.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('keep $e',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step'])"; done
