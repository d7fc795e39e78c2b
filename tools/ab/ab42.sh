# bisect of the fp4k GEMM time over the engine_tc.cu commits after the campaign commit (variant libraries)
nvidia-smi --query-gpu=serial --format=csv,noheader
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for rep in 1 2; do for v in c0 c1 c3 c4 c5 c6 keep; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
for c in 5 4; do
python bench.py --config $c --steps 30 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab42.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v cfg$c',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step']['fp4k gemm'])"
done; done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
