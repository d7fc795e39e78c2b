# pair GEMM without the QADIC_DIAG_NOLOAD branch in the TMA producer (variant library) vs HEAD
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for rep in 1 2 3; do for v in nd keep; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
for c in 5 4; do
python bench.py --config $c --steps 30 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab44.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v cfg$c',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step']['fp4k gemm'])"
done; done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
