# cfg5 A-plane and combine kernels: more resident blocks per SM through launch bounds (variant libraries)
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for v in keep m5 m6 m8 keep m5 m6; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
for c in 5 3; do
python bench.py --config $c --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab39.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v cfg$c',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step'])"
done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
