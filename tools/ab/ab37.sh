# fp4k B-plane kernel: one TMA input buffer (next tile streams in during pass 2) and 4 / 5 resident
# blocks per SM (variant libraries) vs the two-buffer, 3-block default
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for v in keep nb1 nb1m4 nb1m5; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "GFMatmul and (golden or shapes)" -p no:cacheprovider 2>&1 | tail -1
for c in 5 3; do for rep in 1 2; do
python bench.py --config $c --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab37.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v cfg$c',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step'])"
done; done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
