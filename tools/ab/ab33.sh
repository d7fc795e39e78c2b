# cfg1 / cfg2 with the pre-wait L2 prefetch (no loop); cfg1 at 4 pairs per thread (variant library)
line() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[2], round(d['ms_per_step']*1e3,3), 'us frac', r['frac'], 'copy', r.get('copy_ceiling',{}).get('us'))" $1 "$2"; }
for rep in 1 2; do
for c in 1 2; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-variants > gpurun_out/ab33_c$c.json 2>gpurun_out/ab33.err
line gpurun_out/ab33_c$c.json "cfg$c"
done; done
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
cp tools/ab/libqadic_pm4.so paper_0809_0063_b200/libqadic_b200.so
for w in 0 128 256; do
QADIC_PM_WIDTH=$w timeout 600 python bench.py --config 1 --no-cpu-baseline --no-variants > gpurun_out/ab33_c1_pm4_$w.json 2>gpurun_out/ab33.err
line gpurun_out/ab33_c1_pm4_$w.json "cfg1 PM_PER=4 width=$w"
done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
