# cfg1 byte-lane form: pairs per thread / resident blocks / early stores (variant libraries), block width
line() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[2], round(d['ms_per_step']*1e3,3), 'us frac', r['frac'], 'copy', r.get('copy_ceiling',{}).get('us'))" $1 "$2"; }
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "TestPolymul" -p no:cacheprovider 2>&1 | tail -3
cp paper_0809_0063_b200/libqadic_b200.so /tmp/keep.so
for rep in 1 2; do
for v in keep pm4 early pm4early pm8b6 pm16; do
if [ $v = keep ]; then cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so; else cp tools/ab/libqadic_$v.so paper_0809_0063_b200/libqadic_b200.so; fi
for w in 0 128 256; do
QADIC_PM_WIDTH=$w timeout 600 python bench.py --config 1 --no-cpu-baseline --no-variants --no-probe > gpurun_out/ab34_${v}_$w.json 2>gpurun_out/ab34.err
line gpurun_out/ab34_${v}_$w.json "cfg1 $v width=$w"
done; done; done
cp /tmp/keep.so paper_0809_0063_b200/libqadic_b200.so
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "TestPolymul" -p no:cacheprovider 2>&1 | tail -3
