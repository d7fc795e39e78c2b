# cfg1 / cfg2 with the pre-wait L2 prefetch: virtual-block iterations per block (co-resident back-to-back calls) and block width
QADIC_PM_ITERS=2 QADIC_GD_ITERS=2 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "polymul or Polymul or GFDot or gf_dot or fgdp or cfg1 or cfg2" > gpurun_out/ab32_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab32_pytest.log
line() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[2], round(d['ms_per_step']*1e3,3), 'us frac', r['frac'], 'copy', r.get('copy_ceiling',{}).get('us'))" $1 "$2"; }
for it in 1 2 3 4; do for w in 0 128 160; do
QADIC_PM_ITERS=$it QADIC_PM_WIDTH=$w timeout 600 python bench.py --config 1 --no-cpu-baseline --no-variants > gpurun_out/ab32_c1_${it}_${w}.json 2>gpurun_out/ab32.err
line gpurun_out/ab32_c1_${it}_${w}.json "cfg1 iters=$it width=$w"
done; done
for it in 1 2 3 4; do for w in 256 128; do
QADIC_GD_ITERS=$it QADIC_GD_WIDTH=$w timeout 600 python bench.py --config 2 --no-cpu-baseline --no-variants > gpurun_out/ab32_c2_${it}_${w}.json 2>gpurun_out/ab32.err
line gpurun_out/ab32_c2_${it}_${w}.json "cfg2 iters=$it width=$w"
done; done
