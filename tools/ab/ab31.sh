# L2 prefetch ahead of griddepcontrol.wait in the single-wave batched kernels (cfg1, cfg2) and the copy ceiling
set -x
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "polymul or Polymul or GFDot or gf_dot or fgdp or cfg1 or cfg2" > gpurun_out/ab31_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab31_pytest.log
for rep in 1 2; do
for v in 0 1; do
for c in 1 2; do
QADIC_PDL_PREFETCH=$v timeout 600 python bench.py --config $c --no-cpu-baseline --no-variants > gpurun_out/ab31_c${c}_pf$v.json 2>gpurun_out/ab31_c${c}_pf$v.err
python -c "import json;d=json.loads(open('gpurun_out/ab31_c${c}_pf$v.json').read().strip().splitlines()[-1]);r=d['roofline'];print('cfg$c PF=$v', d['ms_per_step'], r['frac'], r.get('copy_ceiling'))"
done
done
done
