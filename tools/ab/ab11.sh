python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "GFDot or gf_dot or fgdp or cfg2" > gpurun_out/ab11_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab11_pytest.log
timeout 600 python bench.py --config 2 --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab11_c2.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab11_c2.json').read().strip().splitlines()[-1]);v=d['variants'];print('cfg2', d['ms_per_step'], d['roofline']['frac'], {k:(v[k]['ms_per_step'],v[k]['frac']) for k in v})"
