python -m pytest tests/test_gpu_exactness.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "f64 or F64 or engine" > gpurun_out/ab14_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab14_pytest.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 1 --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab14_c5.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab14_c5.json').read().strip().splitlines()[-1]);v=d['variants'];print('cfg5', {k:(v[k].get('ms_per_step'),v[k].get('frac'),v[k].get('error')) for k in v})"
timeout 900 python bench.py --config 5 --engine f64 --steps 3 --warmup 1 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab14_c5f64.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab14_c5f64.json').read().strip().splitlines()[-1]);print('cfg5 f64', d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('kernels_ms_per_step'))"
