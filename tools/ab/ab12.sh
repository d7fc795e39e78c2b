python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py tests/test_gpu_domain.py -m gpu -x -q -p no:cacheprovider -k "f64 or F64 or cmm or CMM" > gpurun_out/ab12_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab12_pytest.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 1 --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab12_c5.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab12_c5.json').read().strip().splitlines()[-1]);v=d['variants'];print('cfg5', {k:(v[k].get('ms_per_step'),v[k].get('frac'),v[k].get('error')) for k in v})"
timeout 600 python bench.py --config 3 --engine f64 --steps 5 --warmup 1 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab12_c3.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab12_c3.json').read().strip().splitlines()[-1]);print('cfg3 f64', d['ms_per_step'], d['roofline']['frac'])"
timeout 600 python bench.py --config 4 --engine f64 --steps 3 --warmup 1 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab12_c4.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab12_c4.json').read().strip().splitlines()[-1]);print('cfg4 f64', d['ms_per_step'], d['roofline']['frac'])"
