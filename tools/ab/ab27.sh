python -m pytest tests/test_gpu_exactness.py -m gpu -x -q -p no:cacheprovider -k "f64" 2>&1 | tail -1
timeout 900 python bench.py --config 5 --steps 3 --warmup 1 --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab27.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab27.json').read().strip().splitlines()[-1]);v=d['variants'];print('cfg5', {k:(v[k].get('ms_per_step'),v[k].get('frac'),v[k].get('error')) for k in v})"
