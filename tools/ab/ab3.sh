python -m pytest tests/test_gpu_exactness.py -m gpu -x -q -p no:cacheprovider -k "f64" > gpurun_out/ab3_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab3_pytest.log
for mode in 0 1 2; do
QADIC_F64_FOLD_MODE=$mode timeout 600 python bench.py --config 5 --steps 20 --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab3_m$mode.json 2>gpurun_out/ab3_m$mode.err
python -c "import json;d=json.loads(open('gpurun_out/ab3_m$mode.json').read().strip().splitlines()[-1]);v=d['variants'];print('mode $mode', {k:(v[k]['ms_per_step'],v[k]['frac']) for k in v})"
done
