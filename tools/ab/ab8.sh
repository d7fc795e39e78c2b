python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py -m gpu -x -q -p no:cacheprovider -k "f64 or F64" > gpurun_out/ab8_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab8_pytest.log
for g in 1 8 16 4; do
QADIC_F64_GROUP_M=$g timeout 600 python bench.py --config 5 --engine f64 --steps 3 --warmup 1 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab8_g$g.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab8_g$g.json').read().strip().splitlines()[-1]);print('g=$g cfg5 f64', d['ms_per_step'], d['roofline']['frac'])"
done
QADIC_F64_GROUP_M=8 timeout 600 python bench.py --config 3 --engine f64 --steps 5 --warmup 1 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab8_c3.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab8_c3.json').read().strip().splitlines()[-1]);print('g=8 cfg3 f64', d['ms_per_step'], d['roofline']['frac'])"
QADIC_F64_GROUP_M=1 timeout 600 python bench.py --config 3 --engine f64 --steps 5 --warmup 1 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab8_c3.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab8_c3.json').read().strip().splitlines()[-1]);print('g=1 cfg3 f64', d['ms_per_step'], d['roofline']['frac'])"
