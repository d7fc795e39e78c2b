set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py -m gpu -x -q -p no:cacheprovider > gpurun_out/ab1_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab1_pytest.log
for v in 0 1; do
QADIC_B3=$v timeout 300 python bench.py --config 5 --steps 50 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab1_cfg5_b3$v.json 2>gpurun_out/ab1_cfg5_b3$v.err
python -c "import json;d=json.loads(open('gpurun_out/ab1_cfg5_b3$v.json').read().strip().splitlines()[-1]);print('B3=$v', d['ms_per_step'], d['roofline'].get('kernels_ms_per_step'))"
QADIC_B3=$v timeout 300 python bench.py --config 3 --steps 50 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab1_cfg3_b3$v.json 2>gpurun_out/ab1_cfg3_b3$v.err
python -c "import json;d=json.loads(open('gpurun_out/ab1_cfg3_b3$v.json').read().strip().splitlines()[-1]);print('cfg3 B3=$v', d['ms_per_step'], d['roofline'].get('kernels_ms_per_step'))"
done
for nb in 3 4; do
QADIC_B4_NBUF=$nb timeout 300 python bench.py --config 5 --steps 50 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe > gpurun_out/ab1_cfg5_nb$nb.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab1_cfg5_nb$nb.json').read().strip().splitlines()[-1]);print('NB=$nb', d['ms_per_step'], d['roofline'].get('kernels_ms_per_step'))"
done
