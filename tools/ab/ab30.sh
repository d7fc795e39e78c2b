python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "fused or cfg5 or cfg3" 2>&1 | tail -1
QADIC_FUSE_COMBINE=1 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "cfg5" 2>&1 | tail -1
b() { env $1 timeout 300 python bench.py --config 5 --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line --no-probe > gpurun_out/ab30.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/ab30.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$1', d['ms_per_step'], r['kernels_ms_per_step'])"; }
for r in 1 2; do
b "QADIC_FUSE_COMBINE=0"
b "QADIC_FUSE_COMBINE=1"
b "QADIC_FUSE_COMBINE=1 QADIC_FUSE_ONE_LAUNCH=1"
b "QADIC_FUSE_COMBINE=1 QADIC_FUSE_GROUP=16"
done
