b() { env $1 timeout 300 python bench.py --config 5 --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line --no-probe > gpurun_out/ab29.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/ab29.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$1', d['ms_per_step'], r['kernels_ms_per_step'])"; }
b "QADIC_FUSE_COMBINE=0"
b "QADIC_FUSE_COMBINE=1 QADIC_FUSE_GROUP=8"
b "QADIC_FUSE_COMBINE=1 QADIC_FUSE_GROUP=4"
b "QADIC_FUSE_COMBINE=1 QADIC_FUSE_GROUP=16"
b "QADIC_FUSE_COMBINE=1 QADIC_FUSE_GROUP=32"
b "QADIC_FUSE_COMBINE=0"
