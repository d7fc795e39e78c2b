# cfg5 combine pass: 32-byte output stores (QADIC_COMBINE_ST256=1) vs 16-byte
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "GFMatmul and (golden or shapes)" -p no:cacheprovider 2>&1 | tail -2
QADIC_COMBINE_ST256=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "GFMatmul and (golden or shapes)" -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for v in 0 1; do
QADIC_COMBINE_ST256=$v python bench.py --config 5 --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab35.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('st256=$v',d['ms_per_step'],d['roofline']['kernels_ms_per_step'])"
done; done
