# cfg5 A-plane and combine kernels: resident blocks per SM capped by unused dynamic shared memory
run() { env "$@" python bench.py --config 5 --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab38.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());k=d['roofline']['kernels_ms_per_step'];print('$*',round(d['ms_per_step'],4),'A',k['fp4k planes A'],'combine',k['fp4k combine'])"; }
for rep in 1 2; do
run QADIC_PA_PAD=0
for pad in 30000 40000 52000 70000 110000; do run QADIC_PA_PAD=$pad QADIC_COMBINE_PAD=$pad; done
done
