for r in 1 2; do
for v in 0 1; do
for c in 1 2; do QADIC_NO_PDL=$v timeout 300 python bench.py --config $c --no-cpu-baseline --no-sustained --no-redq-line --no-variants > gpurun_out/ab22.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/ab22.json').read().strip().splitlines()[-1]);print('cfg$c NO_PDL=$v', round(d['ms_per_step']*1e3,3), 'us', d['roofline']['frac'], d['roofline'].get('copy_ceiling',{}).get('us'))"; done
done
done
