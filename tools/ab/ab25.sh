b() { timeout 300 python bench.py --config 1 --no-cpu-baseline --no-sustained --no-redq-line --no-variants > gpurun_out/ab25.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/ab25.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$1', round(d['ms_per_step']*1e3,3), 'us', r['frac'], r.get('copy_ceiling',{}).get('us'))"; }
b PER8; b PER8
cp tools/ab/pm4/libqadic_b200.so paper_0809_0063_b200/libqadic_b200.so
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cfg1 or Polymul or polymul" 2>&1 | tail -1
b PER4; b PER4
