# A/B of the cfg5 plane kernels: interleaved bench runs + one ncu capture each
B="timeout 300 python bench.py --config 5 --steps 50 --no-variants --no-cpu-baseline --no-sustained --no-redq-line --no-probe"
show() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], d['ms_per_step'], d['roofline'].get('kernels_ms_per_step'))" $1 "$2"; }
for r in 1 2; do
  for cfg in "QADIC_B3=0 QADIC_A_STAGE=1" "QADIC_B3=1 QADIC_A_STAGE=0"; do
    env $cfg $B > gpurun_out/ab2.json 2>/dev/null; show gpurun_out/ab2.json "$cfg"
  done
done
python tools/ncu_target.py --config 5 > /dev/null 2>&1 && echo target-ok
NCU="ncu --clock-control none --set full --import-source on"
$NCU -k regex:planes_b4 -c 1 -o gpurun_out/ab2_b4 python tools/ncu_target.py --config 5 > /dev/null 2>&1
QADIC_B3=1 $NCU -k regex:planes_b3 -c 1 -o gpurun_out/ab2_b3 python tools/ncu_target.py --config 5 > /dev/null 2>&1
$NCU -k regex:planes_kernel -c 1 -o gpurun_out/ab2_a1 python tools/ncu_target.py --config 5 > /dev/null 2>&1
QADIC_A_STAGE=0 $NCU -k regex:planes_kernel -c 1 -o gpurun_out/ab2_a0 python tools/ncu_target.py --config 5 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
