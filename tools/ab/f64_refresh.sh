# refresh the F64 lines of the round's campaign after the fold work (same commands as profile_round.sh)
O=gpurun_out/r02
mkdir -p $O
NCU="ncu --clock-control none"
B="python bench.py --no-cpu-baseline --no-variants"
$B --config 3 --engine f64 --steps 3 --warmup 3 > $O/bench_cfg3_f64.json 2>>$O/bench.err
$B --config 5 --engine f64 --steps 3 --warmup 3 > $O/bench_cfg5_f64.json 2>>$O/bench.err
python bench.py --config 5 --steps 20 --no-cpu-baseline --no-sustained > $O/bench_cfg5_variants.json 2>>$O/bench.err
T="python tools/ncu_target.py"
full() {
  $T --config $2 --engine $3 > /dev/null 2>&1 && \
  $NCU --set full --import-source on -k "regex:$4" -s 0 -c 1 -o $O/$1 -f $T --config $2 --engine $3 > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
  rm -f $O/$1.ncu-rep
}
full cfg5_f64_dmma 5 f64 dmma_gemm
full cfg5_f64fold_dmma 5 f64-fold dmma_gemm
ls -la $O
