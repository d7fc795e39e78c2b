#!/bin/bash
# Measurement campaign for one round (run on the GPU box from the repo root):
#   1. bench lines for every config / engine (no profiler attached);
#   2. the ncu launch list of the default bench command;
#   3. one `ncu --set full` capture per hot kernel of the headline (cfg5) and of cfg1-4.
# Every ncu command runs only after the same program exited 0 without ncu.
set -u
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
NCU="ncu --clock-control none"
B="python bench.py --no-cpu-baseline --no-variants"
ok=1
python bench.py > $O/bench_default.json 2>>$O/bench.err || ok=0   # the driver's default command
for c in 1 2; do $B --config $c --warmup 5 > $O/bench_cfg$c.json 2>>$O/bench.err || ok=0; done
for c in 1 2; do python bench.py --config $c --no-cpu-baseline --warmup 5 > $O/bench_cfg${c}_variants.json 2>>$O/bench.err || ok=0; done  # + the paper's forms
for c in redq pack unpack mm64 polylong polylong3 polylong1024; do python bench.py --config $c > $O/bench_$c.json 2>>$O/bench.err || ok=0; done
python bench.py --panels 4 --no-variants --no-cpu-baseline --steps 100 > $O/bench_cfg5_panels4.json 2>>$O/bench.err || ok=0
python tools/small_copy_floor.py > $O/copy_floor.jsonl 2>>$O/bench.err || ok=0
for c in 3 4 5; do
  for e in auto i8 i8k fp4 fp4k; do $B --config $c --engine $e --steps 20 --warmup 3 > $O/bench_cfg${c}_$e.json 2>>$O/bench.err || ok=0; done
done
$B --config 3 --engine f64 --steps 3 --warmup 3 > $O/bench_cfg3_f64.json 2>>$O/bench.err || ok=0
$B --config 5 --engine f64 --steps 3 --warmup 3 > $O/bench_cfg5_f64.json 2>>$O/bench.err || ok=0
python bench.py --config 5 --steps 20 --no-cpu-baseline --no-sustained > $O/bench_cfg5_variants.json 2>>$O/bench.err || ok=0
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launch_cmd.json 2>>$O/bench.err && \
  $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/launches_cfg5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
T="python tools/ncu_target.py"
full() {  # name config engine kernel-regex
  $T --config $2 --engine $3 > /dev/null 2>&1 && \
  $NCU --set full --import-source on -k "regex:$4" -s 0 -c 1 -o $O/$1 -f $T --config $2 --engine $3 > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
}
full cfg5_fp4k_gemm 5 auto gemm_modp
full cfg5_planes_b 5 auto planes_b3
full cfg5_planes_a 5 auto "planes_kernel"
full cfg5_combine 5 auto combine
full cfg3_fp4k_gemm 3 auto gemm_modp
full cfg4_fp4k_gemm 4 auto gemm_modp
full cfg1_polymul 1 auto polymul
full cfg2_gf_dot 2 auto gf_dot
full polylong polylong auto gemm_modp
full cfg5_f64_dmma 5 f64 dmma_gemm
full cfg5_f64fold_dmma 5 f64-fold dmma_gemm
python tools/mm64_profile.py > /dev/null 2>&1 && $NCU --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm_modp -c 8 --csv --log-file $O/mm64_launches.csv python tools/mm64_profile.py > /dev/null 2>&1
python bench.py --config redq --steps 3 > /dev/null 2>&1 && $NCU --set full -k regex:redq_vec -s 2 -c 1 -o $O/redq -f python bench.py --config redq --steps 3 > $O/redq.log 2>&1
ncu -i $O/redq.ncu-rep --page raw --csv > $O/redq_raw.csv 2>/dev/null
full cfg5_i8_gemm 5 i8 gemm_modp
python bench.py --config pack --steps 3 > /dev/null 2>&1 && $NCU --set full -k regex:pack_rows -s 2 -c 1 -o $O/pack -f python bench.py --config pack --steps 3 > $O/pack.log 2>&1
ncu -i $O/pack.ncu-rep --page raw --csv > $O/pack_raw.csv 2>/dev/null
ncu -i $O/pack.ncu-rep --page details --csv > $O/pack_details.csv 2>/dev/null
# measured ceilings and host-side paths on the same box
python tools/pipe_peak.py 1.0 > $O/pipe_peaks.json 2>>$O/bench.err
python bench.py --config unpack --steps 3 > /dev/null 2>&1 && $NCU --set full -k regex:unpack_rows -s 2 -c 1 -o $O/unpack -f python bench.py --config unpack --steps 3 > $O/unpack.log 2>&1
ncu -i $O/unpack.ncu-rep --page raw --csv > $O/unpack_raw.csv 2>/dev/null
REPS=200 python tools/fp4_library_peak.py 8192 residues > $O/fp4_library_ceiling.json 2>>$O/bench.err
python tools/hbm_write_probe.py > $O/hbm_write_probe.json 2>>$O/bench.err
python tools/e2e_probe.py > $O/e2e_probe.txt 2>>$O/bench.err
python tools/pageable_probe.py > $O/pageable_probe.txt 2>>$O/bench.err
# gpurun copies back at most 64 MiB: keep the CSV exports, and of the reports only the headline GEMM's
for f in $O/*.ncu-rep; do case "$f" in *cfg5_fp4k_gemm.ncu-rep) ;; *) rm -f "$f" ;; esac; done
du -sh $O
echo "bench ok=$ok"
ls -la $O | head -80
