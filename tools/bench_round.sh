# Bench lines of one measurement campaign (1 GPU); JSON lines -> gpurun_out/<tag>_*.json
tag=${TAG:-r2}
run() { name=$1; shift; timeout ${TMO:-600} python bench.py "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name rc=$?"; tail -c 600 gpurun_out/${tag}_${name}.json; echo; }
for what in ${WHAT:-default panels4 cfg1 cfg2 cfg3 cfg4 polylong redq ref5}; do
  case $what in
    default) run default ;;
    panels4) run panels4 --panels 4 --no-variants --no-cpu-baseline --steps 50 ;;
    cfg1) run cfg1 --config 1 ;;
    cfg2) run cfg2 --config 2 ;;
    cfg3) run cfg3 --config 3 --no-cpu-baseline ;;
    cfg4) run cfg4 --config 4 --no-cpu-baseline ;;
    polylong) run polylong --config polylong --steps 20 ;;
    polylong3) run polylong3 --config polylong3 --steps 20 ;;
    redq) run redq --config redq ;;
    pack) run pack --config pack ;;
    unpack) run unpack --config unpack ;;
    mm64) run mm64 --config mm64 ;;
    ref5) run ref5 --impl reference --steps 2 --warmup 1 ;;
  esac
done
