python tools/ncu_target.py --config 5 --engine f64 --scale 2 > /dev/null 2>&1 && echo ok
ncu --clock-control none --set full --import-source on -k regex:dmma_gemm -c 1 -o gpurun_out/ab15_dmma python tools/ncu_target.py --config 5 --engine f64 --scale 2 > gpurun_out/ab15.log 2>&1
tail -2 gpurun_out/ab15.log
