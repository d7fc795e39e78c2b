ncu --clock-control none --set full -k regex:gemm_modp -s 2 -c 1 -o gpurun_out/ab19_conv python tools/ab/polylong_prof.py 16 > gpurun_out/ab19.log 2>&1
tail -2 gpurun_out/ab19.log
