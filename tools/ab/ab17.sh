python tools/ab/polylong_prof.py 256 > /dev/null 2>&1 && echo ok
ncu --clock-control none --set full --import-source on -k regex:gemm_modp -s 2 -c 1 -o gpurun_out/ab17_tz python tools/ab/polylong_prof.py 256 > gpurun_out/ab17.log 2>&1
tail -2 gpurun_out/ab17.log
