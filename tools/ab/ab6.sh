for g in 16 8 4 32; do QADIC_U64_GROUP_M=$g python tools/mm64_profile.py | head -1 | sed "s/^/g=$g /"; done
for g in 16 8; do QADIC_U64_GROUP_M=$g python tools/mm64_profile.py | head -1 | sed "s/^/g=$g /"; done
timeout 300 python bench.py --config mm64 > gpurun_out/ab6_mm64.json 2>&1; tail -c 900 gpurun_out/ab6_mm64.json
