# (historical: the switches were removed again, see DESIGN 9) fp4k GEMM: L2 eviction hints on the operand TMA loads (QADIC_L2_HINT=ab: 1 evict_first, 2 evict_last,
# 3 evict_normal) and streaming plane stores (QADIC_STREAM_OUT=1): step time and the GEMM's DRAM bytes
run() { # env...
  env "$@" python bench.py --config 5 --steps 50 --no-cpu-baseline --no-variants --no-sustained --no-redq-line 2>gpurun_out/ab36.err | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$*',round(d['ms_per_step'],4),d['roofline']['kernels_ms_per_step'])"
}
dram() {
  env "$@" ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemm_modp -s 0 -c 1 --csv python tools/ncu_target.py --config 5 --engine auto 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v tag="$*" '{print tag, $(NF-2), $(NF-1), $NF}'
}
QADIC_L2_HINT=12 QADIC_STREAM_OUT=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "GFMatmul and (golden or shapes)" -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
for h in 0 12 21 22 2 20 32; do run QADIC_L2_HINT=$h; done
run QADIC_L2_HINT=0 QADIC_STREAM_OUT=1
run QADIC_L2_HINT=12 QADIC_STREAM_OUT=1
run QADIC_L2_HINT=22 QADIC_STREAM_OUT=1
done
python tools/ncu_target.py --config 5 --engine auto > /dev/null 2>&1
for h in 0 12 22; do dram QADIC_L2_HINT=$h; dram QADIC_L2_HINT=$h QADIC_STREAM_OUT=1; done
