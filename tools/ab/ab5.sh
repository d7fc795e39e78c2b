python tools/mm64_profile.py > gpurun_out/ab5_mm64.txt 2>&1; cat gpurun_out/ab5_mm64.txt
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_modp -c 16 --csv python tools/mm64_profile.py > gpurun_out/ab5_ncu.csv 2>&1
grep -v "^==" gpurun_out/ab5_ncu.csv | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d.get('ID'), d.get('Metric Name'), d.get('Metric Value'))
" | tail -60
