o=gpurun_out/${1:-nk5}; mkdir -p $o
ncu --set full --import-source on --clock-control none -k regex:k5_columns -s 1 -c 1 -o $o/k5 python tools/k5_time.py 0.5 1e-3 > $o/ncu.log 2>&1
python tools/ncu_summarize.py $o/k5.ncu-rep > $o/summary.txt 2>&1
ncu -i $o/k5.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[-1]
for k,x in zip(h,v):
    if k in ('lts__t_sector_hit_rate.pct','dram__bytes_read.sum','l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum','lts__t_bytes.sum','gpu__time_duration.sum'): print(k,x)
" > $o/raw.txt 2>&1
