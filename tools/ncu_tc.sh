o=gpurun_out/${1:-ntc}; mkdir -p $o
ncu --set full --import-source on --clock-control none -k regex:k6_tc_product -s 1 -c 1 -o $o/k6 python tools/tc_time.py 65536 > $o/ncu.log 2>&1
python tools/ncu_summarize.py $o/k6.ncu-rep > $o/summary.txt 2>&1
python tools/ncu_regions.py $o/k6.ncu-rep > $o/regions.txt 2>&1
