o=gpurun_out/${1:-nc2}; mkdir -p $o
SP_AUTOTUNE=0 SP_GEN_WARPS=11 ncu --set full --import-source on --clock-control none -k regex:k1_fused -s 1 -c 1 -o $o/k1_cfg2 \
  python tools/profile_kernel.py --config cfg2 --shots 10002432 --what sample > $o/ncu.log 2>&1
python tools/ncu_regions.py $o/k1_cfg2.ncu-rep > $o/regions.txt 2>&1
python tools/ncu_summarize.py $o/k1_cfg2.ncu-rep > $o/summary.txt 2>&1
ncu -i $o/k1_cfg2.ncu-rep --page details --section SpeedOfLight --print-details all > $o/sol.txt 2>&1
