o=gpurun_out/${1:-nd}; mkdir -p $o
SP_DEBUG_MODE=2 SP_AUTOTUNE=0 SP_GEN_WARPS=10 ncu --set full --import-source on --clock-control none -k regex:k1_fused -s 1 -c 1 -o $o/k1_drain \
  python tools/profile_kernel.py --config cfg3 --shots 2000000 --tiled --what sample > $o/ncu.log 2>&1
python tools/ncu_summarize.py $o/k1_drain.ncu-rep > $o/summary.txt 2>&1
python tools/ncu_regions.py $o/k1_drain.ncu-rep > $o/regions.txt 2>&1
